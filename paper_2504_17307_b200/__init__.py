"""chunknet-b200: B200-native hot path of the chunknet multipath transport
(arXiv 2504.17307; reference /root/reference/proj).

The compute path is libchunknet_b200.so (hand-written sm_100a CUDA behind
the C ABI in include/chunknet_b200.h).  This package is the host-side
mirror of the reference's Transport interface; it has no CPU fallback.
"""
from ._lib import ChunknetError, lib  # noqa: F401
from .scheduler import PathScheduler  # noqa: F401
from .transport import (MAX_PAYLOAD, RxBatch, Stats, Transport, TransportConfig,  # noqa: F401
                        csn_before, decode_header, encode_header, to_device_records)

__version__ = "0.1.0"
