"""Loads the in-tree C-ABI library libchunknet_b200.so (include/chunknet_b200.h).

There is no fallback: if the library is missing or cannot load, every
entry point raises.  Build it with `python -c "import __graft_entry__ as g;
g.build()"` or `make -C paper_2504_17307_b200/csrc`.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHUNKNET_B200_LIB") or os.path.join(HERE, "libchunknet_b200.so")

CN_OK = 0
STATUS_NAMES = {-1: "CN_E_INVALID", -2: "CN_E_LOGIC", -3: "CN_E_FIELD_RANGE",
                -4: "CN_E_OUT_OF_WINDOW", -5: "CN_E_CUDA", -6: "CN_E_UNSUPPORTED",
                -7: "CN_E_CAPACITY"}


class ChunknetError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ControlHeader(ctypes.Structure):
    _fields_ = [("conn_id", ctypes.c_uint8), ("msg_id", ctypes.c_uint8),
                ("csn", ctypes.c_uint8), ("last_chunk", ctypes.c_uint8),
                ("reserved", ctypes.c_uint8)]


class RxConfig(ctypes.Structure):
    _fields_ = [("chunk_bytes", ctypes.c_uint32), ("max_payload", ctypes.c_uint32),
                ("max_conns", ctypes.c_uint32), ("max_msgs", ctypes.c_uint32),
                ("chunk_pool", ctypes.c_uint64), ("arena_bytes", ctypes.c_uint64),
                ("max_batch", ctypes.c_uint32), ("carry_payload", ctypes.c_int32),
                ("reduce_op", ctypes.c_int32), ("max_posts", ctypes.c_uint32),
                ("ordered", ctypes.c_int32), ("pipeline", ctypes.c_int32)]


class PacketizeArgs(ctypes.Structure):
    _fields_ = [("len", ctypes.c_uint64), ("chunk_bytes", ctypes.c_uint32),
                ("max_payload", ctypes.c_uint32), ("src", ctypes.c_int32), ("dst", ctypes.c_int32),
                ("conn_id", ctypes.c_uint32), ("msg_id", ctypes.c_uint32),
                ("msg_seq", ctypes.c_uint64), ("tag", ctypes.c_uint64), ("tx_time", ctypes.c_int64),
                ("d_chunk_paths", ctypes.c_void_p), ("path", ctypes.c_int32),
                ("is_rtx", ctypes.c_int32)]


class TxConfig(ctypes.Structure):
    _fields_ = [("chunk_bytes", ctypes.c_uint32), ("max_payload", ctypes.c_uint32),
                ("dupack_threshold", ctypes.c_uint32), ("rtx_avoid_prev_path", ctypes.c_uint32),
                ("lb_policy", ctypes.c_int32), ("max_inflight_msgs", ctypes.c_uint32),
                ("max_paths", ctypes.c_uint32), ("log_cap", ctypes.c_uint32),
                ("rto_min", ctypes.c_int64), ("rto_max", ctypes.c_int64),
                ("commit_ahead", ctypes.c_int64), ("base_rtt_ns", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("stream_index0", ctypes.c_int64),
                ("chunk_pool", ctypes.c_uint64), ("cc_algo", ctypes.c_int32),
                ("drr_quantum", ctypes.c_uint32), ("mss", ctypes.c_int64), ("cap_bytes", ctypes.c_int64),
                ("swift_target_ns", ctypes.c_int64), ("init_cwnd_pkts", ctypes.c_double),
                ("receiver_driven", ctypes.c_int32), ("credit_quantum", ctypes.c_uint32),
                ("credit_bank_quanta", ctypes.c_int32), ("pad_rd", ctypes.c_int32),
                ("initial_credit", ctypes.c_int64), ("ordered", ctypes.c_int32),
                ("sent_order_cap", ctypes.c_uint32), ("policy", ctypes.c_int32), ("engines", ctypes.c_int32),
                ("conn_split", ctypes.c_int32), ("cc_scope", ctypes.c_int32), ("ecn_as_loss", ctypes.c_int32),
                ("pad_cc", ctypes.c_int32)]


class TxConnState(ctypes.Structure):
    _fields_ = [("credit", ctypes.c_int64), ("unchunked", ctypes.c_int64), ("inflight", ctypes.c_int64),
                ("n_paths", ctypes.c_int32), ("opened", ctypes.c_int32), ("home_engine", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class TxEngineState(ctypes.Structure):
    _fields_ = [("inflight_msgs", ctypes.c_int32), ("ring_len", ctypes.c_int32), ("dispatched", ctypes.c_uint64),
                ("gauge", ctypes.c_int64), ("committed_unsent", ctypes.c_int64)]


class RxResult(ctypes.Structure):
    _fields_ = [("n_acks", ctypes.c_uint32), ("n_completions", ctypes.c_uint32),
                ("status", ctypes.c_uint32), ("n_copied", ctypes.c_uint32),
                ("bytes_copied", ctypes.c_uint64)]


class RxUsage(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("pool_live", "pool_cap", "pool_allocated", "arena_live",
                                                "arena_blocks", "arena_allocated")]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ChunknetError(-5, f"{LIB_PATH} not built (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    L.cn_last_error.restype = ctypes.c_char_p
    L.cn_version.restype = ctypes.c_char_p
    L.cn_encode_header.argtypes = [ctypes.POINTER(ControlHeader), ctypes.POINTER(u32)]
    L.cn_decode_header.argtypes = [u32, ctypes.POINTER(ControlHeader)]
    L.cn_decode_header.restype = None
    L.cn_csn_before.argtypes = [ctypes.c_uint8, ctypes.c_uint8, ctypes.c_uint8, i32,
                                ctypes.POINTER(i32)]
    L.cn_rx_config_default.argtypes = [ctypes.POINTER(RxConfig)]
    L.cn_rx_config_default.restype = None
    L.cn_rx_create.argtypes = [ctypes.POINTER(RxConfig), ctypes.POINTER(vp)]
    L.cn_rx_destroy.argtypes = [vp]
    L.cn_rx_destroy.restype = None
    L.cn_rx_reset.argtypes = [vp, vp]
    if hasattr(L, "cn_rx_flush"):
        L.cn_rx_flush.argtypes = [vp, vp]
    L.cn_rx_batch.argtypes = [vp, vp, vp, u64, u32, vp, u32, vp, u32, vp, vp]
    L.cn_rx_batch_psn.argtypes = [vp, vp, vp, vp, u64, u32, vp, u32, vp, u32, vp, vp]
    if hasattr(L, "cn_rx_batch_packed"):
        L.cn_rx_batch_packed.argtypes = [vp, vp, vp, vp, vp, u32, vp, u32, vp, u32, vp, vp]
    if hasattr(L, "cn_rx_batch_msgdata"):
        L.cn_rx_batch_msgdata.argtypes = [vp, vp, vp, vp, u32, vp, u32, vp, u32, vp, vp]
    L.cn_rx_post.argtypes = [vp, u64, vp, u64, vp]
    L.cn_rx_arena.argtypes = [vp]
    L.cn_rx_arena.restype = vp
    L.cn_rx_arena_bytes.argtypes = [vp]
    L.cn_rx_arena_bytes.restype = u64
    L.cn_rx_last_launches.argtypes = [vp]
    L.cn_rx_get_usage.argtypes = [vp, ctypes.POINTER(RxUsage)]
    L.cn_rx_set_profiling.argtypes = [vp, i32]
    L.cn_rx_profile.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i32,
                                ctypes.POINTER(u64), i32]
    L.cn_rx_kernel_name.restype = ctypes.c_char_p
    L.cn_rx_kernel_name.argtypes = [i32]
    L.cn_sched_create.argtypes = [u32, u32, vp, ctypes.c_double, u64, ctypes.c_char_p,
                                  ctypes.c_int64, ctypes.POINTER(vp)]
    L.cn_sched_destroy.argtypes = [vp]
    L.cn_sched_destroy.restype = None
    L.cn_sched_boards.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.cn_sched_select.argtypes = [vp, i32, i32, vp, vp, vp, u32, u32, vp, vp]
    L.cn_sched_draws.argtypes = [vp, u32, vp, u64, vp, vp]
    L.cn_sched_record.argtypes = [vp, vp, vp, vp, vp, vp, u32, vp]
    L.cn_packet_count.restype = u64
    L.cn_packet_count.argtypes = [u64, u32, u32]
    L.cn_packetize.argtypes = [ctypes.POINTER(PacketizeArgs), vp, vp]
    L.cn_ipc_get_handle.argtypes = [vp, vp]
    L.cn_dev_alloc.argtypes = [u64, ctypes.POINTER(vp)]
    L.cn_dev_free.argtypes = [vp]
    L.cn_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
    L.cn_ipc_close.argtypes = [vp]
    L.cn_flag_signal.argtypes = [vp, vp, u64, vp]
    L.cn_flag_wait.argtypes = [vp, vp, u64, u64, vp, vp]
    if hasattr(L, "cn_flag_post"):
        L.cn_flag_post.argtypes = [vp, u64, vp]
    if hasattr(L, "cn_flag_wait_signal"):
        L.cn_flag_wait_signal.argtypes = [vp, u64, vp, u64, vp, u64, u64, vp, vp]
    L.cn_ctr_wait.argtypes = [vp, vp, u64, ctypes.c_int64, u64, vp, vp]
    L.cn_ctr_signal.argtypes = [vp, vp, u64, ctypes.c_int64, vp]
    L.cn_ctr_advance.argtypes = [vp, vp]
    L.cn_copy_async.argtypes = [vp, vp, u64, vp]
    L.cn_copy_sm.argtypes = [vp, vp, u64, u32, vp]
    if hasattr(L, "cn_copy_sm_signal"):
        L.cn_copy_sm_signal.argtypes = [vp, vp, u64, u32, vp, u64, vp, vp]
    L.cn_eqds_config_default.argtypes = [vp]
    L.cn_eqds_config_default.restype = None
    L.cn_eqds_create.argtypes = [vp, u32, ctypes.POINTER(vp)]
    L.cn_eqds_destroy.argtypes = [vp]
    L.cn_eqds_destroy.restype = None
    L.cn_eqds_run.argtypes = [vp, vp, vp, ctypes.c_int64, vp, vp, vp]
    L.cn_eqds_status.argtypes = [vp, u32, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)]
    L.cn_trace_tsv_bound.restype = u64
    L.cn_trace_tsv_bound.argtypes = [u64]
    L.cn_trace_scratch_bytes.restype = u64
    L.cn_trace_scratch_bytes.argtypes = [u64]
    L.cn_trace_format.argtypes = [vp, u64, vp, u64, vp, vp, vp]
    L.cn_trace_from_packets.argtypes = [vp, vp, u64, i32, i32, vp, vp]
    L.cn_trace_from_acks.argtypes = [vp, u64, i32, i32, vp, vp]
    _tx_protos(L)
    _lib = L
    return L


def _tx_protos(L):
    vp, u32 = ctypes.c_void_p, ctypes.c_uint32
    L.cn_last_error.restype = ctypes.c_char_p
    L.cn_tx_config_default.argtypes = [ctypes.POINTER(TxConfig)]
    L.cn_tx_config_default.restype = None
    L.cn_tx_create.argtypes = [ctypes.POINTER(TxConfig), u32, vp, vp, vp, ctypes.POINTER(vp)]
    L.cn_tx_destroy.argtypes = [vp]
    L.cn_tx_destroy.restype = None
    L.cn_tx_create_empty.argtypes = [ctypes.POINTER(TxConfig), u32, u32, ctypes.POINTER(vp)]
    L.cn_tx_open.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
    L.cn_tx_run.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int64, vp, vp, vp]
    L.cn_tx_status.argtypes = [vp, ctypes.POINTER(ctypes.c_uint)]
    L.cn_tx_n_hosts.argtypes = [vp]
    L.cn_tx_n_hosts.restype = u32
    L.cn_tx_conn_host.argtypes = [vp, u32]
    L.cn_tx_conn_host.restype = ctypes.c_int32
    L.cn_tx_log_counts.argtypes = [vp, vp]
    L.cn_tx_log_consume.argtypes = [vp, vp, vp]
    L.cn_tx_log_clear.argtypes = [vp, vp]
    L.cn_tx_get_conn_state.argtypes = [vp, u32, ctypes.POINTER(TxConnState), vp, u32]
    L.cn_tx_window_available.argtypes = [vp, u32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]
    L.cn_tx_get_engine_state.argtypes = [vp, u32, ctypes.c_int32, ctypes.POINTER(TxEngineState)]
    L.cn_tx_debug_state.argtypes = [vp, u32, vp, ctypes.c_uint64]
    L.cn_tx_debug_state.restype = ctypes.c_int64
    L.cn_libm_eval.argtypes = [ctypes.c_int, vp, vp, ctypes.c_uint64, vp]


USER_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchunknet_b200_user.so")
_user = None


def user_lib():
    """The sender engine built with the example policy plug-in
    (csrc/policies/example_policy.cuh, `make -C csrc user`): cn_tx_* only."""
    global _user
    if _user is None:
        if not os.path.exists(USER_LIB_PATH):
            raise ChunknetError(-5, f"{USER_LIB_PATH} not built (make -C csrc user)")
        L = ctypes.CDLL(USER_LIB_PATH)
        _tx_protos(L)
        _user = L
    return _user


def check(status, what="", L=None):
    if status != CN_OK:
        raise ChunknetError(status, f"{what}: {(L or lib()).cn_last_error().decode()}")
    return status


def exported_symbols():
    """Names declared in include/chunknet_b200.h (for the ABI load test)."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "chunknet_b200.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(cn_[a-z0-9_]+)\s*\(", src)))
