/*
 * chunknet_b200.h -- C ABI of the B200-native hot path of the chunknet
 * multipath transport (arXiv 2504.17307, reference: /root/reference/proj).
 *
 * The boundary is plain C: opaque handles, integer status codes, plain
 * pointers + sizes.  No C++ exceptions and no torch types cross it.  Every
 * entry point names the reference interface it replaces (file:line into
 * /root/reference/proj).
 *
 * Device pointers are marked d_*; host pointers h_*.  Asynchronous calls
 * take a cudaStream_t passed as void* (NULL = legacy default stream) and
 * never synchronise the host unless documented.
 */
#ifndef CHUNKNET_B200_H
#define CHUNKNET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- constants */
/* NetParams::mtu / hdr_overhead defaults (include/chunknet/network.hpp:25-26):
 * 4096-byte MTU including a 64-byte header -> 4032 payload bytes/packet. */
#define CN_MTU 4096u
#define CN_HDR_OVERHEAD 64u
#define CN_MAX_PAYLOAD 4032u
/* kCsnWindow (src/transport.cpp:14): unacked chunks per message. */
#define CN_CSN_WINDOW 128
/* uint32_t packet bitmask per chunk (transport.hpp:195). */
#define CN_MAX_PKTS_PER_CHUNK 32
/* array<MsgRecv,128> / 7-bit msg_id (transport.hpp:222, wire.hpp:15). */
#define CN_MSG_SLOTS 128

/* ----------------------------------------------------------- status codes
 * The reference throws; the ABI returns one of these and records a message
 * retrievable with cn_last_error(). */
#define CN_OK 0
#define CN_E_INVALID (-1)       /* std::invalid_argument                   */
#define CN_E_LOGIC (-2)         /* std::logic_error (policy contract, ...)  */
#define CN_E_FIELD_RANGE (-3)   /* chunknet::FieldRangeError (wire.hpp:29)  */
#define CN_E_OUT_OF_WINDOW (-4) /* chunknet::OutOfWindowError (wire.hpp:37) */
#define CN_E_CUDA (-5)          /* CUDA runtime failure                     */
#define CN_E_UNSUPPORTED (-6)   /* input outside the device path's domain   */
#define CN_E_CAPACITY (-7)      /* a configured table/pool/output is full   */

/* Thread-local description of the last non-OK status. */
const char* cn_last_error(void);
/* Library version string and the sm arch it was compiled for. */
const char* cn_version(void);

/* ------------------------------------------------------------------ wire
 * ControlHeader (include/chunknet/wire.hpp:18-26): [31:24] conn_id,
 * [23:17] msg_id, [16:9] csn, [8] last_chunk, [7:0] reserved. */
typedef struct cn_control_header {
    uint8_t conn_id;
    uint8_t msg_id; /* 0..127 */
    uint8_t csn;
    uint8_t last_chunk; /* 0/1 */
    uint8_t reserved;
} cn_control_header;

/* encode_header (src/wire.cpp:5-14): CN_E_FIELD_RANGE if msg_id > 127. */
int cn_encode_header(const cn_control_header* h, uint32_t* out_word);
/* decode_header (src/wire.cpp:16-24). */
void cn_decode_header(uint32_t word, cn_control_header* out);
/* csn_before (src/wire.cpp:26-40) over SeqWindow{base, width}
 * (wire.hpp:47-62): CN_E_FIELD_RANGE for width outside [1,128],
 * CN_E_OUT_OF_WINDOW if a or b is outside the window. *out = 0/1. */
int cn_csn_before(uint8_t a, uint8_t b, uint8_t base, int width, int* out);

/* ------------------------------------------------------ packet records
 * The 64-byte per-packet header record: the reference's per-packet
 * hdr_overhead (network.hpp:26) carrying the 32-bit control word plus the
 * data fields of chunknet::Packet the receiver reads (packet.hpp:33-86). */
#define CN_PKT_RTX 0x1u     /* Packet::is_rtx  */
#define CN_PKT_ECN 0x2u     /* Packet::ecn     */
#define CN_PKT_TRIMMED 0x4u /* Packet::trimmed */
typedef struct cn_pkt_hdr {
    int32_t src;           /* source host            */
    int32_t dst;           /* destination host       */
    int32_t path_id;       /* path the packet took   */
    uint32_t hdr;          /* encode_header(ControlHeader) */
    uint64_t chunk_offset; /* byte offset of the chunk in its message */
    uint32_t chunk_len;    /* total chunk length     */
    uint16_t payload_len;  /* <= CN_MAX_PAYLOAD      */
    uint8_t seq_in_chunk;  /* < 32                   */
    uint8_t flags;         /* CN_PKT_*               */
    int64_t tx_time;       /* ns, echoed by acks     */
    uint64_t msg_seq;      /* per-connection message generation */
    uint64_t msg_tag;      /* caller's flow tag      */
    uint64_t msg_len;      /* total message length   */
} cn_pkt_hdr;

/* ACK record: the ack fields of chunknet::Packet (packet.hpp:73-79) as
 * built by Transport::send_ack (transport.cpp:763-792) or the stale re-ack
 * (transport.cpp:602-615). */
#define CN_ACK_CUM_VALID 0x1u
#define CN_ACK_ECN_ECHO 0x2u
/* the record is a trimmed-header NACK (transport.cpp:657-674): hdr = the
 * trimmed packet's header, cum_csn = nack_csn; no cum / SACK / echo */
#define CN_ACK_NACK 0x4u
/* receiver-driven mode (EQDS) control packets at the sender: a credit grant
 * (credit bytes in sack[0]) or an RTS acknowledgement */
#define CN_ACK_CREDIT 0x8u
#define CN_ACK_RTS_ACK 0x10u
/* ordered (go-back-N) reliability: a sequence-gap NACK (transport.cpp:
 * 690-707) with nack_psn = the receiver's expected sequence in sack[0];
 * CN_ACK_NACK_TRIM when a trimmed head-of-line packet caused it */
#define CN_ACK_GBN 0x20u
#define CN_ACK_NACK_TRIM 0x40u
typedef struct cn_ack_rec {
    int32_t src;          /* ack source = receiving host   */
    int32_t dst;          /* ack destination = sender host */
    uint32_t hdr;         /* conn_id | msg_id | csn = cause chunk csn */
    int32_t echo_path_id;
    uint8_t cum_csn;
    uint8_t flags;        /* CN_ACK_* */
    uint16_t reserved;
    uint32_t pkt_index;   /* index in the batch of the data packet that triggered it */
    uint64_t msg_seq;
    uint64_t sack[2];     /* SackBitmap, bit j = chunk cum+j complete */
    int64_t echo_tx_time;
    int64_t aux;          /* 0 from the device path (fixtures: delivery time) */
} cn_ack_rec;

/* One delivered message (Transport::maybe_deliver, transport.cpp:794-803). */
typedef struct cn_completion {
    uint64_t tag;
    int32_t src;
    int32_t dst;
    uint64_t len;
    uint64_t msg_seq;
    uint32_t pkt_index;   /* batch index of the packet that completed it */
    uint32_t msg_id;
    uint64_t buf_offset;  /* byte offset of the message in the rx arena */
    uint64_t bytes;       /* MsgRecv::bytes: payload bytes accepted */
    uint64_t reserved;    /* absolute device pointer of the message buffer */
} cn_completion;

/* ------------------------------------------------------------- receiver
 * Device-resident receive side of chunknet::Transport for the selective
 * (multipath) reliability mode with the reference's fixed-size chunking
 * (DefaultPolicy::on_chunk_size, policy.hpp:75-78).  Replaces, for a batch
 * of delivered data packets in arrival order:
 *   Transport::handle_packet/rconn_at   (transport.cpp:546-594)
 *   Transport::handle_data               (transport.cpp:596-688)
 *   Transport::accept_payload            (transport.cpp:719-730)
 *   Transport::chunk_completed           (transport.cpp:732-761)
 *   Transport::send_ack                  (transport.cpp:763-792)
 *   Transport::maybe_deliver             (transport.cpp:794-803)
 * State persists across batches: splitting a packet sequence into batches
 * yields the same ack stream as one batch. */
typedef struct cn_rx_config {
    uint32_t chunk_bytes;    /* TransportConfig::chunk_bytes (transport.hpp:27) */
    uint32_t max_payload;    /* Network::max_payload(); 0 = CN_MAX_PAYLOAD      */
    uint32_t max_conns;      /* receive connections (rounded up to pow2)        */
    uint32_t max_msgs;       /* concurrently live messages (rounded up to pow2) */
    uint64_t chunk_pool;     /* chunk state entries (sum of chunks of live msgs)*/
    uint64_t arena_bytes;    /* device bytes for reassembled message buffers    */
    uint32_t max_batch;      /* max packets per cn_rx_batch                     */
    int32_t carry_payload;   /* TransportConfig::carry_payload                  */
    int32_t reduce_op;       /* CN_REDUCE_*: fuse the scatter with a ring
                                reduction step            */
    uint32_t max_posts;      /* capacity of posted destinations (cn_rx_post)    */
    int32_t ordered;         /* TransportConfig::reliability == ordered: the
                                go-back-N receive filter (transport.cpp:690-717)
                                runs first; batches then come with conn_psn
                                (cn_rx_batch_psn) */
    int32_t pipeline;        /* 0: cn_rx_batch completes (in stream order) with
                                acks, completions AND payload final.  1:
                                pipelined receiver -- the payload scatter of
                                batch k runs on beside batch k+1's ingest and
                                ack path and is joined into the caller's
                                stream at the end of batch k+1 (an empty batch
                                or cn_rx_flush joins it at once).  Acks and
                                completion records of batch k are final when
                                batch k returns; its message bytes when batch
                                k+1 returns.  Inputs of batch k (headers,
                                payload) must stay valid until then. */
} cn_rx_config;

/* Reduce modes of the payload scatter: dst = dst + payload elementwise,
 * each element once (fp32; bf16 with fp32 add + round-to-nearest-even). */
#define CN_REDUCE_NONE 0
#define CN_REDUCE_SUM_F32 1
#define CN_REDUCE_SUM_BF16 2

typedef struct cn_rx cn_rx;

/* Fills *cfg with defaults (chunk_bytes 32768, 1024 conns, 4096 msgs,
 * 1<<22 chunks, 1 GiB arena, 1<<20 packets/batch, carry_payload 1). */
void cn_rx_config_default(cn_rx_config* cfg);
int cn_rx_create(const cn_rx_config* cfg, cn_rx** out);
void cn_rx_destroy(cn_rx* rx);
/* Forget every connection and message (fresh Transport receive state). */
int cn_rx_reset(cn_rx* rx, void* stream);
/* Pipelined receivers: joins the outstanding payload scatter into `stream`
 * (after it, every completed message's bytes are final).  No-op otherwise. */
int cn_rx_flush(cn_rx* rx, void* stream);

/* Batch result counters, written by the device (d_result). */
typedef struct cn_rx_result {
    uint32_t n_acks;
    uint32_t n_completions;
    uint32_t status;      /* 0 or CN_RXF_* bits */
    uint32_t n_copied;    /* packets whose payload was accepted */
    uint64_t bytes_copied;
} cn_rx_result;
#define CN_RXF_UNSUPPORTED 0x1u  /* trimmed pkt / non-fixed chunking / bad seq */
#define CN_RXF_ALIAS 0x2u        /* csn unwrap would alias */
#define CN_RXF_CAPACITY 0x4u     /* table/pool/arena/output overflow */
#define CN_RXF_GENERATION 0x8u   /* msg id reused before completion */

/* Process n data packets (arrival order).  d_payload + i*payload_stride
 * holds packet i's payload_len bytes; payload_stride == 0 means zero-copy
 * source addressing: packet i's payload is at d_payload + chunk_offset +
 * seq_in_chunk*max_payload (the sender's message buffer, e.g. a peer GPU's
 * memory over NVLink).  ACK records are appended in emission
 * order to d_acks (max_acks), completions to d_completions.  Asynchronous
 * on `stream`; d_result is written when the batch finishes. */
int cn_rx_batch(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const void* d_payload,
                uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks,
                uint32_t max_acks, cn_completion* d_completions,
                uint32_t max_completions, cn_rx_result* d_result,
                void* stream);
/* Packets that carry their message's data (Packet::msg_data: the
 * reference's send_message_data path, transport.hpp:88-91, copied from in
 * accept_payload, transport.cpp:719-730): packet i's payload is read at
 * d_msg_data[i] + chunk_offset + seq_in_chunk * max_payload -- each
 * packet names its message's device buffer (e.g. the sender's, over
 * NVLink).  A 0 entry is a packet without data: accepted and counted,
 * nothing copied (:722).  d_psn: conn_psn per packet for an ordered
 * receiver, NULL otherwise. */
int cn_rx_batch_msgdata(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                        const uint64_t* d_msg_data, uint32_t n, cn_ack_rec* d_acks,
                        uint32_t max_acks, cn_completion* d_completions,
                        uint32_t max_completions, cn_rx_result* d_result, void* stream);
/* Packed payloads: packet i's payload_len bytes at d_payload + d_offset[i]
 * (a NIC ring's variable-size packet buffers -- no stride padding to move
 * across PCIe).  d_psn as in cn_rx_batch_msgdata. */
int cn_rx_batch_packed(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                       const uint64_t* d_offset, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                       cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                       void* stream);
/* cn_rx_batch for ordered reliability: d_psn[i] = conn_psn of packet i
 * (Packet::conn_psn, packet.hpp:48; not part of the 64-B header record) */
int cn_rx_batch_psn(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                    uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                    cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                    void* stream);
/* Post a destination buffer for the message with caller tag `tag` (the
 * reference's per-message tag, transport.hpp:88-91): its payload is
 * scattered (or reduced, CN_REDUCE_*) into d_buf instead of the arena.
 * Posts persist across batches and resets; the completion's `reserved` field
 * carries the absolute destination pointer.  Asynchronous on `stream`. */
int cn_rx_post(cn_rx* rx, uint64_t tag, void* d_buf, uint64_t len, void* stream);
/* Device base pointer of the reassembly arena (cn_completion::buf_offset).
 * A delivered message's arena range stays valid until the cn_rx_batch after
 * the one that reported its completion has finished (the reference hands the
 * buffer to on_complete and frees it after, transport.cpp:794-803); post a
 * destination (cn_rx_post) to keep the data. */
void* cn_rx_arena(cn_rx* rx);
/* Bytes of the arena allocation: 2 x arena_bytes (the ring's capacity is
 * arena_bytes; a message's range runs contiguously past the ring's end into
 * the second half instead of wrapping).  The chunk pool is likewise stored
 * at 2 x chunk_pool entries. */
uint64_t cn_rx_arena_bytes(const cn_rx* rx);
/* Occupancy of the receiver's rings (synchronous: waits for the device).
 * Chunk-pool entries and 512-B arena blocks are allocated per
 * message, contiguously, and handed back when the message is delivered. */
typedef struct cn_rx_usage {
    uint64_t pool_live;        /* entries held by undelivered messages (+ ring padding) */
    uint64_t pool_cap;
    uint64_t pool_allocated;   /* entries allocated since create / reset */
    uint64_t arena_live;       /* arena blocks (512 B) held */
    uint64_t arena_blocks;
    uint64_t arena_allocated;
} cn_rx_usage;
int cn_rx_get_usage(cn_rx* rx, cn_rx_usage* out);
/* Number of kernel launches the last cn_rx_batch issued. */
int cn_rx_last_launches(const cn_rx* rx);
/* Optional per-kernel CUDA-event timing of cn_rx_batch (bench/profiling). */
int cn_rx_set_profiling(cn_rx* rx, int enable);
/* Synchronises profiled batches; ms[k] = accumulated milliseconds of
 * kernel k (names from cn_rx_kernel_name); returns the kernel count. */
int cn_rx_profile(cn_rx* rx, double* ms, int max, uint64_t* batches, int reset);
const char* cn_rx_kernel_name(int k);

/* ------------------------------------------------------------ scheduler
 * Batched multipath chunk scheduler: per-connection RngStream
 * (include/chunknet/rng.hpp:29-60; std::mt19937_64 + libstdc++ 13
 * uniform_int_distribution), PathScoreboard (lb.hpp:15-36) and
 * select_path (src/lb.cpp:7-27) / DefaultPolicy's on_select_path and
 * on_tx_rtx_chunk (policy.hpp:80-91), one warp per connection.
 * Path choices are bit-identical to the sequential reference. */
#define CN_LB_OBLIVIOUS 0 /* LbPolicy::oblivious (lb.hpp:39) */
#define CN_LB_P2_RTT 1    /* LbPolicy::p2_rtt                */
#define CN_LB_P2_ECN 2    /* LbPolicy::p2_ecn                */
typedef struct cn_sched cn_sched;

/* n_conns streams RngStream(seed, stream_name, index0 + c) -- the
 * reference's per-connection stream is ("transport.conn", conn idx),
 * transport.cpp:101; index0 < 0 = unindexed RngStream(seed, name).
 * Boards start at PathScoreboard(n_paths[c], base_rtt_ns). */
int cn_sched_create(uint32_t n_conns, uint32_t max_paths, const int32_t* h_n_paths,
                    double base_rtt_ns, uint64_t seed, const char* stream_name,
                    int64_t index0, cn_sched** out);
void cn_sched_destroy(cn_sched* s);
/* Device pointers to the [n_conns][max_paths] rtt / ecn score boards;
 * returns max_paths. */
int cn_sched_boards(cn_sched* s, double** d_rtt, double** d_ecn);
/* Path decisions, in order, for n_groups connections: group g is
 * connection d_conns[g] (NULL = g) with decisions
 * [d_offsets[g], d_offsets[g+1]) (NULL = uniform_count each, packed).
 * d_prev_paths[k] >= 0 marks a retransmission whose previous path is
 * avoided when rtx_avoid_prev_path (DefaultPolicy::on_tx_rtx_chunk);
 * -1 / NULL = fresh chunk (on_select_path).  A connection may appear in
 * at most one group per call. */
int cn_sched_select(cn_sched* s, int policy, int rtx_avoid_prev_path, const uint32_t* d_conns,
                    const uint32_t* d_offsets, const int32_t* d_prev_paths, uint32_t n_groups,
                    uint32_t uniform_count, int32_t* d_out, void* stream);
/* Raw RngStream outputs (d_ns == NULL: next_u64, else next_below(d_ns[i])). */
int cn_sched_draws(cn_sched* s, uint32_t conn, const uint64_t* d_ns, uint64_t count,
                   uint64_t* d_out, void* stream);
/* PathScoreboard::record_rtt + record_ecn for samples grouped per
 * connection (group g = samples [d_offsets[g], d_offsets[g+1]), applied in
 * order), as release_chunk does for RTT-sampled acks (transport.cpp:819-822). */
int cn_sched_record(cn_sched* s, const uint32_t* d_conn, const int32_t* d_path, const int64_t* d_rtt,
                    const uint8_t* d_ecn, const uint32_t* d_offsets, uint32_t n_groups, void* stream);

/* ------------------------------------------------------------ tx engine
 * Device sender (chunknet::Transport's sending half, transport.cpp:84-542,
 * 807-1169; RttEstimator cc.hpp:12-35; OpenLoop / CUBIC / Swift cc.cpp):
 * message dispatch over each host's engines (home engine or least-loaded
 * under conn_split), per-engine factory rotation and commit_ahead, per-path
 * tx / retransmission queues with DRR egress over each engine's ring,
 * window gating (global or per-path CC scope, credit in receiver-driven
 * mode), ack / NACK processing, duplicate-hint fast retransmit, RTO with
 * backoff, go-back-N.  Connections with the same src form one host (the
 * reference's HostState): one warp per host consumes the host's
 * time-ordered input events and fires the timers and deferred pumps the run
 * schedules.  Connection c draws its path choices from
 * RngStream("transport.conn", stream_index0 + c): number connections in the
 * order the reference creates them (first send_message per (src, dst)). */
/* congestion control on the device (CcConfig::Algo, cc.hpp:38-51).  CUBIC's
 * std::cbrt / std::pow are glibc 2.39's, restated bit-exactly. */
enum { CN_CC_NONE = 0, CN_CC_CUBIC = 1, CN_CC_SWIFT = 2 };
enum { CN_CC_SCOPE_GLOBAL = 0, CN_CC_SCOPE_PER_PATH = 1 };
typedef struct cn_tx_config {
    uint32_t chunk_bytes;         /* TransportConfig::chunk_bytes            */
    uint32_t max_payload;         /* 0 = CN_MAX_PAYLOAD                      */
    uint32_t dupack_threshold;    /* TransportConfig::dupack_threshold (8)   */
    uint32_t rtx_avoid_prev_path; /* TransportConfig::rtx_avoid_prev_path    */
    int32_t lb_policy;            /* CN_LB_*                                 */
    uint32_t max_inflight_msgs;   /* per engine (128)                        */
    uint32_t max_paths;           /* paths per connection (upper bound)      */
    uint32_t log_cap;             /* transmit records kept per host          */
    int64_t rto_min;              /* resolved Transport::rto_min_ (> 0)      */
    int64_t rto_max;              /* 0 = 64 * rto_min (transport.cpp:36)     */
    int64_t commit_ahead;         /* Transport::commit_ahead_ (:37-39)       */
    double base_rtt_ns;           /* scoreboard prior (Network::base_rtt_ns) */
    uint64_t seed;                /* Transport seed                          */
    int64_t stream_index0;        /* connection c uses stream index0 + c     */
    uint64_t chunk_pool;          /* chunk state entries; each connection owns
                                     chunk_pool / n_conns of them as a ring that
                                     a finished message hands back            */
    int32_t cc_algo;              /* CN_CC_*                                 */
    uint32_t drr_quantum;         /* TransportConfig::drr_quantum (32768)    */
    int64_t mss;                  /* CcConfig::mss (4032)                    */
    int64_t cap_bytes;            /* CcConfig::cap_bytes, 0 = uncapped       */
    int64_t swift_target_ns;      /* CcConfig::swift_target_ns (resolved)    */
    double init_cwnd_pkts;        /* CcConfig::init_cwnd_pkts (2.0)          */
    /* receiver-driven mode (EQDS glue, transport.cpp:1003-1074): credit
     * gates egress; RTS (logged as records with chunk = 0xFFFFFFFF, msg_seq =
     * demand, is_rtx = retransmissions queued) when credit runs out */
    int32_t receiver_driven;
    uint32_t credit_quantum;      /* TransportConfig::credit_quantum (32768) */
    int32_t credit_bank_quanta;   /* TransportConfig::credit_bank_quanta (4) */
    int32_t pad_rd;
    int64_t initial_credit;       /* resolved (-1 in the reference = one BDP) */
    /* ordered reliability (go-back-N, transport.cpp:433-494, 944-999,
     * 1144-1148): connection packet sequence, rewinds on NACK / RTO; a
     * resend starting mid-chunk is logged with (first packet << 16) in path */
    int32_t ordered;
    uint32_t sent_order_cap;      /* per-connection sent_order entries (0 = 65536) */
    /* transport policy plug-in (TransportPolicy / set_policy_factory,
     * policy.hpp:39-67): CN_POLICY_*; hooks in include/chunknet_policy.cuh */
    int32_t policy;
    int32_t engines;              /* TransportConfig::engines per host (1..16) */
    int32_t conn_split;           /* TransportConfig::conn_split              */
    int32_t cc_scope;             /* CcConfig::scope: CN_CC_SCOPE_*           */
    int32_t ecn_as_loss;          /* CcConfig::ecn_as_loss (CUBIC)            */
    int32_t pad_cc;
} cn_tx_config;
enum {
    CN_POLICY_DEFAULT = 0,      /* DefaultPolicy with lb_policy / rtx_avoid_prev_path */
    CN_POLICY_ROUND_ROBIN = 1,  /* cn_policy::RoundRobinPolicy */
    CN_POLICY_SINGLE_PATH = 2,  /* cn_policy::SinglePathPolicy */
    CN_POLICY_TEST_OUT_OF_RANGE = 3,
    CN_POLICY_USER = 100        /* CnUserPolicy of a `make USER_POLICY=...` build */
};
/* cn_tx_status bits */
#define CN_TX_STATUS_EMPTY_MSG 1u  /* send_message of 0 bytes (invalid_argument) */
#define CN_TX_STATUS_CAPACITY 4u   /* chunk ring / engine ring full */
#define CN_TX_STATUS_RETRY 8u      /* RTS retry queue full */
#define CN_TX_STATUS_STALE 16u     /* stale retransmission-queue entries overflow */
#define CN_TX_STATUS_SENT_ORDER 32u /* go-back-N sent_order overflow */
#define CN_TX_STATUS_POLICY 64u    /* policy contract violation (logic_error) */
#define CN_TX_STATUS_LOG 128u      /* a host logged more than log_cap records: some were lost */
#define CN_TX_STATUS_TIMER 256u    /* more than 8 RTO events armed at one instant */
#define CN_TX_STATUS_INTERNAL 512u /* event for an unknown connection / corrupt chunk state */
typedef struct cn_tx_submit { int64_t t; uint64_t len; uint64_t tag; } cn_tx_submit;
/* one chunk transmission (send_chunk): time, message, chunk index, path,
 * and the connection (cn_tx_create index) and destination it belongs to */
typedef struct cn_tx_rec {
    int64_t t;
    uint32_t msg_id;
    uint32_t chunk;
    int32_t path;
    int32_t is_rtx;
    uint64_t msg_seq;
    uint32_t conn;
    int32_t dst;
} cn_tx_rec;
typedef struct cn_tx_stats {  /* Transport::Stats sender fields (per connection) + estimator */
    uint64_t chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_sent, msgs_completed, backpressured, n_log;
    int64_t srtt, rttvar;     /* subs[0]'s RttEstimator */
    int32_t backoff, live_msgs;
    int64_t cwnd_bytes;   /* subs[0]'s CongestionControl::cwnd_bytes() at the end */
    int64_t inflight;     /* the connection's total inflight at the end */
    double cwnd_pkts;     /* subs[0]'s window in packets (CUBIC / Swift) */
    uint64_t rts_sent, decreases;
} cn_tx_stats;
typedef struct cn_tx cn_tx;
void cn_tx_config_default(cn_tx_config* cfg);
/* h_src: host of each connection (NULL: one host per connection); h_dst,
 * h_n_paths (NULL: 0, max_paths).  Connection indices are cn_tx_create
 * order; hosts are numbered by first appearance in h_src. */
int cn_tx_create(const cn_tx_config* cfg, uint32_t n_conns, const int32_t* h_src, const int32_t* h_dst,
                 const int32_t* h_n_paths, cn_tx** out);
/* An engine whose connections open one at a time, as the reference's
 * conn_to creates them (first send_message per (src, dst)): cn_tx_open
 * returns the new connection's index (>= 0) or a negative status. */
int cn_tx_create_empty(const cn_tx_config* cfg, uint32_t max_conns, uint32_t max_conns_per_host, cn_tx** out);
int cn_tx_open(cn_tx* t, int32_t src, int32_t dst, int32_t n_paths);
void cn_tx_destroy(cn_tx* t);
uint32_t cn_tx_n_hosts(cn_tx* t);
int32_t cn_tx_conn_host(cn_tx* t, uint32_t conn);
/* Events of host h are d_events[d_ev_off[h] .. d_ev_off[h+1]), each
 * (type << 62) | (conn << 40) | index: type 0 = d_submits[index] (a
 * send_message on connection conn), 1 = d_acks[index] (an ack / NACK /
 * credit / rts_ack delivered at the host for connection conn; aux = time),
 * ordered by time (ties: in list order).  Timers fire up to end_time.
 * d_log holds log_cap records per host (emission order), d_stats one record
 * per connection.  State persists across calls. */
int cn_tx_run(cn_tx* t, const uint32_t* d_ev_off, const uint64_t* d_events,
              const cn_tx_submit* d_submits, const cn_ack_rec* d_acks, int64_t end_time,
              cn_tx_rec* d_log, cn_tx_stats* d_stats, void* stream);
int cn_tx_status(cn_tx* t, unsigned int* out);
/* Connection / engine state for introspection (Transport::path_inflight,
 * conn_credit, window_available, engine_*, transport.cpp:1173-1209);
 * synchronous. */
typedef struct cn_tx_conn_state {
    int64_t credit;     /* Connection::credit (receiver-driven bank) */
    int64_t unchunked;  /* dispatched bytes not yet chunked */
    int64_t inflight;   /* sum of the paths' inflight (outstanding_bytes) */
    int32_t n_paths;
    int32_t opened;     /* conn_to ran (first send_message) */
    int32_t home_engine;
    int32_t pad;
} cn_tx_conn_state;
int cn_tx_get_conn_state(cn_tx* t, uint32_t conn, cn_tx_conn_state* out,
                         int64_t* h_path_inflight /* [n_paths] or NULL */, uint32_t max_paths);
int cn_tx_window_available(cn_tx* t, uint32_t conn, int32_t path, int64_t* out);
typedef struct cn_tx_engine_state {
    int32_t inflight_msgs, ring_len;
    uint64_t dispatched;
    int64_t gauge, committed_unsent;
} cn_tx_engine_state;
/* engine `engine` of the host connection `conn` belongs to */
int cn_tx_get_engine_state(cn_tx* t, uint32_t conn, int32_t engine, cn_tx_engine_state* out);
/* Diagnostics: the raw device state of one connection (its shared-memory
 * image, global state, host image, chunk state of its pool share); returns
 * the byte count (pass h_out = NULL to size). */
int64_t cn_tx_debug_state(cn_tx* t, uint32_t conn, void* h_out, uint64_t cap);
/* Transmit records logged per host so far (host array of n_hosts, counting
 * records lost to log_cap); cn_tx_log_consume drops the first h_n[h]
 * records of each host's log (moving the rest to the front);
 * cn_tx_log_clear restarts every log at 0. */
int cn_tx_log_counts(cn_tx* t, uint32_t* h_out);
int cn_tx_log_consume(cn_tx* t, cn_tx_rec* d_log, const uint32_t* h_n);
int cn_tx_log_clear(cn_tx* t, void* stream);
/* The device restatement of glibc's cbrt (mode 0) / pow(x, 3.0) (mode 1)
 * that CUBIC uses, over n doubles (parity hook) */
int cn_libm_eval(int mode, const double* d_in, double* d_out, uint64_t n, void* stream);

/* --------------------------------------------------------- send side
 * Transport::send_chunk's packetization (transport.cpp:433-494) for all
 * chunks of one message (DefaultPolicy chunking, policy.hpp:75-78): packet
 * i of chunk c carries min(max_payload, chunk_len - i*max_payload) bytes at
 * message offset c*chunk_bytes + i*max_payload; header {conn_id, msg_id,
 * csn = c & 0xFF, last = (c == nchunks-1)}.  Records are written in chunk
 * order (the order send_chunk injects them). */
typedef struct cn_packetize_args {
    uint64_t len;            /* message length (> 0; send_message throws on 0) */
    uint32_t chunk_bytes;
    uint32_t max_payload;    /* 0 = CN_MAX_PAYLOAD */
    int32_t src, dst;
    uint32_t conn_id, msg_id;
    uint64_t msg_seq, tag;
    int64_t tx_time;
    const int32_t* d_chunk_paths; /* path per chunk (cn_sched_select), or NULL */
    int32_t path;            /* path of every chunk when d_chunk_paths == NULL */
    int32_t is_rtx;
} cn_packetize_args;
uint64_t cn_packet_count(uint64_t len, uint32_t chunk_bytes, uint32_t max_payload);
int cn_packetize(const cn_packetize_args* a, cn_pkt_hdr* d_out, void* stream);

/* ------------------------------------------------- multi-GPU plumbing
 * CUDA IPC mappings of a peer rank's device buffers (NVLink P2P): 64-byte
 * opaque handles exchanged by the host (torch.distributed in the Python
 * driver). */
int cn_ipc_get_handle(void* d_ptr, void* out64);  /* d_ptr must be an allocation base */
/* Whole-allocation device buffers (zeroed) for IPC sharing. */
int cn_dev_alloc(uint64_t bytes, void** d_ptr);
int cn_dev_free(void* d_ptr);
int cn_ipc_open(const void* handle64, void** d_ptr);
int cn_ipc_close(void* d_ptr);
/* Progress flags between neighbouring ranks: signal = system-scope release
 * store of `value` into up to two (peer) flag words; wait = bounded acquire
 * spin until both local words are >= value (sets *d_err on timeout). */
int cn_flag_signal(unsigned long long* d_a, unsigned long long* d_b, uint64_t value, void* stream);
int cn_flag_wait(const unsigned long long* d_a, const unsigned long long* d_b, uint64_t value,
                 uint64_t max_spins, unsigned int* d_err, void* stream);
/* A notification that publishes no data ("my receive slot is free"): a
 * relaxed system-scope store of value into *d_a, no fence (the stream's
 * earlier kernels have completed). */
int cn_flag_post(unsigned long long* d_a, uint64_t value, void* stream);
/* One kernel for a wait followed by a notice: spin until *d_wa >= va and
 * *d_wb >= vb (a null pointer is met), then, if d_s, store vs into *d_s
 * as cn_flag_post does (a consumption notice: it publishes no data).
 * Saves a launch on the all-to-all's per-piece handshakes. */
int cn_flag_wait_signal(const unsigned long long* d_wa, uint64_t va, const unsigned long long* d_wb,
                        uint64_t vb, unsigned long long* d_s, uint64_t vs, uint64_t max_spins,
                        unsigned int* d_err, void* stream);
/* Graph-replayable progress counters.  Targets are relative to a device
 * iteration counter *d_iter: target = *d_iter * per_iter + offset (offset
 * may be negative; targets below 0 are met).  wait spins (acquire, system
 * scope) until *d_flag >= target; signal stores target into (peer) *d_flag
 * (release, system scope); advance adds 1 to *d_iter. */
int cn_ctr_wait(const unsigned long long* d_flag, const unsigned long long* d_iter, uint64_t per_iter,
                int64_t offset, uint64_t max_spins, unsigned int* d_err, void* stream);
int cn_ctr_signal(unsigned long long* d_flag, const unsigned long long* d_iter, uint64_t per_iter,
                  int64_t offset, void* stream);
int cn_ctr_advance(unsigned long long* d_iter, void* stream);
/* Bulk device-to-device copy on a stream (the copy engines; a peer pointer
 * from cn_ipc_open makes it an NVLink transfer -- the "wire" that delivers
 * a message's payload into the receiver's staging slot). */
int cn_copy_async(void* d_dst, const void* d_src, uint64_t bytes, void* stream);
/* The same transfer driven by SM threads (16-byte aligned pointers and size;
 * blocks = 0 picks one per SM): posted NVLink writes beside the copy engines. */
int cn_copy_sm(void* d_dst, const void* d_src, uint64_t bytes, uint32_t blocks, void* stream);
/* cn_copy_sm whose last block then raises a progress flag as cn_flag_signal
 * does (release-store of value into *d_flag, system scope), saving the
 * separate signal launch.  d_ctr: a zeroed device word private to the
 * stream, left zero again. */
int cn_copy_sm_signal(void* d_dst, const void* d_src, uint64_t bytes, uint32_t blocks,
                      unsigned long long* d_flag, uint64_t value, unsigned int* d_ctr, void* stream);

/* -------------------------------------------------------- transport
 * One object in the shape of chunknet::Transport (transport.hpp:53-107):
 * the sender engine (cn_tx) for every connection it opens plus the receive
 * path (cn_rx), driven by the caller's clock.  The reference's synchronous
 * calls become queued events: send_message / handle_acks queue at their
 * time, cn_transport_advance runs the device sender up to a time, and the
 * transmissions, acks and completions are polled.  Every TransportConfig
 * the reference accepts is supported: engines (home or conn_split
 * dispatch), selective or ordered reliability (ordered: one path, data
 * through cn_transport_handle_data_psn), the policies of
 * chunknet_policy.cuh, CC none / CUBIC / Swift with global or per-path
 * scope, sender- or receiver-driven (credit and rts_ack records through
 * cn_transport_handle_acks; initial_credit resolved to one BDP by the
 * caller).  Connections open in the order send_message first names them
 * (conn_to), which fixes their RngStream index: call send_message in time
 * order. */
typedef struct cn_transport_config {
    /* TransportConfig (transport.hpp:23-51) */
    int32_t engines, conn_split, paths;
    uint32_t chunk_bytes;
    int32_t lb, reliability, receiver_driven, max_inflight_msgs;
    int64_t rto_min, rto_max;            /* resolved (0 rto_max = 64 x rto_min) */
    uint32_t drr_quantum;
    int32_t rtx_avoid_prev_path, dupack_threshold, carry_payload;
    int64_t initial_credit;
    uint32_t credit_quantum;
    int32_t credit_bank_quanta;
    /* CcConfig (cc.hpp:37-51) */
    int32_t cc_algo, cc_scope;
    int64_t mss, cap_bytes;
    int32_t ecn_as_loss, pad0;
    int64_t swift_target_ns;
    double init_cwnd_pkts;
    /* what the reference reads from its Network */
    double base_rtt_ns;                  /* scoreboard prior */
    int64_t commit_ahead;                /* max(2 chunk, 2 quantum, BDP) (transport.cpp:37-39) */
    /* device capacities */
    uint32_t max_conns, max_batch, log_cap;
    int32_t policy;                      /* CN_POLICY_* (set_policy_factory, transport.hpp:95) */
    uint64_t chunk_pool, arena_bytes;
    uint32_t max_conns_per_host;         /* connections one source host may open (0 = as many as fit) */
    uint32_t pad_mcph;
} cn_transport_config;
typedef struct cn_stats {  /* Transport::Stats (transport.hpp:62-75) */
    uint64_t msgs_sent, msgs_completed, backpressured, chunks_sent, chunk_rtx, fast_rtx, rtos,
        acks_sent, nacks_sent, rts_sent, credit_pkts, delivered_msgs;
} cn_stats;
typedef struct cn_transport cn_transport;
void cn_transport_config_default(cn_transport_config* cfg);
int cn_transport_create(const cn_transport_config* cfg, uint64_t seed, cn_transport** out);
void cn_transport_destroy(cn_transport* h);
/* Transport::send_message (transport.hpp:88) at time t: opens the (src,
 * dst) connection on first use (conn_to order = RngStream index); returns 1
 * when queued (backpressure is counted in the stats when the engine runs). */
int cn_transport_send_message(cn_transport* h, int32_t src, int32_t dst, uint64_t len, uint64_t tag, int64_t t);
/* conn_to ahead of the first send_message, with the connection's path count
 * min(paths, topology path_count(src, dst)) (transport.cpp:97-99) -- the
 * caller owns the topology; returns the connection index */
int32_t cn_transport_open_conn(cn_transport* h, int32_t src, int32_t dst, int32_t n_paths);
/* acks and trimmed-header NACKs delivered at the senders (host records, aux = time) */
int cn_transport_handle_acks(cn_transport* h, const cn_ack_rec* acks, uint32_t n);
/* EventQueue::run_until(until): the queued inputs with t <= until and the
 * timers up to `until` (later inputs stay queued for the next advance) */
int cn_transport_advance(cn_transport* h, int64_t until, void* stream);
/* transmissions since the last poll, per connection in emission order;
 * conn_out[i] = connection index of out[i] (optional) */
int64_t cn_transport_poll_transmissions(cn_transport* h, cn_tx_rec* out, uint64_t cap, int32_t* conn_out);
/* Transport::handle_packet for a batch of delivered data packets (device records) */
int cn_transport_handle_data(cn_transport* h, const cn_pkt_hdr* d_hdrs, const void* d_payload, uint64_t stride,
                             uint32_t n, void* stream);
/* ... with each packet's conn_psn (d_psn[n]), required under ordered
 * reliability (TransportConfig::reliability = ordered, go-back-N) */
int cn_transport_handle_data_psn(cn_transport* h, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                                 const void* d_payload, uint64_t stride, uint32_t n, void* stream);
/* ... with each packet's message data pointer (d_msg_data[n], see
 * cn_rx_batch_msgdata): the send_message_data path, where a packet carries
 * its message's data (transport.hpp:88-91) -- the caller's injection code
 * sets it per packet as send_chunk sets Packet::msg_data (transport.cpp:486);
 * d_psn as in cn_transport_handle_data_psn or NULL */
int cn_transport_handle_data_msgdata(cn_transport* h, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                                     const uint64_t* d_msg_data, uint32_t n, void* stream);
/* the last batch's ack / NACK records and completions (host copies) */
int64_t cn_transport_poll_acks(cn_transport* h, cn_ack_rec* out, uint64_t cap);
int64_t cn_transport_poll_completions(cn_transport* h, cn_completion* out, uint64_t cap);
int cn_transport_stats(cn_transport* h, cn_stats* out);
int32_t cn_transport_conn_index(cn_transport* h, int32_t src, int32_t dst);
/* outstanding_bytes (transport.hpp:102): the connection's gated inflight */
int64_t cn_transport_outstanding_bytes(cn_transport* h, int32_t src, int32_t dst);
/* the rest of the reference's introspection (transport.hpp:101-107), as of
 * the last cn_transport_advance; 0 for an unknown connection or path */
int64_t cn_transport_path_inflight(cn_transport* h, int32_t src, int32_t dst, int32_t path);
int64_t cn_transport_window_available(cn_transport* h, int32_t src, int32_t dst, int32_t path);
int64_t cn_transport_conn_credit(cn_transport* h, int32_t src, int32_t dst);
int32_t cn_transport_engine_inflight_msgs(cn_transport* h, int32_t host, int32_t engine);
uint64_t cn_transport_engine_dispatched(cn_transport* h, int32_t host, int32_t engine);
int64_t cn_transport_engine_gauge(cn_transport* h, int32_t host, int32_t engine);

/* ------------------------------------------------------------- EQDS
 * The receiver-driven pull pacer (EqdsReceiver, eqds.cpp:7-104), one per
 * receiving host, run on the device over each receiver's time-ordered input
 * stream.  cn_eqds_config mirrors EqdsParams (eqds.hpp) as Transport builds
 * it (transport.cpp:45-73): quantum = credit_quantum, tick_ns =
 * ser(quantum + pkts * hdr_overhead), bank_cap = credit_bank_quanta * quantum. */
enum { CN_EQ_RTS = 0, CN_EQ_CHUNK = 1, CN_EQ_TRIM = 2 };
typedef struct cn_eqds_config {
    uint32_t quantum;
    int32_t grant_to_idle;
    int64_t tick_ns;
    int64_t bank_cap;
    uint32_t max_senders;  /* distinct senders per receiver */
    uint32_t queue_cap;    /* entries per service list (stale ones included) */
    uint32_t log_cap;      /* log records per receiver and run */
    uint32_t reserved;
} cn_eqds_config;
/* on_rts(sender, demand = arg, rtx = flag) / on_chunk(sender, bytes = arg,
 * was_rtx = flag) / on_trim(sender, chunk_len = arg) at time t */
typedef struct cn_eqds_event { int64_t t; int32_t type; int32_t sender; uint64_t arg; int32_t flag; int32_t pad; } cn_eqds_event;
/* kind 0: grant of `bytes` credit to sender; kind 1: rts_ack to sender */
typedef struct cn_eqds_log { int64_t t; int32_t sender; uint32_t bytes; int32_t kind; int32_t pad; } cn_eqds_log;
typedef struct cn_eqds cn_eqds;
void cn_eqds_config_default(cn_eqds_config* cfg);
int cn_eqds_create(const cn_eqds_config* cfg, uint32_t n_receivers, cn_eqds** out);
void cn_eqds_destroy(cn_eqds* h);
/* Events of receiver r are d_events[d_ev_off[r] .. d_ev_off[r+1]), ordered
 * by time (ties: list order); ticks fire up to end_time.  d_log holds
 * log_cap records per receiver, d_log_n the count per receiver.  State
 * persists across runs. */
int cn_eqds_run(cn_eqds* h, const uint32_t* d_ev_off, const cn_eqds_event* d_events, int64_t end_time,
                cn_eqds_log* d_log, uint32_t* d_log_n, void* stream);
/* status bits: 1 sender table full, 2 service list overflow, 4 log truncated */
int cn_eqds_status(cn_eqds* h, uint32_t receiver, uint32_t* status, uint64_t* grants_sent);

/* ------------------------------------------------------------ trace
 * The reference's packet trace (experiment.cpp:18-40 trace_line over
 * network.hpp:30-35 TraceEvent), one TSV line per record:
 *   <t>\t<event>\t<link_id>\t<src>><dst>:<path_id>\t<csn>\t<kind>[,rtx][,ecn][,trim][,last]\n
 * formatted on the device, byte-identical, in record order. */
enum { CN_TEV_DELIVER = 0, CN_TEV_DROP = 1, CN_TEV_TRIM = 2, CN_TEV_LOSS = 3, CN_TEV_HDR_DROP = 4 };
enum { CN_PK_DATA = 0, CN_PK_ACK = 1, CN_PK_NACK = 2, CN_PK_CREDIT = 3, CN_PK_RTS = 4, CN_PK_RTS_ACK = 5 };
enum { CN_TRF_RTX = 1, CN_TRF_ECN = 2, CN_TRF_TRIM = 4, CN_TRF_LAST = 8 };
typedef struct cn_trace_rec {
    int64_t t;        /* TraceEvent::t                              */
    int32_t link_id;  /* -1 = host delivery                         */
    int32_t src, dst, path_id;
    uint8_t csn, event, kind, flags;  /* CN_TEV_*, CN_PK_*, CN_TRF_* */
    uint32_t reserved;
} cn_trace_rec;
uint64_t cn_trace_tsv_bound(uint64_t n);      /* output bytes that always suffice */
uint64_t cn_trace_scratch_bytes(uint64_t n);  /* device scratch for cn_trace_format */
/* Writes the lines (at most cap bytes) and the full length into *d_len. */
int cn_trace_format(const cn_trace_rec* d_recs, uint64_t n, char* d_out, uint64_t cap, uint64_t* d_len,
                    void* d_scratch, void* stream);
/* Data packets as trace records (t = d_times[i], or tx_time when NULL). */
int cn_trace_from_packets(const cn_pkt_hdr* d_hdrs, const int64_t* d_times, uint64_t n, int32_t event,
                          int32_t link_id, cn_trace_rec* d_out, void* stream);
/* Ack records as trace records (t = aux, the delivery time; path 0 as send_ack leaves it). */
int cn_trace_from_acks(const cn_ack_rec* d_acks, uint64_t n, int32_t event, int32_t link_id,
                       cn_trace_rec* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CHUNKNET_B200_H */
