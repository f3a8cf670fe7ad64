// tx.cu -- device sender engine: ack processing, loss detection,
// retransmission, congestion control and window-gated egress of the
// selective multipath transport (sm_100a).
//
// Restates, per connection, the reference sender's event handling
// (/root/reference/proj/src/transport.cpp):
//   send_message / dispatch          :144-218   (msg ids LIFO, :127-129)
//   pump / commit_chunks             :232-310   (factory rotation, 128-chunk
//                                                window stall, commit_ahead,
//                                                path bound at commit)
//   can_send / gated_inflight        :312-325   (global CC scope)
//   egress                           :329-431   (retransmission queues in
//                                                ring order, then deficit
//                                                round robin over the ring)
//   send_chunk                       :433-494   (attempts, tx_time, deadline)
//   queue_rtx                        :516-542   (path via on_tx_rtx_chunk)
//   release_chunk / advance / finish :807-847
//   handle_ack                       :849-942   (cause release + RTT sample,
//                                                cumulative + SACK release,
//                                                dup hints -> fast retransmit)
//   handle_nack                      :944-965   (trimmed-header NACK -> rtx)
//   cur_rto / arm_rto / rto_fire     :1078-1169 (backoff x2 capped at 64)
//   RttEstimator                     cc.hpp:12-35
//   OpenLoop / Swift                 cc.cpp:19-34, :108-156
// for one engine per host, global CC scope, DefaultPolicy (no pacing).
// Swift is device-exact: its update uses IEEE double + - * / only, each
// rounded explicitly (__d*_rn, no contraction), in the reference's
// evaluation order.  CUBIC stays host-side: std::cbrt has no bit-identical
// device counterpart.
//
// One warp per connection consumes a time-ordered stream of events (message
// submissions, acks delivered at the sender) and fires its own RTO timer in
// between (timers scheduled during the run fire after same-time events).
// Control flow is warp-uniform; chunk-window scans run one chunk per lane
// with ballots; per-path inflight, deficits and queue depths sit in shared
// memory; path choices come from the connection's RngStream (rng.cuh),
// bit-identical to the reference.
//
// Queues.  Each chunk carries a queue tag c_q = kind | seq (seq from a
// per-connection counter, 0 = not queued).  The front of path p's tx or
// retransmission queue is the queued chunk of that kind on p with the
// smallest seq -- the reference's FIFO order.  The reference's queues can
// also hold stale entries (a chunk acked while awaiting retransmission);
// egress pops those without effect, and a stale entry never outlives the
// next egress that sends a fresh chunk (every rtx queue is drained first
// while the window is open), so it can never alias a reused message id.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <new>
#include <string>
#include <vector>

#include "chunknet_policy.cuh"
#include "common.cuh"
#include "rng.cuh"
#ifdef CN_TX_USER_POLICY_HEADER
#include CN_TX_USER_POLICY_HEADER  // defines struct CnUserPolicy (make USER_POLICY=...)
#endif

namespace cnb {

enum : uint32_t { TF_SENT = 1, TF_ACKED = 2, TF_RTXP = 4 };
constexpr uint32_t kQRtx = 0x80000000u;  // c_q kind bit: retransmission queue
constexpr int kTxWindow = 128;           // kCsnWindow (transport.cpp:14)
constexpr int kBackoffCap = 64;          // kBackoffCap (transport.cpp:15)
constexpr int kTxWarps = 4;
constexpr uint32_t kRetryMax = 32;  // pending RTS retry events per connection
constexpr uint32_t kStaleMax = 256;  // stale retransmission-queue entries per connection
constexpr int64_t kNeverDecreased = LLONG_MIN / 2;  // cc.cpp:17
// cc.cpp:11-16
constexpr double kSwiftAi = 1.0, kSwiftMdScale = 0.8, kSwiftMaxMd = 0.5, kMinCwndPkts = 1.0;

struct TxMsg {
    uint64_t seq, tag, len, chunked, chunk_base;
    uint32_t nchunks, base, acked, live, in_factory, pad0;
};

struct TxConn {
    int64_t srtt, rttvar, armed_at, timer_at, committed_unsent, total_inflight, last_decrease;
    uint64_t next_seq, chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_sent, msgs_completed, backpressured,
        ring_pos;
    double w;  // Swift window, packets
    int32_t has_sample, backoff, timer_armed, n_free, fq_head, fq_count, src, dst, conn_id,
        n_paths, live_msgs, ring_len;
    uint32_t q_seq, pump_pending;
    int64_t pump_at;
    // receiver-driven mode (EQDS sender glue, transport.cpp:1003-1074)
    int64_t credit, unchunked, rtxq_bytes;
    uint32_t rts_outstanding, rts_acked, sched_seq, timer_seq, pump_seq, retry_head, retry_n, stale_n;
    int64_t retry_t[kRetryMax];
    uint32_t retry_seq[kRetryMax];
    uint64_t next_psn, last_rewind_psn;  // ordered reliability (go-back-N)
    uint32_t so_n, gq_head, gq_n, pad_gq;   // sent_order refs; gbn_rtxq ring
    uint32_t stale_seq[kStaleMax];  // acked-while-pending rtx queue entries: (queue seq, path)
    uint16_t stale_path[kStaleMax];
    uint32_t live_mask[4];  // message slots in use (bit = msg id)
    uint64_t p_head;        // chunk ring head (monotonic); the tail is the oldest live message
    uint64_t pol_state[4];  // the connection's policy instance (chunknet_policy.cuh)
    uint64_t p_start[128];  // ring position (monotonic) of each live message's chunks
    uint8_t free_ids[128];
    uint8_t fq[128];
    TxMsg msgs[128];
};

struct TxDev {
    uint32_t n_conns, cb, max_pl, dupack, avoid_prev, policy, max_inflight, log_cap, cc_algo, quantum;
    uint32_t rd, ordered, so_cap;
    int32_t pol;  // CN_POLICY_*
    int64_t rto_min, rto_max, commit_ahead, swift_target, mss, cap_bytes, credit_cap, initial_credit;
    double init_cwnd, cap_pkts;
    uint64_t pool_cap, conn_pool;  // conn_pool = pool_cap / n_conns entries per connection
    TxConn* conns;
    int32_t* c_path;
    int64_t* c_txt;
    int64_t* c_dead;
    int32_t* c_att;
    uint32_t* c_fl;
    int32_t* c_dup;
    uint32_t* c_q;
    int64_t* c_psn;     // [pool] ChunkTx::psn_base (ordered)
    uint32_t* so_ref;   // [conn][so_cap] Connection::sent_order, (msg id << 25) | chunk
    uint32_t* gq_ref;   // [conn][so_cap] Connection::gbn_rtxq refs
    uint64_t* gq_from;  // [conn][so_cap] ... and their resend-from sequence
    // per connection x path (SubConn, transport.hpp), persisted across runs
    int64_t* s_inflight;
    int64_t* s_deficit;
    uint32_t* s_txq;
    uint32_t* s_rtxq;
    uint16_t* s_ring;  // engine ring: paths in order of first use
    uint8_t* s_inring;
    unsigned long long* pool_top;
    SchedDev s;
    unsigned int* status;
};

// ------------------------------------------------------------ per warp
struct Tx {
    const TxDev& d;
    TxConn* C;
    const uint32_t conn;
    const int lane;
    WarpRng r;
    double* rtt_s;  // PathScoreboard (lb.hpp:15-36), shared-memory copy
    double* ecn_s;
    int64_t* inflight;  // SubConn::inflight per path
    int64_t* deficit;   // SubConn::deficit
    uint32_t* txq_n;    // live tx-queue entries per path
    uint32_t* rtxq_n;   // live retransmission-queue entries per path
    uint16_t* ring;
    uint8_t* in_ring;
    int n;  // paths of this connection
    cn_tx_rec* log;
    uint32_t log_n;
    // RttEstimator, CC, timer, ring and counters (warp-uniform registers)
    int64_t srtt, rttvar, armed_at, timer_at, committed_unsent, total_inflight, last_decrease;
    double w;
    int has_sample, backoff, timer_armed, ring_len;
    uint64_t ring_pos;
    uint32_t ring_idx;       // ring_pos % ring_len
    uint32_t n_txq, n_rtxq;  // live entries over all tx / retransmission queues
    uint32_t q_seq, pump_pending;
    int64_t pump_at;  // schedule_pump (:219-230): one deferred pump per engine
    uint32_t sched_seq, timer_seq, pump_seq;  // (time, seq) order of run-scheduled events
    uint32_t n_stale;                         // register copy of C->stale_n
    uint32_t n_retry;                         // register copy of C->retry_n
    int64_t credit, unchunked, rtxq_bytes;    // receiver-driven state
    uint64_t chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_completed;
    uint32_t live[4];  // live message slots, iterated in slot order

    __device__ int64_t cur_rto() const {  // cc.hpp:27-33 via transport.cpp:1078-1081
        int64_t x = srtt + 4 * rttvar;
        if (x < d.rto_min) return d.rto_min;
        if (x > d.rto_max) return d.rto_max;
        return x;
    }
    __device__ void est_sample(int64_t rtt) {  // RttEstimator::sample (cc.hpp:17-28)
        if (!has_sample) {
            srtt = rtt;
            rttvar = rtt / 2;
            has_sample = 1;
            return;
        }
        int64_t err = srtt > rtt ? srtt - rtt : rtt - srtt;
        rttvar = (3 * rttvar + err) / 4;
        srtt = (7 * srtt + rtt) / 8;
    }
    // CongestionControl::cwnd_bytes: OpenLoop (cc.cpp:21-22), Swift (:146-148)
    __device__ int64_t cwnd_bytes() const {
        if (d.cc_algo == 0) return d.cap_bytes > 0 ? d.cap_bytes : LLONG_MAX / 4;
        return llround(__dmul_rn(w, static_cast<double>(d.mss)));
    }
    __device__ void cc_on_ack(int64_t now, int64_t acked, int64_t rtt) {  // cc.cpp:23-25, :117-131
        if (rtt > 0) est_sample(rtt);
        if (d.cc_algo == 0) return;
        if (rtt <= d.swift_target) {
            if (acked > 0) {
                double a = __ddiv_rn(static_cast<double>(acked), static_cast<double>(d.mss));
                double nw = __dadd_rn(w, __ddiv_rn(__dmul_rn(kSwiftAi, a), w));
                w = d.cap_pkts < nw ? d.cap_pkts : nw;
            }
            return;
        }
        if (now - last_decrease < srtt) return;
        double q = __ddiv_rn(__dmul_rn(kSwiftMdScale, static_cast<double>(rtt - d.swift_target)),
                             static_cast<double>(rtt));
        double f = __dsub_rn(1.0, q);
        if (f < kSwiftMaxMd) f = kSwiftMaxMd;
        double nw = __dmul_rn(w, f);
        w = nw < kMinCwndPkts ? kMinCwndPkts : nw;
        last_decrease = now;
    }
    __device__ void cc_on_loss(int64_t now) {  // cc.cpp:133-138
        if (d.cc_algo == 0) return;
        if (has_sample && now - last_decrease < srtt) return;
        double nw = __dmul_rn(w, kSwiftMaxMd);
        w = nw < kMinCwndPkts ? kMinCwndPkts : nw;
        last_decrease = now;
    }
    __device__ void cc_on_rto(int64_t now) {  // cc.cpp:140-144
        if (d.cc_algo == 0) return;
        w = kMinCwndPkts;
        last_decrease = now;
    }
    // can_send (:312-325), global scope: the connection's total inflight
    __device__ bool can_send() const {  // + the credit gate of receiver-driven mode (:314)
        return total_inflight < cwnd_bytes() && (!d.rd || credit > 0);
    }
    __device__ void add_inflight(int p, int64_t delta) {  // clamped at 0 (:520-521, :813-814)
        int64_t v = inflight[p] + delta;
        if (v < 0) v = 0;
        total_inflight += v - inflight[p];
        __syncwarp();
        if (lane == 0) inflight[p] = v;
        __syncwarp();
    }
    __device__ void ring_insert(int p) {  // :296-300, :537-540
        if (in_ring[p]) return;
        __syncwarp();
        if (lane == 0) {
            in_ring[p] = 1;
            ring[ring_len] = static_cast<uint16_t>(p);
        }
        __syncwarp();
        ++ring_len;
        ring_idx = static_cast<uint32_t>(ring_pos % static_cast<uint64_t>(ring_len));
    }
    __device__ void arm_rto(int64_t now) {  // transport.cpp:1083-1092
        if (timer_armed) return;
        timer_armed = 1;
        armed_at = now;
        timer_at = now + cur_rto() * backoff;
        timer_seq = ++sched_seq;
    }
    // maybe_send_rts (:1026-1053): ask the receiver's pacer for credit once
    // credit is spent with bytes still pending; retried every rto_min until
    // acknowledged (every retry event pending at once, as the reference
    // schedules them)
    __device__ void maybe_send_rts(int64_t now) {
        if (!d.rd || C->rts_outstanding) return;
        const int64_t pending = unchunked + committed_unsent + rtxq_bytes;  // pending_bytes (:1005-1024)
        if (pending <= 0 || credit > 0) return;
        const bool has_rtx = n_rtxq + n_stale > 0;  // raw queue emptiness, stale entries included
        __syncwarp();
        if (lane == 0) {
            C->rts_outstanding = 1;
            C->rts_acked = 0;
            if (C->retry_n < kRetryMax) {
                const uint32_t k = (C->retry_head + C->retry_n) % kRetryMax;
                C->retry_t[k] = now + d.rto_min;
                C->retry_seq[k] = sched_seq + 1;
                C->retry_n += 1;
            } else {
                atomicOr(d.status, 8u);
            }
        }
        __syncwarp();
        ++sched_seq;
        if (n_retry < kRetryMax) ++n_retry;
        record(now, 0, 0xFFFFFFFFu, -1, has_rtx ? 1 : 0, static_cast<uint64_t>(pending));  // the RTS
    }
    // on_select_path / on_tx_rtx_chunk of the connection's policy for chunk
    // ci of message m (view_of, transport.cpp:496-512); prev_path >= 0 for a
    // retransmission
    __device__ int select(int prev_path, const TxMsg& m, uint32_t mid, uint32_t ci, int attempts) {
        if (d.pol == CN_POLICY_DEFAULT) {  // DefaultPolicy (policy.hpp:80-91)
            int p = select_seq(r, d.policy, n, d.policy == 2 ? ecn_s : rtt_s, lane);
            if (prev_path >= 0 && d.avoid_prev && n > 1 && p == prev_path) p = (p + 1) % n;
            return p;
        }
        cn_chunk_view v;
        v.src = C->src;
        v.dst = C->dst;
        v.msg_id = mid;
        v.csn = ci & 0xFF;
        v.msg_seq = m.seq;
        v.msg_len = m.len;
        v.offset = static_cast<uint64_t>(ci) * d.cb;
        v.len = chunk_len(m, ci);
        v.last = v.offset + v.len == m.len;
        v.attempts = attempts;
        v.prev_path = prev_path;
        // a fresh chunk is counted as chunked before the hook runs (:271-283)
        v.remaining = m.len - (prev_path >= 0 ? m.chunked : m.chunked + v.len);
        switch (d.pol) {
            case CN_POLICY_ROUND_ROBIN: return pick<cn_policy::RoundRobinPolicy>(v);
            case CN_POLICY_SINGLE_PATH: return pick<cn_policy::SinglePathPolicy>(v);
            case CN_POLICY_TEST_OUT_OF_RANGE: return pick<cn_policy::OutOfRangePolicy>(v);
#ifdef CN_TX_USER_POLICY_HEADER
            case CN_POLICY_USER: return pick<CnUserPolicy>(v);
#endif
            default: return pick<cn_policy::OutOfRangePolicy>(v);
        }
    }
    struct PolicyRng {  // the connection's RngStream, warp-collective draws
        WarpRng& r;
        int lane;
        __device__ uint64_t next_below(uint64_t k) { return next_below_warp(r, k, lane); }
    };
    template <class P>
    __device__ int pick(const cn_chunk_view& v) {
        cn_path_board b;
        b.rtt_ewma = rtt_s;
        b.ecn_ewma = ecn_s;
        b.n_paths = n;
        PolicyRng g{r, lane};
        uint64_t st[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) st[k] = C->pol_state[k];
        int p = v.prev_path >= 0 ? P::rtx_path(v, b, g, st) : -1;
        if (p == -1) p = P::select_path(v, b, g, st);
        const bool bad = p < 0 || p >= n || P::pacing(v) != 0;
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) C->pol_state[k] = st[k];
            if (bad) atomicOr(d.status, 64u);  // the reference's logic_error (:283-290, :528-531)
        }
        __syncwarp();
        return bad ? 0 : p;
    }
    __device__ void record(int64_t t, uint32_t mid, uint32_t ci, int32_t path, int rtx, uint64_t seq) {
        if (lane == 0 && log_n < d.log_cap) {
            cn_tx_rec x;
            x.t = t;
            x.msg_id = mid;
            x.chunk = ci;
            x.path = path;
            x.is_rtx = rtx;
            x.msg_seq = seq;
            log[log_n] = x;
        }
        ++log_n;
    }
    __device__ uint32_t chunk_len(const TxMsg& m, uint32_t ci) const {
        uint64_t off = static_cast<uint64_t>(ci) * d.cb;
        return m.len - off < d.cb ? static_cast<uint32_t>(m.len - off) : d.cb;
    }
    // send_chunk (transport.cpp:433-494) on the path the chunk is queued on
    __device__ void send_chunk(int64_t now, uint32_t mid, const TxMsg& m, uint32_t ci, bool rtx,
                               uint64_t from_psn = 0) {
        const uint64_t e = m.chunk_base + ci;
        const int64_t dl = now + cur_rto() * backoff;
        const int32_t path = d.c_path[e];
        const int32_t att = d.c_att[e] + 1;
        uint32_t start = 0;  // first packet sent (a go-back-N resend may start mid-chunk, :438-447)
        if (d.ordered) {
            if (att == 1) {
                const uint32_t npk = (chunk_len(m, ci) + d.max_pl - 1) / d.max_pl;
                __syncwarp();
                if (lane == 0) {
                    d.c_psn[e] = static_cast<int64_t>(C->next_psn);
                    C->next_psn += npk;
                    if (C->so_n < d.so_cap)
                        d.so_ref[static_cast<uint64_t>(conn) * d.so_cap + C->so_n] = (mid << 25) | ci;
                    else
                        atomicOr(d.status, 32u);
                    C->so_n += 1;
                }
                __syncwarp();
            } else {
                const uint64_t base = static_cast<uint64_t>(d.c_psn[e]);
                if (from_psn > base) start = static_cast<uint32_t>(from_psn - base);
            }
        }
        __syncwarp();
        if (lane == 0) {
            d.c_att[e] = att;
            d.c_fl[e] = TF_SENT | (d.c_fl[e] & TF_ACKED);
            d.c_dup[e] = 0;
            d.c_txt[e] = now;
            d.c_dead[e] = dl;
            d.c_q[e] = 0;
        }
        __syncwarp();
        add_inflight(path, chunk_len(m, ci));
        if (d.rd) credit -= chunk_len(m, ci) - start * d.max_pl;  // the bytes actually sent (:486)
        if (rtx) ++chunk_rtx;
        else ++chunks_sent;
        record(now, mid, ci, path | static_cast<int32_t>(start << 16), rtx || att > 1, m.seq);
        __syncwarp();
        arm_rto(now);
    }
    // queue_rtx (transport.cpp:516-542); caller checked sent && !acked && !rtx_pending
    __device__ void queue_rtx(int64_t now, const TxMsg& m, uint32_t mid, uint32_t ci) {
        const uint64_t e = m.chunk_base + ci;
        const int prev = d.c_path[e];  // attempts > 0: prev_path = ch.path (view_of, :509)
        add_inflight(prev, -static_cast<int64_t>(chunk_len(m, ci)));
        cc_on_loss(now);
        const int p = select(prev, m, mid, ci, d.c_att[e]);
        ++q_seq;
        __syncwarp();
        if (lane == 0) {
            d.c_fl[e] |= TF_RTXP;
            d.c_dup[e] = 0;
            d.c_path[e] = p;
            d.c_q[e] = kQRtx | q_seq;
            rtxq_n[p] += 1;
        }
        ++n_rtxq;
        rtxq_bytes += chunk_len(m, ci);
        __syncwarp();
        ring_insert(p);
        if (!pump_pending) {  // schedule_pump (:541): runs after the events queued at `now`
            pump_pending = 1;
            pump_at = now;
            pump_seq = ++sched_seq;
        }
    }
};

__device__ __forceinline__ TxMsg load_msg(const TxConn* C, uint32_t mid) { return C->msgs[mid]; }
__device__ __forceinline__ void store_msg(TxConn* C, uint32_t mid, const TxMsg& m, int lane) {
    __syncwarp();
    if (lane == 0) C->msgs[mid] = m;
    __syncwarp();
}
__device__ __forceinline__ void set_u32(uint32_t* p, uint32_t v, int lane) {
    __syncwarp();
    if (lane == 0) *p = v;
    __syncwarp();
}

// Front of path p's tx (rtx = false) or retransmission queue.
__device__ bool queue_front(const Tx& x, int p, bool rtx, uint32_t* out_mid, uint32_t* out_ci) {
    uint32_t best = 0xFFFFFFFFu, bmid = 0, bci = 0;
    for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            const TxMsg m = load_msg(x.C, mid);
            for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
                const uint32_t ci = w0 + x.lane;
                uint32_t key = 0xFFFFFFFFu;
                if (ci < m.nchunks) {
                    const uint64_t e = m.chunk_base + ci;
                    const uint32_t qv = x.d.c_q[e];
                    if (qv && ((qv & kQRtx) != 0) == rtx && x.d.c_path[e] == p) key = qv & ~kQRtx;
                }
                const uint32_t mn = __reduce_min_sync(0xffffffffu, key);
                if (mn < best) {
                    best = mn;
                    bmid = mid;
                    bci = w0 + __ffs(__ballot_sync(0xffffffffu, key == mn)) - 1;
                }
            }
        }
    *out_mid = bmid;
    *out_ci = bci;
    return best != 0xFFFFFFFFu;
}

// `visits` DRR visits that cannot send (window shut or nothing queued):
// each visits a distinct path of the ring once, so they are independent --
// a tx-queued path tops its deficit up to one quantum, an idle one resets it
// (:385-391) -- and run lane-parallel.
__device__ void drr_idle(Tx& x, uint32_t visits) {
    const uint32_t nr = static_cast<uint32_t>(x.ring_len);
    const int64_t q = x.d.quantum;
    __syncwarp();
    for (uint32_t j = x.lane; j < visits; j += 32) {
        uint32_t k = x.ring_idx + j;
        k = k >= nr ? k - nr : k;
        const int p = x.ring[k];
        const int64_t def = x.deficit[p] + q;
        x.deficit[p] = x.txq_n[p] ? (def > q ? q : def) : 0;
    }
    __syncwarp();
    x.ring_pos += visits;
    x.ring_idx = static_cast<uint32_t>((x.ring_idx + visits) % nr);
}

// gbn_rewind (transport.cpp:969-999): re-queue every unacked chunk whose
// packets reach the receiver's expected sequence, in first-send order;
// chunks wholly below it stay (or come back) in flight.
__device__ void gbn_rewind(Tx& x, int64_t now, uint64_t expected) {
    TxConn* C = x.C;
    if (expected == C->last_rewind_psn) return;  // duplicate gap report
    x.cc_on_loss(now);
    __syncwarp();
    if (x.lane == 0) {
        C->last_rewind_psn = expected;
        C->gq_head = 0;
        C->gq_n = 0;
    }
    __syncwarp();
    const uint64_t so = static_cast<uint64_t>(x.conn) * x.d.so_cap;
    const uint32_t n = C->so_n < x.d.so_cap ? C->so_n : x.d.so_cap;
    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
        const uint32_t k = k0 + x.lane;
        int act = 0;  // 1: back in flight, 2: re-queue
        uint32_t ref = 0, len = 0;
        uint64_t from = 0;
        uint64_t e = 0;
        if (k < n) {
            ref = x.d.so_ref[so + k];
            const uint32_t mid = ref >> 25, ci = ref & ((1u << 25) - 1);
            const TxMsg m = load_msg(C, mid);  // the slot's current message (:978-980)
            if (m.live && ci < m.nchunks) {
                e = m.chunk_base + ci;
                const uint32_t fl = x.d.c_fl[e];
                if ((fl & TF_SENT) && !(fl & TF_ACKED)) {
                    len = x.chunk_len(m, ci);
                    const uint64_t base = static_cast<uint64_t>(x.d.c_psn[e]);
                    const uint64_t end = base + (len + x.d.max_pl - 1) / x.d.max_pl;
                    if (end <= expected) {
                        act = (fl & TF_RTXP) ? 1 : 0;
                    } else {
                        act = (fl & TF_RTXP) ? 3 : 2;  // 3: already pending, just re-queued
                        from = base > expected ? base : expected;
                    }
                }
            }
        }
        for (unsigned b = __ballot_sync(0xffffffffu, act != 0); b; b &= b - 1) {  // in order
            const int j = __ffs(b) - 1;
            const int aj = __shfl_sync(0xffffffffu, act, j);
            const uint32_t lj = __shfl_sync(0xffffffffu, len, j);
            const uint64_t ej = __shfl_sync(0xffffffffu, e, j);
            if (aj == 1) {  // delivered but unacked: in flight again
                __syncwarp();
                if (x.lane == 0) x.d.c_fl[ej] &= ~TF_RTXP;
                __syncwarp();
                x.add_inflight(0, lj);
            } else {
                if (aj == 2) {
                    __syncwarp();
                    if (x.lane == 0) x.d.c_fl[ej] |= TF_RTXP;
                    __syncwarp();
                    x.add_inflight(0, -static_cast<int64_t>(lj));
                }
                const uint32_t rj = __shfl_sync(0xffffffffu, ref, j);
                const uint64_t fj = __shfl_sync(0xffffffffu, from, j);
                __syncwarp();
                if (x.lane == 0) {
                    x.d.c_dup[ej] = 0;
                    const uint32_t q = (C->gq_head + C->gq_n) % x.d.so_cap;
                    x.d.gq_ref[so + q] = rj;
                    x.d.gq_from[so + q] = fj;
                    C->gq_n += 1;
                }
                __syncwarp();
            }
        }
    }
    if (!x.pump_pending) {  // schedule_pump (:998)
        x.pump_pending = 1;
        x.pump_at = now;
        x.pump_seq = ++x.sched_seq;
    }
}

// Index of the stale retransmission-queue entry of path p with the smallest
// queue seq, or -1.
__device__ int stale_front(const Tx& x, int p) {
    const TxConn* C = x.C;
    uint32_t best = 0xFFFFFFFFu;
    int bi = -1;
    for (uint32_t k0 = 0; k0 < C->stale_n; k0 += 32) {
        const uint32_t k = k0 + x.lane;
        const uint32_t key = (k < C->stale_n && C->stale_path[k] == p) ? C->stale_seq[k] : 0xFFFFFFFFu;
        const uint32_t mn = __reduce_min_sync(0xffffffffu, key);
        if (mn < best) {
            best = mn;
            bi = static_cast<int>(k0 + __ffs(__ballot_sync(0xffffffffu, key == mn)) - 1);
        }
    }
    return bi;
}

// egress (transport.cpp:329-431): retransmission queues in ring order, then
// deficit round robin over the ring, every send gated by can_send.
__device__ uint32_t egress(Tx& x, int64_t now) {
    uint32_t sent = 0;
    for (int k = 0; (x.n_rtxq || x.n_stale || (x.d.ordered && x.C->gq_n)) && k < x.ring_len; ++k) {  // :333-369
        const int p = x.ring[k];
        while (x.d.ordered && p == 0 && x.C->gq_n && x.can_send()) {  // gbn_rtxq (:336-352)
            TxConn* C = x.C;
            const uint64_t so = static_cast<uint64_t>(x.conn) * x.d.so_cap;
            const uint32_t ref = x.d.gq_ref[so + C->gq_head];
            const uint64_t from = x.d.gq_from[so + C->gq_head];
            __syncwarp();
            if (x.lane == 0) {
                C->gq_head = (C->gq_head + 1) % x.d.so_cap;
                C->gq_n -= 1;
            }
            __syncwarp();
            const uint32_t mid = ref >> 25, ci = ref & ((1u << 25) - 1);
            const TxMsg m = load_msg(C, mid);
            if (!m.live || ci >= m.nchunks) continue;
            const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
            if ((fl & TF_ACKED) || !(fl & TF_RTXP)) continue;
            x.send_chunk(now, mid, m, ci, true, from);
            ++sent;
        }
        while ((x.rtxq_n[p] > 0 || (x.n_stale && stale_front(x, p) >= 0)) && x.can_send()) {
            uint32_t mid = 0, ci = 0;
            const bool live = x.rtxq_n[p] > 0 && queue_front(x, p, true, &mid, &ci);
            const uint32_t lseq = live ? (x.d.c_q[load_msg(x.C, mid).chunk_base + ci] & ~kQRtx) : 0xFFFFFFFFu;
            const int si = x.n_stale ? stale_front(x, p) : -1;
            if (si >= 0 && x.C->stale_seq[si] < lseq) {  // a stale entry at the front: popped, nothing sent
                __syncwarp();
                if (x.lane == 0) {
                    TxConn* C = x.C;
                    const uint32_t last = C->stale_n - 1;
                    C->stale_seq[si] = C->stale_seq[last];
                    C->stale_path[si] = C->stale_path[last];
                    C->stale_n = last;
                }
                __syncwarp();
                --x.n_stale;
                continue;
            }
            if (!live) break;
            const TxMsg m = load_msg(x.C, mid);
            set_u32(&x.rtxq_n[p], x.rtxq_n[p] - 1, x.lane);
            --x.n_rtxq;
            x.rtxq_bytes -= x.chunk_len(m, ci);
            x.send_chunk(now, mid, m, ci, true);
            ++sent;
        }
    }
    const uint32_t nr = static_cast<uint32_t>(x.ring_len);
    if (nr == 0) {
        if (x.d.rd) x.maybe_send_rts(now);  // :372-377
        return sent;
    }
    uint32_t idle = 0;
    while (idle < nr) {  // :378-424
        if (x.n_txq == 0 || !x.can_send()) {  // the remaining visits cannot send
            drr_idle(x, nr - idle);
            break;
        }
        const int p = x.ring[x.ring_idx];
        ++x.ring_pos;
        if (++x.ring_idx == nr) x.ring_idx = 0;
        if (x.txq_n[p] == 0) {
            __syncwarp();
            if (x.lane == 0) x.deficit[p] = 0;
            __syncwarp();
            ++idle;
            continue;
        }
        int64_t def = x.deficit[p] + static_cast<int64_t>(x.d.quantum);
        if (def > static_cast<int64_t>(x.d.quantum)) def = x.d.quantum;
        bool sent_any = false;
        while (x.txq_n[p] > 0 && def > 0 && x.can_send()) {
            uint32_t mid, ci;
            if (!queue_front(x, p, false, &mid, &ci)) break;
            const TxMsg m = load_msg(x.C, mid);
            const uint32_t len = x.chunk_len(m, ci);
            set_u32(&x.txq_n[p], x.txq_n[p] - 1, x.lane);
            --x.n_txq;
            x.committed_unsent -= len;
            def -= len;
            x.send_chunk(now, mid, m, ci, false);
            sent_any = true;
            ++sent;
        }
        if (x.txq_n[p] == 0) def = 0;
        __syncwarp();
        if (x.lane == 0) x.deficit[p] = def;
        __syncwarp();
        idle = sent_any ? 0 : idle + 1;
    }
    if (x.d.rd) x.maybe_send_rts(now);  // :427-430
    return sent;
}

// commit_chunks (transport.cpp:244-310): one chunk per message per turn of
// the factory rotation, window-stalled at 128 unacked chunks, bounded by
// commit_ahead bytes; each chunk is bound to a path and queued on it.
__device__ void commit_chunks(Tx& x) {
    TxConn* C = x.C;
    int32_t head = C->fq_head, count = C->fq_count;
    uint32_t stalled = 0;
    while (count > 0 && stalled < static_cast<uint32_t>(count) && x.committed_unsent < x.d.commit_ahead) {
        const uint32_t mid = C->fq[head];
        head = (head + 1) & 127;
        --count;
        TxMsg m = load_msg(C, mid);
        if (!m.live || m.chunked >= m.len) {
            m.in_factory = 0;
            store_msg(C, mid, m, x.lane);
            stalled = 0;
            continue;
        }
        if (m.nchunks - m.base >= static_cast<uint32_t>(kTxWindow)) {
            __syncwarp();
            if (x.lane == 0) C->fq[(head + count) & 127] = static_cast<uint8_t>(mid);
            __syncwarp();
            ++count;
            ++stalled;
            continue;
        }
        const uint64_t rem = m.len - m.chunked;
        const uint32_t sz = rem < x.d.cb ? static_cast<uint32_t>(rem) : x.d.cb;
        const uint32_t ci = m.nchunks;
        const int p = x.select(-1, m, mid, ci, 0);  // on_select_path (:281-287)
        ++x.q_seq;
        __syncwarp();
        if (x.lane == 0) {
            const uint64_t e = m.chunk_base + ci;
            x.d.c_path[e] = p;
            x.d.c_fl[e] = 0;
            x.d.c_att[e] = 0;
            x.d.c_dup[e] = 0;
            x.d.c_q[e] = x.q_seq;
            x.txq_n[p] += 1;
        }
        ++x.n_txq;
        __syncwarp();
        x.ring_insert(p);
        m.nchunks = ci + 1;
        m.chunked += sz;
        x.committed_unsent += sz;
        x.unchunked -= sz;
        if (m.chunked < m.len) {
            __syncwarp();
            if (x.lane == 0) C->fq[(head + count) & 127] = static_cast<uint8_t>(mid);
            __syncwarp();
            ++count;
        } else {
            m.in_factory = 0;
        }
        store_msg(C, mid, m, x.lane);
        stalled = 0;
    }
    __syncwarp();
    if (x.lane == 0) {
        C->fq_head = head;
        C->fq_count = count;
    }
    __syncwarp();
}

// Inlined into every caller.  Resuming a Swift replay across cn_tx_run
// calls faults with run_deferred inlined (-DCN_TX_DEFERRED_INLINE) and not
// with this layout or the pump out of line (-DCN_TX_PUMP_NOINLINE); the
// cause is not pinned down.  test_tx_gpu.py::
// test_tx_engine_resumes_across_runs, tests/tx_resume_sweep_tool.py and the
// endpoint introspection tests guard the layout that passes.
#ifdef CN_TX_PUMP_NOINLINE  // diagnostic build of the faulting layout
__device__ __noinline__ void pump(Tx& x, int64_t now) {
#else
__device__ __forceinline__ void pump(Tx& x, int64_t now) {  // transport.cpp:232-240
#endif
    for (;;) {
        commit_chunks(x);
        if (egress(x, now) == 0) break;
    }
}

// try_advance_base (:825-829): first unacked chunk at or after base
__device__ uint32_t advance_base(const Tx& x, const TxMsg& m) {
    uint32_t b = m.base;
    while (b < m.nchunks) {
        const uint32_t ci = b + x.lane;
        const bool acked = ci < m.nchunks ? (x.d.c_fl[m.chunk_base + ci] & TF_ACKED) != 0 : false;
        const unsigned un = __ballot_sync(0xffffffffu, !acked);
        if (un) return b + __ffs(un) - 1;
        b += 32;
    }
    return m.nchunks;
}

// msg_finished (:831-847)
__device__ void msg_finished(Tx& x, uint32_t mid) {
    TxConn* C = x.C;
    TxMsg m;
    memset(&m, 0, sizeof m);
    store_msg(C, mid, m, x.lane);
    x.live[mid >> 5] &= ~(1u << (mid & 31));
    if (x.lane == 0) {
        C->free_ids[C->n_free] = static_cast<uint8_t>(mid);
        C->n_free += 1;
        C->live_msgs -= 1;
    }
    __syncwarp();
    ++x.msgs_completed;
}

// release_chunk (:807-823) of a chunk the caller found sent && !acked.  A
// chunk awaiting retransmission leaves its queue (the reference's entry
// turns stale and is popped without effect).
__device__ void release(Tx& x, int64_t now, const TxMsg& m, uint32_t ci, int64_t rtt, bool ecn) {
    const uint64_t e = m.chunk_base + ci;
    const uint32_t fl = x.d.c_fl[e];
    const int path = x.d.c_path[e];
    const uint32_t len = x.chunk_len(m, ci);
    const uint32_t rq = x.rtxq_n[path];
    const uint32_t qv = x.d.c_q[e];
    __syncwarp();
    if (x.lane == 0) {
        x.d.c_fl[e] = (fl | TF_ACKED) & ~TF_RTXP;
        if (fl & TF_RTXP) {
            x.rtxq_n[path] = rq - 1;
            x.d.c_q[e] = 0;
            // its queue entry stays behind, stale, until egress pops it (:347-351)
            TxConn* C = x.C;
            if (C->stale_n < kStaleMax) {
                C->stale_seq[C->stale_n] = qv & ~kQRtx;
                C->stale_path[C->stale_n] = static_cast<uint16_t>(path);
                C->stale_n += 1;
            } else {
                atomicOr(x.d.status, 16u);
            }
        }
    }
    __syncwarp();
    if (fl & TF_RTXP) {
        --x.n_rtxq;
        x.rtxq_bytes -= len;
        if (x.n_stale < kStaleMax) ++x.n_stale;
    } else {
        x.add_inflight(path, -static_cast<int64_t>(len));
    }
    x.cc_on_ack(now, len, rtt);
    if (rtt > 0) {  // board.record_rtt / record_ecn (:819-822)
        __syncwarp();
        if (x.lane == 0) {
            x.rtt_s[path] += (static_cast<double>(rtt) - x.rtt_s[path]) / 8.0;
            x.ecn_s[path] += ((ecn ? 1.0 : 0.0) - x.ecn_s[path]) / 8.0;
        }
        __syncwarp();
    }
}

// Releases, in ascending order, every sent && !acked chunk of [lo, hi)
// that `pick` selects (CC sees the acks in the reference's order).
template <class Pick>
__device__ uint32_t release_range(Tx& x, int64_t now, TxMsg& m, uint32_t lo, uint32_t hi, Pick pick) {
    uint32_t n_rel = 0;
    for (uint32_t w0 = lo; w0 < hi; w0 += 32) {
        const uint32_t ci = w0 + x.lane;
        bool want = false;
        if (ci < hi && pick(ci)) {
            const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
            want = (fl & TF_SENT) && !(fl & TF_ACKED);
        }
        for (unsigned b = __ballot_sync(0xffffffffu, want); b; b &= b - 1) {
            release(x, now, m, w0 + __ffs(b) - 1, 0, false);
            ++n_rel;
        }
    }
    m.acked += n_rel;
    return n_rel;
}

// handle_ack (:849-942)
__device__ void handle_ack(Tx& x, int64_t now, const cn_ack_rec& a) {
    TxConn* C = x.C;
    const uint32_t mid = (a.hdr >> 17) & 0x7F;
    TxMsg m = load_msg(C, mid);
    if (!m.live || m.seq != a.msg_seq) return;  // :855 (no pump)
    const uint8_t base_csn = static_cast<uint8_t>(m.base & 0xFF);
    const uint32_t nch = m.nchunks;
    uint32_t newly = 0;
    int64_t cause = -1;
    {
        const uint8_t rel = static_cast<uint8_t>(((a.hdr >> 9) & 0xFF) - base_csn);
        if (rel < kTxWindow && m.base + rel < nch) cause = m.base + rel;
    }
    if (cause >= 0) {  // cause chunk: the only trustworthy RTT echo (:869-887)
        const uint64_t e = m.chunk_base + cause;
        const uint32_t fl = x.d.c_fl[e];
        if ((fl & TF_SENT) && !(fl & TF_ACKED)) {
            int64_t rtt = 0;
            if (x.d.c_att[e] == 1 && a.echo_tx_time == x.d.c_txt[e] && now > a.echo_tx_time)
                rtt = now - a.echo_tx_time;
            release(x, now, m, static_cast<uint32_t>(cause), rtt, (a.flags & CN_ACK_ECN_ECHO) != 0);
            m.acked += 1;
            ++newly;
        }
    }
    // cumulative bound (:890-897)
    uint32_t rcum = m.base;
    if (a.flags & CN_ACK_CUM_VALID) {
        const uint8_t rel1 = static_cast<uint8_t>(static_cast<uint8_t>(a.cum_csn + 1) - base_csn);
        if (rel1 <= kTxWindow) rcum = m.base + rel1;
    } else {
        rcum = 0;
    }
    const uint32_t cend = rcum < nch ? rcum : nch;
    newly += release_range(x, now, m, m.base, cend, [](uint32_t) { return true; });  // :898-904
    {  // selective bitmap relative to rcum (:905-914)
        const uint32_t send_ = rcum + 128 < nch ? rcum + 128 : nch;
        const uint64_t s0 = a.sack[0], s1 = a.sack[1];
        const uint32_t rc = rcum;
        newly += release_range(x, now, m, rcum < send_ ? rcum : send_, send_, [=](uint32_t ci) {
            const uint32_t j = ci - rc;
            return ((j < 64 ? s0 >> j : s1 >> (j - 64)) & 1ull) != 0;
        });
    }
    // duplicate hints -> fast retransmit, ascending chunk order (:918-929; selective only)
    if (cause >= 0 && !x.d.ordered) {
        for (uint32_t w0 = m.base; w0 < static_cast<uint32_t>(cause); w0 += 32) {
            const uint32_t ci = w0 + x.lane;
            bool trig = false;
            if (ci < static_cast<uint32_t>(cause)) {
                const uint64_t e = m.chunk_base + ci;
                const uint32_t fl = x.d.c_fl[e];
                if ((fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP))) {
                    const int32_t dup = x.d.c_dup[e] + 1;
                    x.d.c_dup[e] = dup;
                    trig = dup >= static_cast<int32_t>(x.d.dupack);
                }
            }
            __syncwarp();
            for (unsigned b = __ballot_sync(0xffffffffu, trig); b; b &= b - 1) {
                ++x.fast_rtx;
                x.queue_rtx(now, m, mid, w0 + __ffs(b) - 1);
            }
        }
    }
    m.base = advance_base(x, m);  // :931
    const bool done = m.chunked >= m.len && nch > 0 && m.acked == nch && !m.in_factory;
    store_msg(C, mid, m, x.lane);
    if (done) msg_finished(x, mid);  // :932-934
    if (newly > 0) {                 // :936-940
        x.backoff = 1;
        x.timer_armed = 0;
        x.arm_rto(now);
    }
    pump(x, now);  // :941
}

// handle_nack (:944-965), selective mode: a trimmed header's NACK names a
// chunk that never arrived -- retransmit it now.
__device__ void handle_nack(Tx& x, int64_t now, const cn_ack_rec& a) {
    if (x.d.ordered) {  // :950-954
        gbn_rewind(x, now, a.sack[0]);
        pump(x, now);
        return;
    }
    const uint32_t mid = (a.hdr >> 17) & 0x7F;
    const TxMsg m = load_msg(x.C, mid);
    if (!m.live || m.seq != a.msg_seq) return;
    const uint8_t rel = static_cast<uint8_t>(a.cum_csn - static_cast<uint8_t>(m.base & 0xFF));
    if (rel >= kTxWindow || m.base + rel >= m.nchunks) return;
    const uint32_t ci = m.base + rel;
    const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
    if ((fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP))) x.queue_rtx(now, m, mid, ci);
    pump(x, now);
}

// rto_fire (:1094-1169), the live timer at x.timer_at
__device__ void rto_fire(Tx& x) {
    TxConn* C = x.C;
    const int64_t now = x.timer_at;
    x.timer_armed = 0;
    // scan: oldest deadline and the number of expired chunks
    int64_t best = 0;
    bool have = false;
    uint32_t n_exp = 0;
    for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            const TxMsg m = load_msg(C, mid);
            for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
                const uint32_t ci = w0 + x.lane;
                bool elig = false;
                int64_t dl = 0;
                if (ci < m.nchunks) {
                    const uint64_t e = m.chunk_base + ci;
                    const uint32_t fl = x.d.c_fl[e];
                    elig = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP));
                    dl = x.d.c_dead[e];
                }
                long long mn = elig ? dl : LLONG_MAX;
                for (int o = 16; o > 0; o >>= 1) {
                    const long long t = __shfl_xor_sync(0xffffffffu, mn, o);
                    mn = t < mn ? t : mn;
                }
                if (__ballot_sync(0xffffffffu, elig) && (!have || mn < best)) {
                    best = mn;
                    have = true;
                }
                n_exp += __popc(__ballot_sync(0xffffffffu, elig && dl <= now));
            }
        }
    if (!have) return;  // :1131 nothing outstanding
    if (n_exp == 0) {   // :1132-1140 re-arm for the earliest deadline
        x.timer_armed = 1;
        x.armed_at = now;
        x.timer_at = best;
        x.timer_seq = ++x.sched_seq;
        return;
    }
    ++x.rtos;
    x.backoff = x.backoff * 2 < kBackoffCap ? x.backoff * 2 : kBackoffCap;
    x.cc_on_rto(now);  // once per distinct CC -- global scope has one (:1154-1160)
    if (x.d.ordered) {  // :1144-1148: rewind from the oldest outstanding chunk's first packet
        uint64_t psn0 = 0;
        bool found = false;
        for (uint32_t q = 0; q < 4 && !found; ++q)
            for (uint32_t lb = x.live[q]; lb && !found; lb &= lb - 1) {
                const uint32_t mid = q * 32 + __ffs(lb) - 1;
                const TxMsg m = load_msg(C, mid);
                for (uint32_t w0 = m.base; w0 < m.nchunks && !found; w0 += 32) {
                    const uint32_t ci = w0 + x.lane;
                    bool hit = false;
                    if (ci < m.nchunks) {
                        const uint64_t e = m.chunk_base + ci;
                        const uint32_t fl = x.d.c_fl[e];
                        hit = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP)) && x.d.c_dead[e] == best;
                    }
                    const unsigned b = __ballot_sync(0xffffffffu, hit);
                    if (b) {
                        const uint32_t cj = w0 + __ffs(b) - 1;
                        psn0 = static_cast<uint64_t>(x.d.c_psn[m.chunk_base + cj]);
                        found = true;
                    }
                }
            }
        __syncwarp();
        if (x.lane == 0) C->last_rewind_psn = ~0ull;
        __syncwarp();
        gbn_rewind(x, now, psn0);
        if (x.d.rd) x.maybe_send_rts(now);
        x.arm_rto(now);
        pump(x, now);
        return;
    }
    for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            const TxMsg m = load_msg(C, mid);
            for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
                const uint32_t ci = w0 + x.lane;
                bool ex = false;
                if (ci < m.nchunks) {
                    const uint64_t e = m.chunk_base + ci;
                    const uint32_t fl = x.d.c_fl[e];
                    ex = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP)) && x.d.c_dead[e] <= now;
                }
                for (unsigned b = __ballot_sync(0xffffffffu, ex); b; b &= b - 1)
                    x.queue_rtx(now, m, mid, w0 + __ffs(b) - 1);
            }
        }
    if (x.d.rd) x.maybe_send_rts(now);  // :1166
    x.arm_rto(now);  // :1167
    pump(x, now);    // :1168
}

// send_message (:144-196) + dispatch (:198-218)
__device__ void submit(Tx& x, int64_t now, const cn_tx_submit& s) {
    TxConn* C = x.C;
    if (s.len == 0 || C->n_free == 0) {  // len 0 throws in the reference; flagged here
        __syncwarp();
        if (x.lane == 0) C->backpressured += 1;
        if (s.len == 0 && x.lane == 0) atomicOr(x.d.status, 1u);
        __syncwarp();
        return;
    }
    const uint32_t mid = C->free_ids[C->n_free - 1];
    const uint64_t seq = C->next_seq;
    __syncwarp();
    if (x.lane == 0) C->next_seq = seq + 1;
    __syncwarp();
    if (static_cast<uint32_t>(C->live_msgs) >= x.d.max_inflight) {
        __syncwarp();
        if (x.lane == 0) C->backpressured += 1;
        __syncwarp();
        return;
    }
    // the connection's share of the chunk pool is a ring: a message takes
    // nc contiguous entries (the ring's end is skipped when too short) and
    // frees them when it finishes (msg_finished, :831-847); the tail is the
    // oldest live message
    const uint64_t nc = (s.len + x.d.cb - 1) / x.d.cb;
    const uint64_t pc = x.d.conn_pool;
    const uint64_t h = C->p_head;
    uint64_t tl = h;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if ((x.live[k] >> x.lane) & 1u) {
            const uint64_t ps = C->p_start[k * 32 + x.lane];
            tl = ps < tl ? ps : tl;
        }
    for (int o = 16; o; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, tl, o);
        tl = y < tl ? y : tl;
    }
    const uint64_t pp = h % pc;
    const uint64_t start = pp + nc > pc ? h + (pc - pp) : h;
    if (nc > pc || start + nc - tl > pc) {
        if (x.lane == 0) atomicOr(x.d.status, 4u);
        return;
    }
    const uint64_t base = static_cast<uint64_t>(x.conn) * pc + start % pc;
    for (uint64_t k = x.lane; k < nc; k += 32) {  // a reused range starts unsent
        x.d.c_fl[base + k] = 0;
        x.d.c_q[base + k] = 0;
    }
    __syncwarp();
    if (x.lane == 0) {
        C->p_head = start + nc;
        C->p_start[mid] = start;
    }
    TxMsg m;
    memset(&m, 0, sizeof m);
    m.seq = seq;
    m.tag = s.tag;
    m.len = s.len;
    m.chunk_base = base;
    m.live = 1;
    m.in_factory = 1;
    store_msg(C, mid, m, x.lane);
    x.live[mid >> 5] |= 1u << (mid & 31);
    if (x.lane == 0) {
        C->n_free -= 1;
        C->live_msgs += 1;
        C->msgs_sent += 1;
        C->fq[(C->fq_head + C->fq_count) & 127] = static_cast<uint8_t>(mid);
        C->fq_count += 1;
    }
    __syncwarp();
    // dispatch's RTS check (:216) runs before the message is live, so its
    // bytes are not pending yet
    if (x.d.rd) x.maybe_send_rts(now);
    x.unchunked += s.len;
    pump(x, now);
}

// handle_credit (:1061-1074): bank the grant up to the cap, clear the
// outstanding RTS, pump, and ask again if needed
__device__ void handle_credit(Tx& x, int64_t now, uint64_t bytes) {
    const int64_t cap = x.d.credit_cap;
    if (x.credit < cap) {
        const int64_t v = x.credit + static_cast<int64_t>(bytes);
        x.credit = v < cap ? v : cap;
    }
    __syncwarp();
    if (x.lane == 0) x.C->rts_outstanding = 0;
    __syncwarp();
    pump(x, now);
    x.maybe_send_rts(now);
}

// an RTS retry event (:1046-1052)
__device__ void rts_retry(Tx& x, int64_t now) {
    TxConn* C = x.C;
    const bool again = C->rts_outstanding && !C->rts_acked;
    __syncwarp();
    if (x.lane == 0) {
        C->retry_head = (C->retry_head + 1) % kRetryMax;
        C->retry_n -= 1;
        if (again) C->rts_outstanding = 0;
    }
    __syncwarp();
    --x.n_retry;
    if (again) x.maybe_send_rts(now);
}

// Fires the events the run itself scheduled -- the RTO timer and the
// deferred pump -- that precede an input event at time t (inclusive = false)
// or the horizon t (inclusive = true), in the event queue's (time, seq)
// order: input events were all queued first, so they win ties; a timer due
// at the deferred pump's time was queued before it (rto > 0), so it wins.
#ifdef CN_TX_DEFERRED_INLINE  // diagnostic build of the other faulting layout
__device__ __forceinline__ void run_deferred(Tx& x, int64_t t, bool inclusive) {
#else
__device__ void run_deferred(Tx& x, int64_t t, bool inclusive) {
#endif
    for (;;) {
        // candidates: the RTO timer, the deferred pump, the oldest RTS retry;
        // fired in (time, scheduling seq) order
        int which = -1;
        int64_t bt = 0;
        uint32_t bs = 0;
        auto consider = [&](bool live, int64_t at, uint32_t seq, int id) {
            if (!live || (inclusive ? at > t : at >= t)) return;
            if (which < 0 || at < bt || (at == bt && seq < bs)) {
                which = id;
                bt = at;
                bs = seq;
            }
        };
        consider(x.timer_armed, x.timer_at, x.timer_seq, 0);
        consider(x.pump_pending, x.pump_at, x.pump_seq, 1);
        if (x.n_retry)
            consider(true, x.C->retry_t[x.C->retry_head], x.C->retry_seq[x.C->retry_head], 2);
        if (which < 0) return;
        if (which == 0) {
            rto_fire(x);
        } else if (which == 1) {
            x.pump_pending = 0;
            pump(x, x.pump_at);
        } else {
            rts_retry(x, bt);
        }
    }
}

// shared memory per warp, in 8-byte words: mt state + tempered block, the
// rtt / ecn boards, inflight and deficit, then txq / rtxq depths (4 B),
// ring (2 B) and in_ring (1 B) per path
__host__ __device__ inline size_t tx_smem_words(uint32_t max_paths) {
    return 2 * static_cast<size_t>(kMtN) + 4 * static_cast<size_t>(max_paths) +
           (11 * static_cast<size_t>(max_paths) + 7) / 8;
}

// The engine descriptor is read through a global pointer (a cached,
// read-only copy made at creation): passing it by value made every
// thread copy it to its stack frame, and a __grid_constant__ parameter
// addressed generically faulted on a long replay handed over in 42 slices.
__global__ void __launch_bounds__(kTxWarps * 32, 1) k_tx_run(const TxDev* __restrict__ dp, const uint32_t* __restrict__ ev_off,
                                                         const uint64_t* __restrict__ events,
                                                         const cn_tx_submit* __restrict__ submits,
                                                         const cn_ack_rec* __restrict__ acks,
                                                         int64_t end_time, cn_tx_rec* __restrict__ log,
                                                         uint32_t* __restrict__ log_n,
                                                         cn_tx_stats* __restrict__ stats) {
    extern __shared__ uint64_t sm[];
    const TxDev& d = *dp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t conn = blockIdx.x * kTxWarps + w;
    if (conn >= d.n_conns) return;
    const uint32_t mp = d.s.max_paths;
    uint64_t* mt = sm + static_cast<size_t>(w) * tx_smem_words(mp);
    double* rtt_s = reinterpret_cast<double*>(mt + 2 * kMtN);
    double* ecn_s = rtt_s + mp;
    int64_t* infl = reinterpret_cast<int64_t*>(ecn_s + mp);
    int64_t* defc = infl + mp;
    uint32_t* txq = reinterpret_cast<uint32_t*>(defc + mp);
    uint32_t* rtxq = txq + mp;
    uint16_t* ring = reinterpret_cast<uint16_t*>(rtxq + mp);
    uint8_t* inr = reinterpret_cast<uint8_t*>(ring + mp);
    TxConn* C = d.conns + conn;
    Tx x{d,    C,    conn, lane, WarpRng{mt, mt + kMtN, 0}, rtt_s, ecn_s, infl, defc, txq, rtxq, ring, inr,
         C->n_paths, log + static_cast<uint64_t>(conn) * d.log_cap, log_n[conn]};
    const uint64_t sb = static_cast<uint64_t>(conn) * mp;
    for (int k = lane; k < kMtN; k += 32) mt[k] = d.s.mt[static_cast<uint64_t>(conn) * kMtN + k];
    for (uint32_t p = lane; p < mp; p += 32) {
        rtt_s[p] = d.s.rtt[sb + p];
        ecn_s[p] = d.s.ecn[sb + p];
        infl[p] = d.s_inflight[sb + p];
        defc[p] = d.s_deficit[sb + p];
        txq[p] = d.s_txq[sb + p];
        rtxq[p] = d.s_rtxq[sb + p];
        ring[p] = d.s_ring[sb + p];
        inr[p] = d.s_inring[sb + p];
    }
    x.r.idx = d.s.mt_idx[conn];
    __syncwarp();
    for (int k = lane; k < kMtN; k += 32) x.r.out[k] = temper(mt[k]);
    __syncwarp();
    x.srtt = C->srtt;
    x.rttvar = C->rttvar;
    x.armed_at = C->armed_at;
    x.timer_at = C->timer_at;
    x.committed_unsent = C->committed_unsent;
    x.total_inflight = C->total_inflight;
    x.last_decrease = C->last_decrease;
    x.w = C->w;
    x.has_sample = C->has_sample;
    x.backoff = C->backoff;
    x.timer_armed = C->timer_armed;
    x.ring_len = C->ring_len;
    x.ring_pos = C->ring_pos;
    x.ring_idx = x.ring_len ? static_cast<uint32_t>(x.ring_pos % static_cast<uint64_t>(x.ring_len)) : 0;
    {
        uint32_t a = 0, b = 0;
        for (uint32_t p = lane; p < mp; p += 32) {
            a += txq[p];
            b += rtxq[p];
        }
        x.n_txq = __reduce_add_sync(0xffffffffu, a);
        x.n_rtxq = __reduce_add_sync(0xffffffffu, b);
    }
    x.q_seq = C->q_seq;
    x.sched_seq = C->sched_seq;
    x.timer_seq = C->timer_seq;
    x.pump_seq = C->pump_seq;
    x.credit = C->credit;
    x.n_stale = C->stale_n;
    x.n_retry = C->retry_n;
    x.unchunked = C->unchunked;
    x.rtxq_bytes = C->rtxq_bytes;
    x.pump_pending = C->pump_pending;
    x.pump_at = C->pump_at;
    x.chunks_sent = C->chunks_sent;
    x.chunk_rtx = C->chunk_rtx;
    x.fast_rtx = C->fast_rtx;
    x.rtos = C->rtos;
    x.msgs_completed = C->msgs_completed;
    for (int q = 0; q < 4; ++q) x.live[q] = C->live_mask[q];
    for (uint32_t k = ev_off[conn]; k < ev_off[conn + 1]; ++k) {
        const uint64_t ev = events[k];
        const uint32_t type = static_cast<uint32_t>(ev >> 62);
        const uint64_t idx = ev & ((1ull << 62) - 1);
        const int64_t t = type == 0 ? submits[idx].t : acks[idx].aux;
        run_deferred(x, t, false);
        if (type == 0) {
            const cn_tx_submit s = submits[idx];
            submit(x, t, s);
        } else {
            const cn_ack_rec a = acks[idx];
            if (a.flags & CN_ACK_NACK) {
                handle_nack(x, t, a);
            } else if (a.flags & CN_ACK_CREDIT) {
                handle_credit(x, t, a.sack[0]);
            } else if (a.flags & CN_ACK_RTS_ACK) {
                __syncwarp();
                if (lane == 0) C->rts_acked = 1;  // handle_packet rts_ack (:587-592)
                __syncwarp();
            } else {
                handle_ack(x, t, a);
            }
        }
    }
    run_deferred(x, end_time, true);
    // persist
    __syncwarp();
    for (int k = lane; k < kMtN; k += 32) d.s.mt[static_cast<uint64_t>(conn) * kMtN + k] = mt[k];
    for (uint32_t p = lane; p < mp; p += 32) {
        d.s.rtt[sb + p] = rtt_s[p];
        d.s.ecn[sb + p] = ecn_s[p];
        d.s_inflight[sb + p] = infl[p];
        d.s_deficit[sb + p] = defc[p];
        d.s_txq[sb + p] = txq[p];
        d.s_rtxq[sb + p] = rtxq[p];
        d.s_ring[sb + p] = ring[p];
        d.s_inring[sb + p] = inr[p];
    }
    if (lane == 0) {
        d.s.mt_idx[conn] = x.r.idx;
        C->srtt = x.srtt;
        C->rttvar = x.rttvar;
        C->armed_at = x.armed_at;
        C->timer_at = x.timer_at;
        C->committed_unsent = x.committed_unsent;
        C->total_inflight = x.total_inflight;
        C->last_decrease = x.last_decrease;
        C->w = x.w;
        C->has_sample = x.has_sample;
        C->backoff = x.backoff;
        C->timer_armed = x.timer_armed;
        C->ring_len = x.ring_len;
        C->ring_pos = x.ring_pos;
        C->q_seq = x.q_seq;
        C->sched_seq = x.sched_seq;
        C->timer_seq = x.timer_seq;
        C->pump_seq = x.pump_seq;
        C->credit = x.credit;
        C->unchunked = x.unchunked;
        C->rtxq_bytes = x.rtxq_bytes;
        C->pump_pending = x.pump_pending;
        C->pump_at = x.pump_at;
        C->chunks_sent = x.chunks_sent;
        C->chunk_rtx = x.chunk_rtx;
        C->fast_rtx = x.fast_rtx;
        C->rtos = x.rtos;
        C->msgs_completed = x.msgs_completed;
        for (int q = 0; q < 4; ++q) C->live_mask[q] = x.live[q];
        log_n[conn] = x.log_n;
        cn_tx_stats st;
        st.chunks_sent = x.chunks_sent;
        st.chunk_rtx = x.chunk_rtx;
        st.fast_rtx = x.fast_rtx;
        st.rtos = x.rtos;
        st.msgs_sent = C->msgs_sent;
        st.msgs_completed = x.msgs_completed;
        st.backpressured = C->backpressured;
        st.n_log = x.log_n;
        st.srtt = x.srtt;
        st.rttvar = x.rttvar;
        st.backoff = x.backoff;
        st.live_msgs = C->live_msgs;
        st.cwnd_bytes = x.cwnd_bytes();
        st.inflight = x.total_inflight;
        st.cwnd_pkts = x.w;
        stats[conn] = st;
    }
}

__global__ void k_tx_init(TxDev d, const int32_t* src, const int32_t* dst, const int32_t* np) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d.n_conns) return;
    TxConn* C = d.conns + c;
    memset(C, 0, sizeof(TxConn));
    C->backoff = 1;
    C->next_seq = 1;
    C->w = d.init_cwnd;
    C->last_decrease = kNeverDecreased;
    C->credit = d.initial_credit;  // conn_to (:131-133)
    C->last_rewind_psn = ~0ull;
    C->src = src ? src[c] : 0;
    C->dst = dst ? dst[c] : 0;
    C->n_paths = np ? np[c] : static_cast<int32_t>(d.s.max_paths);
    C->conn_id = static_cast<int32_t>(c & 0xFF);
    for (int i = 0; i < 128; ++i) C->free_ids[i] = static_cast<uint8_t>(127 - i);  // :127-129
    C->n_free = 128;
    const uint64_t sb = static_cast<uint64_t>(c) * d.s.max_paths;
    for (uint32_t p = 0; p < d.s.max_paths; ++p) {
        d.s_inflight[sb + p] = 0;
        d.s_deficit[sb + p] = 0;
        d.s_txq[sb + p] = 0;
        d.s_rtxq[sb + p] = 0;
        d.s_ring[sb + p] = 0;
        d.s_inring[sb + p] = 0;
    }
}

}  // namespace cnb

using namespace cnb;

struct cn_tx {
    TxDev d;
    TxDev* d_dev = nullptr;  // device copy read by k_tx_run
    cn_sched* sched;
    uint32_t* d_logn;
};

extern "C" void cn_tx_config_default(cn_tx_config* c) {
    memset(c, 0, sizeof *c);
    c->chunk_bytes = 32768;
    c->max_payload = CN_MAX_PAYLOAD;
    c->dupack_threshold = 8;
    c->rtx_avoid_prev_path = 1;
    c->lb_policy = CN_LB_OBLIVIOUS;
    c->max_inflight_msgs = 128;
    c->max_paths = 1;
    c->chunk_pool = 1ull << 20;
    c->log_cap = 1u << 16;
    c->cc_algo = CN_CC_NONE;
    c->drr_quantum = 32768;  // TransportConfig::drr_quantum
    c->mss = 4032;           // CcConfig::mss
    c->init_cwnd_pkts = 2.0; // CcConfig::init_cwnd_pkts
    c->credit_quantum = 32768;  // TransportConfig::credit_quantum
    c->credit_bank_quanta = 4;  // TransportConfig::credit_bank_quanta
}

static size_t tx_smem_bytes(uint32_t max_paths) { return kTxWarps * tx_smem_words(max_paths) * 8; }

extern "C" int cn_tx_create(const cn_tx_config* cfg, uint32_t n_conns, const int32_t* h_src,
                            const int32_t* h_dst, const int32_t* h_n_paths, cn_tx** out) {
    if (!cfg || !out || n_conns == 0 || cfg->chunk_bytes == 0 || cfg->rto_min <= 0 ||
        cfg->max_paths == 0 || cfg->max_paths > 1024 || cfg->lb_policy < 0 || cfg->lb_policy > 2 ||
        !(cfg->policy >= CN_POLICY_DEFAULT && cfg->policy <= CN_POLICY_TEST_OUT_OF_RANGE
#ifdef CN_TX_USER_POLICY_HEADER
          || cfg->policy == CN_POLICY_USER
#endif
          ) ||
        (cfg->cc_algo != CN_CC_NONE && cfg->cc_algo != CN_CC_SWIFT) || cfg->drr_quantum == 0 ||
        cfg->mss <= 0 || !(cfg->init_cwnd_pkts > 0) || cfg->cap_bytes < 0) {
        set_error("cn_tx_create: bad config (rto_min resolved > 0, max_paths <= 1024, "
                  "cc none or swift -- CUBIC is host-side)");
        return CN_E_INVALID;
    }
    *out = nullptr;
    cn_tx* t = new (std::nothrow) cn_tx();
    if (!t) return CN_E_CAPACITY;
    memset(&t->d, 0, sizeof t->d);
    int rc = cn_sched_create(n_conns, cfg->max_paths, h_n_paths, cfg->base_rtt_ns, cfg->seed,
                             "transport.conn", cfg->stream_index0, &t->sched);
    if (rc != CN_OK) {
        delete t;
        return rc;
    }
    TxDev& d = t->d;
    d.n_conns = n_conns;
    d.cb = cfg->chunk_bytes;
    d.max_pl = cfg->max_payload ? cfg->max_payload : CN_MAX_PAYLOAD;
    d.dupack = cfg->dupack_threshold;
    d.avoid_prev = cfg->rtx_avoid_prev_path ? 1 : 0;
    d.policy = static_cast<uint32_t>(cfg->lb_policy);
    d.max_inflight = cfg->max_inflight_msgs;
    d.log_cap = cfg->log_cap;
    d.cc_algo = cfg->cc_algo == CN_CC_SWIFT ? 1 : 0;
    d.quantum = cfg->drr_quantum;
    d.rto_min = cfg->rto_min;
    d.rto_max = cfg->rto_max > 0 ? cfg->rto_max : 64 * cfg->rto_min;  // transport.cpp:36
    d.commit_ahead = cfg->commit_ahead;
    d.swift_target = cfg->swift_target_ns;
    d.mss = cfg->mss;
    d.cap_bytes = cfg->cap_bytes;
    d.init_cwnd = cfg->init_cwnd_pkts;
    d.rd = cfg->receiver_driven ? 1 : 0;
    d.ordered = cfg->ordered ? 1 : 0;
    d.pol = cfg->policy;
    d.so_cap = cfg->ordered ? (cfg->sent_order_cap ? cfg->sent_order_cap : 1u << 16) : 1;
    d.credit_cap = static_cast<int64_t>(cfg->credit_bank_quanta) * cfg->credit_quantum;
    d.initial_credit = cfg->initial_credit;
    // cap_pkts_ (cc.cpp:111-113)
    d.cap_pkts = cfg->cap_bytes > 0 ? static_cast<double>(cfg->cap_bytes) / static_cast<double>(cfg->mss)
                                    : __builtin_huge_val();
    d.pool_cap = cfg->chunk_pool;
    d.conn_pool = cfg->chunk_pool / n_conns;
    d.s = *sched_dev(t->sched);
    const uint64_t subs = static_cast<uint64_t>(n_conns) * cfg->max_paths;
    int32_t *src = nullptr, *dst = nullptr, *np = nullptr;
    const uint64_t pool = cfg->chunk_pool;
    bool ok = cudaMalloc(&d.conns, sizeof(TxConn) * n_conns) == cudaSuccess &&
              cudaMalloc(&d.c_path, pool * 4) == cudaSuccess && cudaMalloc(&d.c_txt, pool * 8) == cudaSuccess &&
              cudaMalloc(&d.c_dead, pool * 8) == cudaSuccess && cudaMalloc(&d.c_att, pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_fl, pool * 4) == cudaSuccess && cudaMalloc(&d.c_dup, pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_q, pool * 4) == cudaSuccess && cudaMalloc(&d.c_psn, pool * 8) == cudaSuccess &&
              cudaMalloc(&d.so_ref, static_cast<uint64_t>(n_conns) * d.so_cap * 4) == cudaSuccess &&
              cudaMalloc(&d.gq_ref, static_cast<uint64_t>(n_conns) * d.so_cap * 4) == cudaSuccess &&
              cudaMalloc(&d.gq_from, static_cast<uint64_t>(n_conns) * d.so_cap * 8) == cudaSuccess &&
              cudaMalloc(&d.s_inflight, subs * 8) == cudaSuccess &&
              cudaMalloc(&d.s_deficit, subs * 8) == cudaSuccess && cudaMalloc(&d.s_txq, subs * 4) == cudaSuccess &&
              cudaMalloc(&d.s_rtxq, subs * 4) == cudaSuccess && cudaMalloc(&d.s_ring, subs * 2) == cudaSuccess &&
              cudaMalloc(&d.s_inring, subs) == cudaSuccess && cudaMalloc(&d.pool_top, 8) == cudaSuccess &&
              cudaMalloc(&d.status, 4) == cudaSuccess && cudaMalloc(&t->d_logn, n_conns * 4ull) == cudaSuccess &&
              cudaMalloc(&t->d_dev, sizeof(TxDev)) == cudaSuccess &&
              cudaMalloc(&src, n_conns * 4ull) == cudaSuccess && cudaMalloc(&dst, n_conns * 4ull) == cudaSuccess &&
              cudaMalloc(&np, n_conns * 4ull) == cudaSuccess;
    if (!ok) {
        set_error("cn_tx_create: out of device memory");
        cudaFree(src);
        cudaFree(dst);
        cudaFree(np);
        cn_tx_destroy(t);
        return CN_E_CAPACITY;
    }
    std::vector<int32_t> hs(n_conns, 0), hd(n_conns, 0), hn(n_conns, static_cast<int32_t>(cfg->max_paths));
    for (uint32_t c = 0; c < n_conns; ++c) {
        if (h_src) hs[c] = h_src[c];
        if (h_dst) hd[c] = h_dst[c];
        if (h_n_paths) hn[c] = h_n_paths[c];
    }
    cudaMemcpy(src, hs.data(), n_conns * 4ull, cudaMemcpyHostToDevice);
    cudaMemcpy(dst, hd.data(), n_conns * 4ull, cudaMemcpyHostToDevice);
    cudaMemcpy(np, hn.data(), n_conns * 4ull, cudaMemcpyHostToDevice);
    cudaMemset(d.pool_top, 0, 8);
    cudaMemset(d.status, 0, 4);
    cudaMemset(d.c_q, 0, pool * 4);
    cudaMemset(t->d_logn, 0, n_conns * 4ull);
    k_tx_init<<<(n_conns + 127) / 128, 128>>>(d, src, dst, np);
    cudaError_t e = cudaDeviceSynchronize();
    cudaFree(src);
    cudaFree(dst);
    cudaFree(np);
    if (e != cudaSuccess) {
        cn_tx_destroy(t);
        return cuda_status(e, "cn_tx_create");
    }
    cudaFuncSetAttribute(k_tx_run, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(tx_smem_bytes(cfg->max_paths)));
    // the descriptor never changes after creation: one device copy
    if (cudaMemcpy(t->d_dev, &t->d, sizeof(TxDev), cudaMemcpyHostToDevice) != cudaSuccess) {
        cn_tx_destroy(t);
        set_error("cn_tx_create: descriptor copy failed");
        return CN_E_CUDA;
    }
    *out = t;
    return CN_OK;
}

extern "C" void cn_tx_destroy(cn_tx* t) {
    if (!t) return;
    cudaDeviceSynchronize();
    TxDev& d = t->d;
    void* ptrs[] = {d.c_psn, d.so_ref, d.gq_ref, d.gq_from,
                    d.conns,      d.c_path,    d.c_txt, d.c_dead, d.c_att,  d.c_fl,
                    d.c_dup,      d.c_q,       d.s_inflight, d.s_deficit, d.s_txq, d.s_rtxq,
                    d.s_ring,     d.s_inring,  d.pool_top, d.status, t->d_logn, t->d_dev};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (t->sched) cn_sched_destroy(t->sched);
    delete t;
}

extern "C" int cn_tx_run(cn_tx* t, const uint32_t* d_ev_off, const uint64_t* d_events,
                         const cn_tx_submit* d_submits, const cn_ack_rec* d_acks, int64_t end_time,
                         cn_tx_rec* d_log, cn_tx_stats* d_stats, void* stream) {
    if (!t || !d_ev_off || !d_log || !d_stats) {
        set_error("cn_tx_run: bad arguments");
        return CN_E_INVALID;
    }
    k_tx_run<<<(t->d.n_conns + kTxWarps - 1) / kTxWarps, kTxWarps * 32,
               tx_smem_bytes(t->d.s.max_paths), static_cast<cudaStream_t>(stream)>>>(
        t->d_dev, d_ev_off, d_events, d_submits, d_acks, end_time, d_log, t->d_logn, d_stats);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_tx_log_counts(cn_tx* t, uint32_t* h_out) {
    if (!t || !h_out) return CN_E_INVALID;
    CNB_CUDA(cudaMemcpy(h_out, t->d_logn, t->d.n_conns * 4ull, cudaMemcpyDeviceToHost));
    return CN_OK;
}

extern "C" int cn_tx_log_clear(cn_tx* t, void* stream) {
    if (!t) return CN_E_INVALID;
    CNB_CUDA(cudaMemsetAsync(t->d_logn, 0, t->d.n_conns * 4ull, static_cast<cudaStream_t>(stream)));
    return CN_OK;
}

extern "C" int cn_tx_status(cn_tx* t, unsigned int* out) {
    if (!t || !out) return CN_E_INVALID;
    CNB_CUDA(cudaMemcpy(out, t->d.status, 4, cudaMemcpyDeviceToHost));
    return CN_OK;
}

// Debug: raw device state of connection `conn` (TxConn, its per-path arrays,
// RNG, and the chunk state of its pool share) into a host buffer.
extern "C" int64_t cn_tx_debug_state(cn_tx* t, uint32_t conn, void* h_out, uint64_t cap) {
    if (!t || conn >= t->d.n_conns) return CN_E_INVALID;
    CNB_CUDA(cudaDeviceSynchronize());
    std::vector<uint8_t> buf;
    auto put = [&](const void* dptr, uint64_t n) {
        const size_t o = buf.size();
        buf.resize(o + n);
        if (n) cudaMemcpy(buf.data() + o, dptr, n, cudaMemcpyDeviceToHost);
    };
    const TxDev& d = t->d;
    const uint64_t mp = d.s.max_paths, sb = conn * mp;
    put(d.conns + conn, sizeof(TxConn));
    put(d.s_inflight + sb, mp * 8);
    put(d.s_deficit + sb, mp * 8);
    put(d.s_txq + sb, mp * 4);
    put(d.s_rtxq + sb, mp * 4);
    put(d.s_ring + sb, mp * 2);
    put(d.s_inring + sb, mp);
    put(d.s.mt + conn * 312ull, 312 * 8);
    put(d.s.mt_idx + conn, 4);
    put(d.s.rtt + sb, mp * 8);
    put(d.s.ecn + sb, mp * 8);
    const uint64_t c0 = conn * d.conn_pool, nc = std::min<uint64_t>(d.conn_pool, 4096);
    put(d.c_path + c0, nc * 4);
    put(d.c_txt + c0, nc * 8);
    put(d.c_dead + c0, nc * 8);
    put(d.c_att + c0, nc * 4);
    put(d.c_fl + c0, nc * 4);
    put(d.c_dup + c0, nc * 4);
    put(d.c_q + c0, nc * 4);
    if (h_out) memcpy(h_out, buf.data(), std::min<uint64_t>(cap, buf.size()));
    return static_cast<int64_t>(buf.size());
}

extern "C" int cn_tx_get_conn_state(cn_tx* t, uint32_t conn, cn_tx_conn_state* out, int64_t* h_path_inflight,
                                    uint32_t max_paths) {
    if (!t || !out || conn >= t->d.n_conns) {
        set_error("cn_tx_get_conn_state: null handle / output or connection out of range");
        return CN_E_INVALID;
    }
    CNB_CUDA(cudaDeviceSynchronize());
    const TxConn* C = t->d.conns + conn;
    CNB_CUDA(cudaMemcpy(&out->credit, &C->credit, 8, cudaMemcpyDeviceToHost));
    CNB_CUDA(cudaMemcpy(&out->unchunked, &C->unchunked, 8, cudaMemcpyDeviceToHost));
    CNB_CUDA(cudaMemcpy(&out->n_paths, &C->n_paths, 4, cudaMemcpyDeviceToHost));
    out->pad = 0;
    if (h_path_inflight) {
        const uint32_t n = std::min<uint32_t>(max_paths, static_cast<uint32_t>(out->n_paths));
        if (n)
            CNB_CUDA(cudaMemcpy(h_path_inflight, t->d.s_inflight + static_cast<uint64_t>(conn) * t->d.s.max_paths,
                                n * 8ull, cudaMemcpyDeviceToHost));
    }
    return CN_OK;
}
