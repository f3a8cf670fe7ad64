// tx.cu -- device sender engine: message dispatch over a host's engines,
// chunk commit and window-gated egress, ack processing, loss detection,
// retransmission and congestion control of the selective multipath
// transport (sm_100a).
//
// Restates the reference sender's event handling per SOURCE HOST
// (/root/reference/proj/src/transport.cpp) -- everything a host's engines
// share is shared here too:
//   conn_to (home engine)            :84-137    (least-loaded gauge at creation)
//   send_message / dispatch          :144-218   (msg ids LIFO :127-129; engine:
//                                                home, or least-loaded under
//                                                conn_split; max_inflight_msgs
//                                                per engine)
//   schedule_pump / pump             :222-240   (one deferred pump per engine)
//   commit_chunks                    :244-310   (per-engine factory rotation over
//                                                the host's messages, 128-chunk
//                                                window stall, per-engine
//                                                commit_ahead, path bound at
//                                                commit, cross-engine pumps)
//   can_send / gated_inflight        :312-325   (global or per-path CC scope,
//                                                credit gate)
//   egress                           :329-431   (retransmission queues in ring
//                                                order, then DRR over the
//                                                engine's ring of (conn, path))
//   send_chunk                       :433-494   queue_rtx :516-542
//   release / advance / finish       :807-847   handle_ack :849-942
//   handle_nack / gbn_rewind         :944-999   receiver-driven glue :1003-1074
//   cur_rto / arm_rto / rto_fire     :1078-1169 (on_rto once per distinct CC)
//   RttEstimator cc.hpp:12-35; OpenLoop / CUBIC / Swift cc.cpp:19-156
// CUBIC's std::cbrt / std::pow are glibc's, restated bit-exactly in
// libm_exact.cuh; every IEEE operation of the CC updates is an explicit
// round-to-nearest intrinsic in the reference's evaluation order.
//
// Execution model.  One warp per source host consumes the host's
// time-ordered input events (message submissions, acks / NACKs / credits /
// rts_acks delivered at the host) and fires, in the event queue's
// (time, seq) order, what the run itself schedules: RTO timers per
// connection, deferred pumps per engine, RTS retries.  All warp-uniform
// state lives ONCE in shared memory (the host header, its engines, and per
// connection: counters, timer / retry lists, Mersenne state, per-path
// arrays, CC instances); every lane reads it, lane 0 writes it between
// __syncwarp barriers (wr()), so lanes cannot hold diverging copies.  Lanes
// work in parallel on chunk windows (one chunk per lane, ballots), queue
// fronts and idle DRR visits.  The shared-memory image of a host and of
// each connection is a contiguous blob persisted in global memory between
// launches (cn_tx_run calls resume where the last one stopped).
//
// Queues.  Each chunk carries a queue tag c_q = kind | seq (seq from a
// per-connection counter, 0 = not queued).  The front of sub-connection
// (c, p)'s tx or retransmission queue is c's queued chunk of that kind on p
// with the smallest seq -- the reference's FIFO order.  Stale entries (a
// chunk acked while awaiting retransmission) are kept per connection as
// (seq, path) and popped by egress without effect (:347-351).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "chunknet_policy.cuh"
#include "common.cuh"
#include "libm_exact.cuh"
#include "rng.cuh"
#ifdef CN_TX_USER_POLICY_HEADER
#include CN_TX_USER_POLICY_HEADER  // defines struct CnUserPolicy (make USER_POLICY=...)
#endif

namespace cnb {

enum : uint32_t { TF_SENT = 1, TF_ACKED = 2, TF_RTXP = 4 };
constexpr uint32_t kQRtx = 0x80000000u;  // c_q kind bit: retransmission queue
constexpr int kTxWindow = 128;           // kCsnWindow (transport.cpp:14)
constexpr int kBackoffCap = 64;          // kBackoffCap (transport.cpp:15)
constexpr int kMaxEngines = 16;
constexpr uint32_t kTmrMax = 8;     // RTO timer events pending for one arming instant
constexpr uint32_t kRetryMax = 32;  // pending RTS retry events per connection
constexpr uint32_t kStaleMax = 256;  // stale retransmission-queue entries per connection
constexpr int64_t kNeverDecreased = LLONG_MIN / 2;  // cc.cpp:17
// cc.cpp:11-16
constexpr double kCubicC = 0.4, kCubicBeta = 0.7;
constexpr double kSwiftAi = 1.0, kSwiftMdScale = 0.8, kSwiftMaxMd = 0.5, kMinCwndPkts = 1.0;
enum : int32_t { CC_NONE = 0, CC_CUBIC = 1, CC_SWIFT = 2 };

struct TxMsg {  // MsgSend (transport.hpp:129-142)
    uint64_t seq, tag, len, chunked, chunk_base;
    uint32_t nchunks, base, acked, live, in_factory, engine;
};

// per connection, global memory (touched at submit / finish / ordered mode)
struct TxConnG {
    uint64_t next_seq, msgs_sent, backpressured, p_head;
    int32_t n_free, src, dst, conn_id;
    uint64_t next_psn, last_rewind_psn;  // ordered reliability (go-back-N)
    uint32_t so_n, gq_head, gq_n, stale_n;
    uint32_t stale_seq[kStaleMax];  // acked-while-pending rtx queue entries: (queue seq, path)
    uint16_t stale_path[kStaleMax];
    uint64_t p_start[128];  // ring position (monotonic) of each live message's chunks
    uint8_t free_ids[128];
    TxMsg msgs[128];
};

// CongestionControl instance (cc.cpp) + its RttEstimator (cc.hpp:12-35)
struct Cc {
    double w, w_max, ssthresh, k;
    int64_t epoch_start, last_decrease, srtt, rttvar, cwnd;  // cwnd: cwnd_bytes() after the last update
    int32_t has_sample, pad;
    uint64_t decreases;
};

// Engine (transport.hpp:244-253)
struct Eng {
    int64_t committed_unsent, gauge, pump_at;
    uint64_t dispatched, ring_pos;
    int32_t inflight_msgs, ring_len;
    uint32_t fq_head, fq_count, pump_pending, pump_seq;
};

struct HostHdr {
    uint32_t n_conns, sched_seq, log_n, pad;
    uint64_t sends;  // chunks_sent + chunk_rtx of the host (pump's progress test, :236-238)
};

// per connection, shared memory (the warp-uniform hot state)
struct CHot {
    int64_t total_inflight;  // sum of the subs' inflight (global-scope gate)
    int64_t armed_at, credit, unchunked, rtxq_bytes, txq_bytes;
    uint64_t chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_completed, rts_sent;
    int32_t backoff, timer_armed, n_paths, home, opened, conn;
    uint32_t n_txq, n_rtxq, n_stale, q_seq, mt_idx, tmr_n, retry_head, retry_n, rts_outstanding, rts_acked;
    uint32_t live[4];
    int64_t tmr_t[kTmrMax];
    uint32_t tmr_seq[kTmrMax];
    int64_t retry_t[kRetryMax];
    uint32_t retry_seq[kRetryMax];
    uint64_t pol_state[4];
};

struct TxDev {
    uint32_t n_conns, n_hosts, max_paths, mcph, engines, conn_split, per_path, n_cc;
    uint32_t cb, max_pl, dupack, avoid_prev, lbp, max_inflight, log_cap, cc_algo, quantum;
    uint32_t rd, ordered, so_cap, ecn_as_loss;
    int32_t pol;  // CN_POLICY_*
    int64_t rto_min, rto_max, commit_ahead, swift_target, mss, cap_bytes, credit_cap, initial_credit;
    double init_cwnd, cap_pkts, base_rtt;
    uint64_t pool_cap, conn_pool;  // conn_pool = pool_cap / n_conns entries per connection
    uint32_t host_bytes, conn_bytes;  // shared-memory blob sizes
    uint32_t ring_cap, fq_cap;
    // blob offsets inside a connection blob (bytes)
    uint32_t o_mt, o_rtt, o_ecn, o_infl, o_def, o_cc, o_txq, o_rtxq, o_inr;
    TxConnG* conns;
    uint8_t* host_blob;  // [n_hosts][host_bytes]
    uint8_t* conn_blob;  // [n_conns][conn_bytes]
    uint32_t* host_conns;  // [n_hosts][mcph] global connection indices
    uint32_t* host_nconns;  // [n_hosts]
    uint32_t* conn_local;   // [n_conns] index within its host
    uint32_t* ring;         // [n_hosts][engines][ring_cap] (conn local << 16 | path)
    uint32_t* fq;           // [n_hosts][engines][fq_cap] (conn local << 8 | msg id)
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
    unsigned int* status;
};

// Debug builds (make EXTRA=-DCN_TX_CHECK_UNIFORM): every value the warp
// branches on at the handlers' decision points must be equal in all 32
// lanes; a divergent one sets CN_TX_STATUS_INTERNAL.
#ifdef CN_TX_CHECK_UNIFORM
#define CN_UNIFORM(d_, v_)                                                                      \
    do {                                                                                        \
        int pred_;                                                                              \
        __match_all_sync(0xffffffffu, static_cast<unsigned long long>(v_), &pred_);             \
        if (!pred_) atomicOr((d_).status, CN_TX_STATUS_INTERNAL);                               \
    } while (0)
#else
#define CN_UNIFORM(d_, v_) \
    do {                   \
    } while (0)
#endif

template <class T>
__device__ __forceinline__ void wr(T& ref, T v, int lane) {  // single-writer store of warp-uniform state
    __syncwarp();
    if (lane == 0) ref = v;
    __syncwarp();
}

// ------------------------------------------------------------ CC (lane 0)
// CongestionControl::cwnd_bytes: OpenLoop (cc.cpp:21-22), CUBIC (:79-81), Swift (:146-148)
__device__ __forceinline__ int64_t cc_cwnd(const TxDev& d, const Cc& c) {
    if (d.cc_algo == CC_NONE) return d.cap_bytes > 0 ? d.cap_bytes : LLONG_MAX / 4;
    return llround(__dmul_rn(c.w, static_cast<double>(d.mss)));
}
__device__ __forceinline__ void est_sample(Cc& c, int64_t rtt) {  // RttEstimator::sample (cc.hpp:17-28)
    if (!c.has_sample) {
        c.srtt = rtt;
        c.rttvar = rtt / 2;
        c.has_sample = 1;
        return;
    }
    const int64_t err = c.srtt > rtt ? c.srtt - rtt : rtt - c.srtt;
    c.rttvar = (3 * c.rttvar + err) / 4;
    c.srtt = (7 * c.srtt + rtt) / 8;
}
__device__ __forceinline__ double kdiv_cubic(double w_max) {  // cbrt(w_max * (1 - beta) / C)
    return libm_cbrt(__ddiv_rn(__dmul_rn(w_max, 1.0 - kCubicBeta), kCubicC));
}
__device__ void cubic_decrease(const TxDev& d, Cc& c, int64_t now) {  // Cubic::decrease (cc.cpp:84-95)
    if (c.has_sample && now - c.last_decrease < c.srtt) return;
    c.last_decrease = now;
    c.decreases += 1;
    c.w_max = c.w;
    const double nw = __dmul_rn(c.w, kCubicBeta);
    c.w = nw > kMinCwndPkts ? nw : kMinCwndPkts;
    c.ssthresh = c.w;
    c.k = kdiv_cubic(c.w_max);
    c.epoch_start = now;
}
__device__ void cc_on_ack(const TxDev& d, Cc& c, int64_t now, int64_t acked, int64_t rtt, bool ecn) {
    if (rtt > 0) est_sample(c, rtt);  // every algorithm samples (cc.cpp:23-25, :46, :117)
    if (d.cc_algo == CC_CUBIC) {  // cc.cpp:45-66
        if (ecn && d.ecn_as_loss) {
            cubic_decrease(d, c, now);
        } else if (acked > 0) {
            const double acked_pkts = __ddiv_rn(static_cast<double>(acked), static_cast<double>(d.mss));
            if (c.w < c.ssthresh) {
                const double nw = __dadd_rn(c.w, acked_pkts);
                c.w = d.cap_pkts < nw ? d.cap_pkts : nw;
            } else {
                if (c.epoch_start < 0) {
                    c.epoch_start = now;
                    if (c.w_max < c.w) c.w_max = c.w;
                    c.k = kdiv_cubic(c.w_max);
                }
                const double t = __dmul_rn(static_cast<double>(now - c.epoch_start), 1e-9);
                const double target = __dadd_rn(__dmul_rn(kCubicC, libm_pow3(__dsub_rn(t, c.k))), c.w_max);
                if (target > c.w)
                    c.w = __dadd_rn(c.w, __dmul_rn(__ddiv_rn(__dsub_rn(target, c.w), c.w), acked_pkts));
                c.w = d.cap_pkts < c.w ? d.cap_pkts : c.w;
            }
        }
    } else if (d.cc_algo == CC_SWIFT) {  // cc.cpp:115-131
        if (rtt <= d.swift_target) {
            if (acked > 0) {
                const double a = __ddiv_rn(static_cast<double>(acked), static_cast<double>(d.mss));
                const double nw = __dadd_rn(c.w, __ddiv_rn(__dmul_rn(kSwiftAi, a), c.w));
                c.w = d.cap_pkts < nw ? d.cap_pkts : nw;
            }
        } else if (!(now - c.last_decrease < c.srtt)) {
            const double q = __ddiv_rn(__dmul_rn(kSwiftMdScale, static_cast<double>(rtt - d.swift_target)),
                                       static_cast<double>(rtt));
            double f = __dsub_rn(1.0, q);
            if (f < kSwiftMaxMd) f = kSwiftMaxMd;
            const double nw = __dmul_rn(c.w, f);
            c.w = nw < kMinCwndPkts ? kMinCwndPkts : nw;
            c.last_decrease = now;
            c.decreases += 1;
        }
    }
    c.cwnd = cc_cwnd(d, c);
}
__device__ void cc_on_loss(const TxDev& d, Cc& c, int64_t now) {
    if (d.cc_algo == CC_CUBIC) {
        cubic_decrease(d, c, now);  // cc.cpp:68
    } else if (d.cc_algo == CC_SWIFT) {  // cc.cpp:133-138
        if (c.has_sample && now - c.last_decrease < c.srtt) return;
        const double nw = __dmul_rn(c.w, kSwiftMaxMd);
        c.w = nw < kMinCwndPkts ? kMinCwndPkts : nw;
        c.last_decrease = now;
        c.decreases += 1;
    }
    c.cwnd = cc_cwnd(d, c);
}
__device__ void cc_on_rto(const TxDev& d, Cc& c, int64_t now) {
    if (d.cc_algo == CC_CUBIC) {  // cc.cpp:70-77
        const double s = __dmul_rn(c.w, kCubicBeta);
        c.ssthresh = s > kMinCwndPkts ? s : kMinCwndPkts;
        c.w_max = c.w;
        c.w = kMinCwndPkts;
        c.epoch_start = -1;
        c.last_decrease = now;
        c.decreases += 1;
    } else if (d.cc_algo == CC_SWIFT) {  // cc.cpp:140-144
        c.w = kMinCwndPkts;
        c.last_decrease = now;
        c.decreases += 1;
    }
    c.cwnd = cc_cwnd(d, c);
}
__device__ __forceinline__ int64_t rto_of(const TxDev& d, const Cc& c) {  // RttEstimator::rto (cc.hpp:30-35)
    const int64_t x = c.srtt + 4 * c.rttvar;
    if (x < d.rto_min) return d.rto_min;
    if (x > d.rto_max) return d.rto_max;
    return x;
}

// ------------------------------------------------------------ per warp
struct Tx {
    const TxDev& d;
    const uint32_t host;
    const int lane;
    HostHdr* hh;
    Eng* eng;         // [engines]
    uint8_t* cblob;   // connection blobs, conn_bytes apart
    uint32_t* ring;   // this host's rings [engines][ring_cap]
    uint32_t* fq;     // this host's factories [engines][fq_cap]
    cn_tx_rec* log;

    __device__ CHot* H(int k) const { return reinterpret_cast<CHot*>(cblob + static_cast<size_t>(k) * d.conn_bytes); }
    __device__ uint8_t* B(int k) const { return cblob + static_cast<size_t>(k) * d.conn_bytes; }
    __device__ uint64_t* mt(int k) const { return reinterpret_cast<uint64_t*>(B(k) + d.o_mt); }
    __device__ double* rtt_s(int k) const { return reinterpret_cast<double*>(B(k) + d.o_rtt); }
    __device__ double* ecn_s(int k) const { return reinterpret_cast<double*>(B(k) + d.o_ecn); }
    __device__ int64_t* infl(int k) const { return reinterpret_cast<int64_t*>(B(k) + d.o_infl); }
    __device__ int64_t* defc(int k) const { return reinterpret_cast<int64_t*>(B(k) + d.o_def); }
    __device__ uint32_t* txq_n(int k) const { return reinterpret_cast<uint32_t*>(B(k) + d.o_txq); }
    __device__ uint32_t* rtxq_n(int k) const { return reinterpret_cast<uint32_t*>(B(k) + d.o_rtxq); }
    __device__ uint8_t* in_ring(int k) const { return B(k) + d.o_inr; }
    // the CongestionControl of sub-connection (k, p): cc_store[0] under
    // global scope, cc_store[p] under per-path scope (conn_to, :113-123)
    __device__ Cc* cc(int k, int p) const {
        return reinterpret_cast<Cc*>(B(k) + d.o_cc) + (d.per_path ? p : 0);
    }
    __device__ TxConnG* G(int k) const { return d.conns + H(k)->conn; }
    __device__ uint32_t* eng_ring(int e) const { return ring + static_cast<size_t>(e) * d.ring_cap; }
    __device__ uint32_t* eng_fq(int e) const { return fq + static_cast<size_t>(e) * d.fq_cap; }
    __device__ int sub_engine(int k, int p) const {  // SubConn::engine (:112)
        return d.conn_split ? p % static_cast<int>(d.engines) : H(k)->home;
    }

    __device__ uint32_t next_seq() {  // the host's event scheduling sequence
        const uint32_t s = hh->sched_seq + 1;
        wr(hh->sched_seq, s, lane);
        return s;
    }
    // gated_inflight (:320-325) and can_send (:312-316)
    __device__ int64_t gated(int k, int p) const {
        return d.per_path ? infl(k)[p] : H(k)->total_inflight;
    }
    __device__ bool can_send(int k, int p) const {
        return gated(k, p) < cc(k, p)->cwnd && (!d.rd || H(k)->credit > 0);
    }
    __device__ void add_inflight(int k, int p, int64_t delta) {  // clamped at 0 (:520-521, :813-814)
        int64_t* ip = infl(k) + p;
        const int64_t old = *ip;
        int64_t v = old + delta;
        if (v < 0) v = 0;
        const int64_t tot = H(k)->total_inflight + (v - old);
        __syncwarp();
        if (lane == 0) {
            *ip = v;
            H(k)->total_inflight = tot;
        }
        __syncwarp();
    }
    __device__ void ring_insert(int k, int p) {  // :296-300, :537-540
        if (in_ring(k)[p]) return;
        const int e = sub_engine(k, p);
        const int32_t n = eng[e].ring_len;
        if (static_cast<uint32_t>(n) >= d.ring_cap) {
            if (lane == 0) atomicOr(d.status, CN_TX_STATUS_CAPACITY);
            return;
        }
        __syncwarp();
        if (lane == 0) {
            in_ring(k)[p] = 1;
            eng_ring(e)[n] = (static_cast<uint32_t>(k) << 16) | static_cast<uint32_t>(p);
            eng[e].ring_len = n + 1;
        }
        __syncwarp();
    }
    __device__ void schedule_pump(int e, int64_t now) {  // :222-230
        if (eng[e].pump_pending) return;
        const uint32_t s = next_seq();
        __syncwarp();
        if (lane == 0) {
            eng[e].pump_pending = 1;
            eng[e].pump_at = now;
            eng[e].pump_seq = s;
        }
        __syncwarp();
    }
    // arm_rto (:1083-1092): one live timer per connection; the event list
    // holds the events armed at the current armed_at (older ones are
    // superseded and can never fire, :1096-1097)
    __device__ void add_timer(int k, int64_t now, int64_t at) {
        CHot* h = H(k);
        const uint32_t s = next_seq();
        const uint32_t n = h->armed_at == now && h->timer_armed ? h->tmr_n : 0;
        __syncwarp();
        if (lane == 0) {
            h->timer_armed = 1;
            h->armed_at = now;
            if (n < kTmrMax) {
                h->tmr_t[n] = at;
                h->tmr_seq[n] = s;
                h->tmr_n = n + 1;
            } else {
                atomicOr(d.status, CN_TX_STATUS_TIMER);
            }
        }
        __syncwarp();
    }
    __device__ void arm_rto(int k, int64_t now) {
        CHot* h = H(k);
        if (h->timer_armed) return;
        add_timer(k, now, now + rto_of(d, *cc(k, 0)) * h->backoff);
    }
    // handle_ack's re-arm (:936-940): timer_armed = false then arm_rto; the
    // events armed at this same instant stay live
    __device__ void rearm(int k, int64_t now) {
        CHot* h = H(k);
        const bool keep = h->timer_armed && h->armed_at == now;
        __syncwarp();
        if (lane == 0) {
            h->backoff = 1;
            if (!keep) h->tmr_n = 0;
            h->timer_armed = 0;
        }
        __syncwarp();
        const uint32_t s = next_seq();
        const int64_t at = now + rto_of(d, *cc(k, 0));
        __syncwarp();
        if (lane == 0) {
            const uint32_t n = h->tmr_n;
            h->timer_armed = 1;
            h->armed_at = now;
            if (n < kTmrMax) {
                h->tmr_t[n] = at;
                h->tmr_seq[n] = s;
                h->tmr_n = n + 1;
            } else {
                atomicOr(d.status, CN_TX_STATUS_TIMER);
            }
        }
        __syncwarp();
    }
    __device__ void record(int64_t t, int k, uint32_t mid, uint32_t ci, int32_t path, int rtx, uint64_t seq) {
        const uint32_t n = hh->log_n;
        __syncwarp();
        if (lane == 0) {
            if (n < d.log_cap) {
                cn_tx_rec x;
                x.t = t;
                x.msg_id = mid;
                x.chunk = ci;
                x.path = path;
                x.is_rtx = rtx;
                x.msg_seq = seq;
                x.conn = static_cast<uint32_t>(H(k)->conn);
                x.dst = static_cast<uint32_t>(G(k)->dst);
                log[n] = x;
            } else {
                atomicOr(d.status, CN_TX_STATUS_LOG);
            }
            hh->log_n = n + 1;
        }
        __syncwarp();
    }
    // pending_bytes (:1005-1024): unchunked + queued fresh + pending rtx
    __device__ void maybe_send_rts(int k, int64_t now) {  // :1026-1053
        CHot* h = H(k);
        if (!d.rd || h->rts_outstanding) return;
        const int64_t pending = h->unchunked + h->txq_bytes + h->rtxq_bytes;
        if (pending <= 0 || h->credit > 0) return;
        const bool has_rtx = h->n_rtxq + h->n_stale > 0 || (d.ordered && G(k)->gq_n > 0);
        const uint32_t s = next_seq();
        __syncwarp();
        if (lane == 0) {
            h->rts_outstanding = 1;
            h->rts_acked = 0;
            h->rts_sent += 1;
            if (h->retry_n < kRetryMax) {
                const uint32_t q = (h->retry_head + h->retry_n) % kRetryMax;
                h->retry_t[q] = now + d.rto_min;
                h->retry_seq[q] = s;
                h->retry_n += 1;
            } else {
                atomicOr(d.status, CN_TX_STATUS_RETRY);
            }
        }
        __syncwarp();
        record(now, k, 0, 0xFFFFFFFFu, -1, has_rtx ? 1 : 0, static_cast<uint64_t>(pending));  // the RTS
    }
    __device__ uint32_t chunk_len(const TxMsg& m, uint32_t ci) const {
        const uint64_t off = static_cast<uint64_t>(ci) * d.cb;
        return m.len - off < d.cb ? static_cast<uint32_t>(m.len - off) : d.cb;
    }
    // on_select_path / on_tx_rtx_chunk of connection k's policy for chunk ci
    // (view_of, transport.cpp:496-512); prev_path >= 0 for a retransmission
    __device__ int select(int k, int prev_path, const TxMsg& m, uint32_t mid, uint32_t ci, int attempts) {
        CHot* h = H(k);
        WarpRng r{mt(k), nullptr, h->mt_idx};
        const int n = h->n_paths;
        int p;
        if (d.pol == CN_POLICY_DEFAULT) {  // DefaultPolicy (policy.hpp:80-91)
            p = select_tempered(r, static_cast<int>(d.lbp), n, d.lbp == 2 ? ecn_s(k) : rtt_s(k));
            if (prev_path >= 0 && d.avoid_prev && n > 1 && p == prev_path) p = (p + 1) % n;
        } else {
            cn_chunk_view v;
            v.src = G(k)->src;
            v.dst = G(k)->dst;
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
                case CN_POLICY_ROUND_ROBIN: p = pick<cn_policy::RoundRobinPolicy>(k, r, v); break;
                case CN_POLICY_SINGLE_PATH: p = pick<cn_policy::SinglePathPolicy>(k, r, v); break;
#ifdef CN_TX_USER_POLICY_HEADER
                case CN_POLICY_USER: p = pick<CnUserPolicy>(k, r, v); break;
#endif
                default: p = pick<cn_policy::OutOfRangePolicy>(k, r, v); break;
            }
        }
        wr(h->mt_idx, r.idx, lane);
        return p;
    }
    // select_path (lb.cpp:7-27), draws tempered on the fly from the raw state
    __device__ int select_tempered(WarpRng& r, int policy, int n, const double* s) {
        if (n == 1) return 0;
        if (policy == 0) return static_cast<int>(draw_below(r, static_cast<uint64_t>(n)));
        int a = static_cast<int>(draw_below(r, static_cast<uint64_t>(n)));
        int b = static_cast<int>(draw_below(r, static_cast<uint64_t>(n - 1)));
        if (b >= a) b++;
        return pick_p2(a, b, s);
    }
    __device__ uint64_t draw_u64(WarpRng& r) {
        if (r.idx >= kMtN) {
            warp_twist(r.mt, lane);
            r.idx = 0;
        }
        const uint64_t v = temper(r.mt[r.idx]);
        r.idx++;
        return v;
    }
    // libstdc++ uniform_int_distribution<uint64_t>(0, n-1) (uniform_int_dist.h:296-320)
    __device__ uint64_t draw_below(WarpRng& r, uint64_t n) {
        const uint64_t urange = n - 1;
        if (urange == ~0ull) return draw_u64(r);
        const uint64_t range = urange + 1;
        uint64_t u = draw_u64(r);
        uint64_t lo = u * range, hi = __umul64hi(u, range);
        if (lo < range) {
            const uint64_t threshold = (0 - range) % range;
            while (lo < threshold) {
                u = draw_u64(r);
                lo = u * range;
                hi = __umul64hi(u, range);
            }
        }
        return hi;
    }
    struct PolicyRng {  // the connection's RngStream, warp-collective draws
        Tx& x;
        WarpRng& r;
        __device__ uint64_t next_below(uint64_t k) { return x.draw_below(r, k); }
    };
    template <class P>
    __device__ int pick(int k, WarpRng& r, const cn_chunk_view& v) {
        cn_path_board b;
        b.rtt_ewma = rtt_s(k);
        b.ecn_ewma = ecn_s(k);
        b.n_paths = H(k)->n_paths;
        PolicyRng g{*this, r};
        uint64_t st[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) st[j] = H(k)->pol_state[j];
        int p = v.prev_path >= 0 ? P::rtx_path(v, b, g, st) : -1;
        if (p == -1) p = P::select_path(v, b, g, st);
        const bool bad = p < 0 || p >= b.n_paths || P::pacing(v) != 0;
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) H(k)->pol_state[j] = st[j];
            if (bad) atomicOr(d.status, CN_TX_STATUS_POLICY);  // the reference's logic_error (:283-290, :528-531)
        }
        __syncwarp();
        return bad ? 0 : p;
    }

    // send_chunk (transport.cpp:433-494) on the path the chunk is queued on
    __device__ void send_chunk(int64_t now, int k, uint32_t mid, const TxMsg& m, uint32_t ci, bool rtx,
                               uint64_t from_psn = 0) {
        CHot* h = H(k);
        const uint64_t e = m.chunk_base + ci;
        const int32_t path = d.c_path[e];
        const int64_t dl = now + rto_of(d, *cc(k, path)) * h->backoff;  // cur_rto(c, s) (:1078-1081)
        const int32_t att = d.c_att[e] + 1;
        const uint32_t len = chunk_len(m, ci);
        uint32_t start = 0;  // first packet sent (a go-back-N resend may start mid-chunk, :438-447)
        if (d.ordered) {
            TxConnG* g = G(k);
            if (att == 1) {
                const uint32_t npk = (len + d.max_pl - 1) / d.max_pl;
                __syncwarp();
                if (lane == 0) {
                    d.c_psn[e] = static_cast<int64_t>(g->next_psn);
                    g->next_psn += npk;
                    if (g->so_n < d.so_cap)
                        d.so_ref[static_cast<uint64_t>(h->conn) * d.so_cap + g->so_n] = (mid << 25) | ci;
                    else
                        atomicOr(d.status, CN_TX_STATUS_SENT_ORDER);
                    g->so_n += 1;
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
            if (d.rd) h->credit -= len - start * d.max_pl;  // the bytes actually sent (:486)
            if (rtx) h->chunk_rtx += 1;
            else h->chunks_sent += 1;
            hh->sends += 1;
        }
        __syncwarp();
        add_inflight(k, path, len);
        record(now, k, mid, ci, path | static_cast<int32_t>(start << 16), rtx || att > 1, m.seq);
        arm_rto(k, now);
    }
    // queue_rtx (transport.cpp:516-542); caller checked sent && !acked && !rtx_pending
    __device__ void queue_rtx(int64_t now, int k, const TxMsg& m, uint32_t mid, uint32_t ci) {
        CHot* h = H(k);
        const uint64_t e = m.chunk_base + ci;
        const int prev = d.c_path[e];  // attempts > 0: prev_path = ch.path (view_of, :509)
        const uint32_t len = chunk_len(m, ci);
        add_inflight(k, prev, -static_cast<int64_t>(len));
        __syncwarp();
        if (lane == 0) cc_on_loss(d, *cc(k, prev), now);
        __syncwarp();
        const int p = select(k, prev, m, mid, ci, d.c_att[e]);
        CN_UNIFORM(d, p);
        const uint32_t qs = h->q_seq + 1;
        __syncwarp();
        if (lane == 0) {
            h->q_seq = qs;
            d.c_fl[e] |= TF_RTXP;
            d.c_dup[e] = 0;
            d.c_path[e] = p;
            d.c_q[e] = kQRtx | qs;
            rtxq_n(k)[p] += 1;
            h->n_rtxq += 1;
            h->rtxq_bytes += len;
        }
        __syncwarp();
        ring_insert(k, p);
        schedule_pump(sub_engine(k, p), now);  // :541
    }
};

__device__ __forceinline__ TxMsg load_msg(const TxConnG* g, uint32_t mid) { return g->msgs[mid]; }
__device__ __forceinline__ void store_msg(TxConnG* g, uint32_t mid, const TxMsg& m, int lane) {
    __syncwarp();
    if (lane == 0) g->msgs[mid] = m;
    __syncwarp();
}

// Front of sub-connection (k, p)'s tx (rtx = false) or retransmission queue.
__device__ bool queue_front(const Tx& x, int k, int p, bool rtx, uint32_t* out_mid, uint32_t* out_ci) {
    const TxConnG* g = x.G(k);
    const CHot* h = x.H(k);
    uint32_t best = 0xFFFFFFFFu, bmid = 0, bci = 0;
    for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = h->live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            const TxMsg m = load_msg(g, mid);
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

// Index of connection k's stale retransmission-queue entry of path p with
// the smallest queue seq, or -1.
__device__ int stale_front(const Tx& x, int k, int p) {
    const TxConnG* g = x.G(k);
    const uint32_t n = x.H(k)->n_stale;
    uint32_t best = 0xFFFFFFFFu;
    int bi = -1;
    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
        const uint32_t j = k0 + x.lane;
        const uint32_t key = (j < n && g->stale_path[j] == p) ? g->stale_seq[j] : 0xFFFFFFFFu;
        const uint32_t mn = __reduce_min_sync(0xffffffffu, key);
        if (mn < best) {
            best = mn;
            bi = static_cast<int>(k0 + __ffs(__ballot_sync(0xffffffffu, key == mn)) - 1);
        }
    }
    return bi;
}

// gbn_rewind (transport.cpp:969-999): re-queue every unacked chunk whose
// packets reach the receiver's expected sequence, in first-send order;
// chunks wholly below it stay (or come back) in flight.  (Ordered mode:
// one path, one engine.)
__device__ void gbn_rewind(Tx& x, int k, int64_t now, uint64_t expected) {
    TxConnG* g = x.G(k);
    const uint32_t conn = static_cast<uint32_t>(x.H(k)->conn);
    if (expected == g->last_rewind_psn) return;  // duplicate gap report
    __syncwarp();
    if (x.lane == 0) cc_on_loss(x.d, *x.cc(k, 0), now);
    __syncwarp();
    if (x.lane == 0) {
        g->last_rewind_psn = expected;
        g->gq_head = 0;
        g->gq_n = 0;
    }
    __syncwarp();
    const uint64_t so = static_cast<uint64_t>(conn) * x.d.so_cap;
    const uint32_t n = g->so_n < x.d.so_cap ? g->so_n : x.d.so_cap;
    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
        const uint32_t j = k0 + x.lane;
        int act = 0;  // 1: back in flight, 2: re-queue, 3: already pending, re-queued
        uint32_t ref = 0, len = 0;
        uint64_t from = 0;
        uint64_t e = 0;
        if (j < n) {
            ref = x.d.so_ref[so + j];
            const uint32_t mid = ref >> 25, ci = ref & ((1u << 25) - 1);
            const TxMsg m = load_msg(g, mid);  // the slot's current message (:978-980)
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
                        act = (fl & TF_RTXP) ? 3 : 2;
                        from = base > expected ? base : expected;
                    }
                }
            }
        }
        for (unsigned b = __ballot_sync(0xffffffffu, act != 0); b; b &= b - 1) {  // in order
            const int jj = __ffs(b) - 1;
            const int aj = __shfl_sync(0xffffffffu, act, jj);
            const uint32_t lj = __shfl_sync(0xffffffffu, len, jj);
            const uint64_t ej = __shfl_sync(0xffffffffu, e, jj);
            if (aj == 1) {  // delivered but unacked: in flight again (:985-989)
                __syncwarp();
                if (x.lane == 0) x.d.c_fl[ej] &= ~TF_RTXP;
                __syncwarp();
                x.add_inflight(k, 0, lj);
            } else {
                if (aj == 2) {
                    __syncwarp();
                    if (x.lane == 0) x.d.c_fl[ej] |= TF_RTXP;
                    __syncwarp();
                    x.add_inflight(k, 0, -static_cast<int64_t>(lj));
                }
                const uint32_t rj = __shfl_sync(0xffffffffu, ref, jj);
                const uint64_t fj = __shfl_sync(0xffffffffu, from, jj);
                __syncwarp();
                if (x.lane == 0) {
                    x.d.c_dup[ej] = 0;
                    const uint32_t q = (g->gq_head + g->gq_n) % x.d.so_cap;
                    x.d.gq_ref[so + q] = rj;
                    x.d.gq_from[so + q] = fj;
                    g->gq_n += 1;
                }
                __syncwarp();
            }
        }
    }
    x.schedule_pump(x.sub_engine(k, 0), now);  // :998
}

// One DRR visit can send iff the sub has queued fresh chunks, a positive
// deficit after the top-up (:390-391), and an open gate.
__device__ __forceinline__ bool visit_can_send(const Tx& x, int k, int p) {
    if (x.txq_n(k)[p] == 0) return false;
    const int64_t q = x.d.quantum;
    int64_t def = x.defc(k)[p] + q;
    if (def > q) def = q;
    return def > 0 && x.can_send(k, p);
}

// egress (transport.cpp:329-431) of engine en
__device__ void egress(Tx& x, int en, int64_t now) {
    Eng& E = x.eng[en];
    uint32_t* rg = x.eng_ring(en);
    // retransmission pass (:333-369), exempt from the deficit
    for (int r = 0; r < E.ring_len; ++r) {
        const uint32_t ent = rg[r];
        const int k = static_cast<int>(ent >> 16), p = static_cast<int>(ent & 0xFFFF);
        CHot* h = x.H(k);
        if (!(h->n_rtxq || h->n_stale || (x.d.ordered && x.G(k)->gq_n))) continue;
        while (x.d.ordered && p == 0 && x.G(k)->gq_n && x.can_send(k, p)) {  // gbn_rtxq (:336-352)
            TxConnG* g = x.G(k);
            const uint64_t so = static_cast<uint64_t>(h->conn) * x.d.so_cap;
            const uint32_t ref = x.d.gq_ref[so + g->gq_head];
            const uint64_t from = x.d.gq_from[so + g->gq_head];
            __syncwarp();
            if (x.lane == 0) {
                g->gq_head = (g->gq_head + 1) % x.d.so_cap;
                g->gq_n -= 1;
            }
            __syncwarp();
            const uint32_t mid = ref >> 25, ci = ref & ((1u << 25) - 1);
            const TxMsg m = load_msg(g, mid);
            if (!m.live || ci >= m.nchunks) continue;
            const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
            if ((fl & TF_ACKED) || !(fl & TF_RTXP)) continue;
            x.send_chunk(now, k, mid, m, ci, true, from);
        }
        while ((x.rtxq_n(k)[p] > 0 || (h->n_stale && stale_front(x, k, p) >= 0)) && x.can_send(k, p)) {
            uint32_t mid = 0, ci = 0;
            const bool live = x.rtxq_n(k)[p] > 0 && queue_front(x, k, p, true, &mid, &ci);
            const uint32_t lseq = live ? (x.d.c_q[load_msg(x.G(k), mid).chunk_base + ci] & ~kQRtx) : 0xFFFFFFFFu;
            const int si = h->n_stale ? stale_front(x, k, p) : -1;
            TxConnG* g = x.G(k);
            if (si >= 0 && g->stale_seq[si] < lseq) {  // a stale entry at the front: popped, nothing sent
                __syncwarp();
                if (x.lane == 0) {
                    const uint32_t last = h->n_stale - 1;
                    g->stale_seq[si] = g->stale_seq[last];
                    g->stale_path[si] = g->stale_path[last];
                    g->stale_n = last;
                    h->n_stale = last;
                }
                __syncwarp();
                continue;
            }
            if (!live) break;
            const TxMsg m = load_msg(g, mid);
            const uint32_t len = x.chunk_len(m, ci);
            __syncwarp();
            if (x.lane == 0) {
                x.rtxq_n(k)[p] -= 1;
                h->n_rtxq -= 1;
                h->rtxq_bytes -= len;
            }
            __syncwarp();
            x.send_chunk(now, k, mid, m, ci, true);
        }
    }
    const uint32_t nr = static_cast<uint32_t>(E.ring_len);
    if (nr == 0) {  // :372-377
        if (x.d.rd)
            for (uint32_t k = 0; k < x.hh->n_conns; ++k) x.maybe_send_rts(static_cast<int>(k), now);
        return;
    }
    // deficit round robin over the ring (:378-424).  Runs of visits that
    // cannot send touch distinct subs once each (a queued sub tops its
    // deficit up, an idle one resets it) and are applied lane-parallel.
    const int64_t q = x.d.quantum;
    uint32_t idle = 0;
    while (idle < nr) {
        const uint32_t pos0 = static_cast<uint32_t>(E.ring_pos % nr);
        const uint32_t left = nr - idle;
        // first visit (within the next `left`) that can send
        uint32_t first = left;
        for (uint32_t j0 = 0; j0 < left && first == left; j0 += 32) {
            const uint32_t j = j0 + x.lane;
            bool ok = false;
            if (j < left) {
                uint32_t pos = pos0 + j;
                while (pos >= nr) pos -= nr;
                const uint32_t ent = rg[pos];
                ok = visit_can_send(x, static_cast<int>(ent >> 16), static_cast<int>(ent & 0xFFFF));
            }
            const unsigned b = __ballot_sync(0xffffffffu, ok);
            if (b) first = j0 + __ffs(b) - 1;
        }
        // the `first` idle visits before it
        __syncwarp();
        for (uint32_t j = x.lane; j < first; j += 32) {
            uint32_t pos = pos0 + j;
            while (pos >= nr) pos -= nr;
            const uint32_t ent = rg[pos];
            const int k = static_cast<int>(ent >> 16), p = static_cast<int>(ent & 0xFFFF);
            int64_t* dp = x.defc(k) + p;
            const int64_t def = *dp + q;
            *dp = x.txq_n(k)[p] ? (def > q ? q : def) : 0;
        }
        __syncwarp();
        CN_UNIFORM(x.d, first);
        if (first == left) {
            wr(E.ring_pos, E.ring_pos + left, x.lane);
            break;
        }
        idle += first;
        uint32_t pos = pos0 + first;
        while (pos >= nr) pos -= nr;
        const uint32_t ent = rg[pos];
        const int k = static_cast<int>(ent >> 16), p = static_cast<int>(ent & 0xFFFF);
        wr(E.ring_pos, E.ring_pos + first + 1, x.lane);
        CHot* h = x.H(k);
        int64_t def = x.defc(k)[p] + q;
        if (def > q) def = q;
        bool sent_any = false;
        while (x.txq_n(k)[p] > 0 && def > 0 && x.can_send(k, p)) {
            uint32_t mid, ci;
            if (!queue_front(x, k, p, false, &mid, &ci)) break;
            const TxMsg m = load_msg(x.G(k), mid);
            const uint32_t len = x.chunk_len(m, ci);
            __syncwarp();
            if (x.lane == 0) {
                x.txq_n(k)[p] -= 1;
                h->n_txq -= 1;
                h->txq_bytes -= len;
                x.eng[m.engine].committed_unsent -= len;  // the dispatch engine's (:416)
            }
            __syncwarp();
            def -= len;
            x.send_chunk(now, k, mid, m, ci, false);
            sent_any = true;
        }
        if (x.txq_n(k)[p] == 0) def = 0;
        wr(x.defc(k)[p], def, x.lane);
        idle = sent_any ? 0 : idle + 1;
    }
    if (x.d.rd)  // :427-430, in ring order
        for (uint32_t r = 0; r < nr; ++r) x.maybe_send_rts(static_cast<int>(rg[r] >> 16), now);
}

// commit_chunks (transport.cpp:244-310) of engine en: one chunk per message
// per turn of the factory rotation, window-stalled at 128 unacked chunks,
// bounded by the engine's commit_ahead bytes; each chunk is bound to a path
// and queued on that sub-connection (whose engine may be another one).
__device__ void commit_chunks(Tx& x, int en, int64_t now) {
    Eng& E = x.eng[en];
    uint32_t* fq = x.eng_fq(en);
    const uint32_t cap = x.d.fq_cap;
    uint32_t stalled = 0;
    while (E.fq_count > 0 && stalled < E.fq_count && E.committed_unsent < x.d.commit_ahead) {
        const uint32_t head = E.fq_head;
        const uint32_t ent = fq[head];
        const int k = static_cast<int>(ent >> 8);
        const uint32_t mid = ent & 0xFF;
        CHot* h = x.H(k);
        TxConnG* g = x.G(k);
        TxMsg m = load_msg(g, mid);
        __syncwarp();
        if (x.lane == 0) {
            E.fq_head = head + 1 == cap ? 0 : head + 1;
            E.fq_count -= 1;
        }
        __syncwarp();
        if (!m.live || m.chunked >= m.len) {
            m.in_factory = 0;
            store_msg(g, mid, m, x.lane);
            stalled = 0;
            continue;
        }
        if (m.nchunks - m.base >= static_cast<uint32_t>(kTxWindow)) {  // :258-262
            __syncwarp();
            if (x.lane == 0) {
                uint32_t t = E.fq_head + E.fq_count;
                if (t >= cap) t -= cap;
                fq[t] = ent;
                E.fq_count += 1;
            }
            __syncwarp();
            ++stalled;
            continue;
        }
        const uint64_t rem = m.len - m.chunked;
        const uint32_t sz = rem < x.d.cb ? static_cast<uint32_t>(rem) : x.d.cb;
        const uint32_t ci = m.nchunks;
        const int p = x.select(k, -1, m, mid, ci, 0);  // on_select_path (:281-287)
        CN_UNIFORM(x.d, p);
        const uint32_t qs = h->q_seq + 1;
        __syncwarp();
        if (x.lane == 0) {
            const uint64_t e = m.chunk_base + ci;
            h->q_seq = qs;
            x.d.c_path[e] = p;
            x.d.c_fl[e] = 0;
            x.d.c_att[e] = 0;
            x.d.c_dup[e] = 0;
            x.d.c_q[e] = qs;
            x.txq_n(k)[p] += 1;
            h->n_txq += 1;
            h->txq_bytes += sz;
            h->unchunked -= sz;
            E.gauge -= sz;
            E.committed_unsent += sz;
        }
        __syncwarp();
        x.ring_insert(k, p);
        const int se = x.sub_engine(k, p);
        if (se != en) x.schedule_pump(se, now);  // :301-302
        m.nchunks = ci + 1;
        m.chunked += sz;
        if (m.chunked < m.len) {
            __syncwarp();
            if (x.lane == 0) {
                uint32_t t = E.fq_head + E.fq_count;
                if (t >= cap) t -= cap;
                fq[t] = ent;
                E.fq_count += 1;
            }
            __syncwarp();
        } else {
            m.in_factory = 0;
        }
        store_msg(g, mid, m, x.lane);
        stalled = 0;
    }
}

__device__ void pump(Tx& x, int en, int64_t now) {  // transport.cpp:232-240
    for (;;) {
        commit_chunks(x, en, now);
        const uint64_t before = x.hh->sends;
        egress(x, en, now);
        if (x.hh->sends == before) break;
    }
}

__device__ void pump_all(Tx& x, int64_t now) {  // for (e : engines) pump(host, e)
    for (uint32_t e = 0; e < x.d.engines; ++e) pump(x, static_cast<int>(e), now);
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
__device__ void msg_finished(Tx& x, int k, uint32_t mid, uint32_t engine) {
    TxConnG* g = x.G(k);
    CHot* h = x.H(k);
    TxMsg m;
    memset(&m, 0, sizeof m);
    store_msg(g, mid, m, x.lane);
    __syncwarp();
    if (x.lane == 0) {
        h->live[mid >> 5] &= ~(1u << (mid & 31));
        g->free_ids[g->n_free] = static_cast<uint8_t>(mid);
        g->n_free += 1;
        x.eng[engine].inflight_msgs -= 1;
        h->msgs_completed += 1;
    }
    __syncwarp();
}

// release_chunk (:807-823) of a chunk the caller found sent && !acked.  A
// chunk awaiting retransmission leaves its queue (the reference's entry
// turns stale and is popped without effect).
__device__ void release(Tx& x, int k, int64_t now, const TxMsg& m, uint32_t ci, int64_t rtt, bool ecn) {
    CHot* h = x.H(k);
    const uint64_t e = m.chunk_base + ci;
    const uint32_t fl = x.d.c_fl[e];
    const int path = x.d.c_path[e];
    if (path < 0 || path >= h->n_paths) {  // unreachable: a chunk's path is bound at commit
        if (x.lane == 0) atomicOr(x.d.status, CN_TX_STATUS_INTERNAL);
        return;
    }
    const uint32_t len = x.chunk_len(m, ci);
    const uint32_t qv = x.d.c_q[e];
    __syncwarp();
    if (x.lane == 0) {
        x.d.c_fl[e] = (fl | TF_ACKED) & ~TF_RTXP;
        if (fl & TF_RTXP) {
            x.rtxq_n(k)[path] -= 1;
            h->n_rtxq -= 1;
            h->rtxq_bytes -= len;
            x.d.c_q[e] = 0;
            // its queue entry stays behind, stale, until egress pops it (:347-351)
            TxConnG* g = x.G(k);
            if (h->n_stale < kStaleMax) {
                g->stale_seq[h->n_stale] = qv & ~kQRtx;
                g->stale_path[h->n_stale] = static_cast<uint16_t>(path);
                h->n_stale += 1;
                g->stale_n = h->n_stale;
            } else {
                atomicOr(x.d.status, CN_TX_STATUS_STALE);
            }
        }
    }
    __syncwarp();
    if (!(fl & TF_RTXP)) x.add_inflight(k, path, -static_cast<int64_t>(len));
    __syncwarp();
    if (x.lane == 0) {
        cc_on_ack(x.d, *x.cc(k, path), now, len, rtt, ecn);
        if (rtt > 0) {  // board.record_rtt / record_ecn (:819-822)
            double* rs = x.rtt_s(k);
            double* es = x.ecn_s(k);
            rs[path] = __dadd_rn(rs[path], __ddiv_rn(__dsub_rn(static_cast<double>(rtt), rs[path]), 8.0));
            es[path] = __dadd_rn(es[path], __ddiv_rn(__dsub_rn(ecn ? 1.0 : 0.0, es[path]), 8.0));
        }
    }
    __syncwarp();
}

// Releases, in ascending order, every sent && !acked chunk of [lo, hi)
// that `pick` selects (CC sees the acks in the reference's order).
template <class Pick>
__device__ uint32_t release_range(Tx& x, int k, int64_t now, TxMsg& m, uint32_t lo, uint32_t hi, Pick pick) {
    uint32_t n_rel = 0;
    for (uint32_t w0 = lo; w0 < hi; w0 += 32) {
        const uint32_t ci = w0 + x.lane;
        bool want = false;
        if (ci < hi && pick(ci)) {
            const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
            want = (fl & TF_SENT) && !(fl & TF_ACKED);
        }
        for (unsigned b = __ballot_sync(0xffffffffu, want); b; b &= b - 1) {
            release(x, k, now, m, w0 + __ffs(b) - 1, 0, false);
            ++n_rel;
        }
    }
    m.acked += n_rel;
    return n_rel;
}

// handle_ack (:849-942)
__device__ void handle_ack(Tx& x, int k, int64_t now, const cn_ack_rec& a) {
    TxConnG* g = x.G(k);
    const uint32_t mid = (a.hdr >> 17) & 0x7F;
    TxMsg m = load_msg(g, mid);
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
            release(x, k, now, m, static_cast<uint32_t>(cause), rtt, (a.flags & CN_ACK_ECN_ECHO) != 0);
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
    newly += release_range(x, k, now, m, m.base, cend, [](uint32_t) { return true; });  // :898-904
    {  // selective bitmap relative to rcum (:905-914)
        const uint32_t send_ = rcum + 128 < nch ? rcum + 128 : nch;
        const uint64_t s0 = a.sack[0], s1 = a.sack[1];
        const uint32_t rc = rcum;
        newly += release_range(x, k, now, m, rcum < send_ ? rcum : send_, send_, [=](uint32_t ci) {
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
                __syncwarp();
                if (x.lane == 0) x.H(k)->fast_rtx += 1;
                __syncwarp();
                x.queue_rtx(now, k, m, mid, w0 + __ffs(b) - 1);
            }
        }
    }
    m.base = advance_base(x, m);  // :931
    CN_UNIFORM(x.d, m.base);
    CN_UNIFORM(x.d, m.acked);
    CN_UNIFORM(x.d, newly);
    CN_UNIFORM(x.d, rcum);
    const bool done = m.chunked >= m.len && nch > 0 && m.acked == nch && !m.in_factory;
    store_msg(g, mid, m, x.lane);
    if (done) msg_finished(x, k, mid, m.engine);  // :932-934
    if (newly > 0) x.rearm(k, now);                // :936-940
    pump_all(x, now);                              // :941
}

// handle_nack (:944-965)
__device__ void handle_nack(Tx& x, int k, int64_t now, const cn_ack_rec& a) {
    if (x.d.ordered) {  // :950-954
        gbn_rewind(x, k, now, a.sack[0]);
        pump_all(x, now);
        return;
    }
    const uint32_t mid = (a.hdr >> 17) & 0x7F;
    const TxMsg m = load_msg(x.G(k), mid);
    if (!m.live || m.seq != a.msg_seq) return;
    const uint8_t rel = static_cast<uint8_t>(a.cum_csn - static_cast<uint8_t>(m.base & 0xFF));
    if (rel >= kTxWindow || m.base + rel >= m.nchunks) return;
    const uint32_t ci = m.base + rel;
    const uint32_t fl = x.d.c_fl[m.chunk_base + ci];
    if ((fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP))) x.queue_rtx(now, k, m, mid, ci);
    pump_all(x, now);
}

// rto_fire (:1094-1169) of connection k's live timer, firing at `now`
__device__ void rto_fire(Tx& x, int k, int64_t now) {
    CHot* h = x.H(k);
    TxConnG* g = x.G(k);
    __syncwarp();
    if (x.lane == 0) {
        h->timer_armed = 0;
        h->tmr_n = 0;  // events armed at the same instant are superseded now
    }
    __syncwarp();
    // scan: oldest deadline and the number of expired chunks
    int64_t best = 0;
    bool have = false;
    uint32_t n_exp = 0;
    for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = h->live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            const TxMsg m = load_msg(g, mid);
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
    CN_UNIFORM(x.d, n_exp);
    CN_UNIFORM(x.d, best);
    if (!have) return;  // :1131 nothing outstanding
    if (n_exp == 0) {   // :1132-1140 re-arm for the earliest deadline
        x.add_timer(k, now, best);
        return;
    }
    __syncwarp();
    if (x.lane == 0) {
        h->rtos += 1;
        h->backoff = h->backoff * 2 < kBackoffCap ? h->backoff * 2 : kBackoffCap;
    }
    __syncwarp();
    if (x.d.ordered) {  // :1144-1148: rewind from the oldest outstanding chunk's first packet
        __syncwarp();
        if (x.lane == 0) cc_on_rto(x.d, *x.cc(k, 0), now);
        __syncwarp();
        uint64_t psn0 = 0;
        bool found = false;
        for (uint32_t q = 0; q < 4 && !found; ++q)
            for (uint32_t lb = h->live[q]; lb && !found; lb &= lb - 1) {
                const uint32_t mid = q * 32 + __ffs(lb) - 1;
                const TxMsg m = load_msg(g, mid);
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
                        psn0 = static_cast<uint64_t>(x.d.c_psn[m.chunk_base + w0 + __ffs(b) - 1]);
                        found = true;
                    }
                }
            }
        __syncwarp();
        if (x.lane == 0) g->last_rewind_psn = ~0ull;
        __syncwarp();
        gbn_rewind(x, k, now, psn0);
    } else {
        // every overdue chunk lost in one shot, in scan order; on_rto once per
        // distinct CC before its first loss (:1149-1162)
        uint64_t punished[4] = {0, 0, 0, 0};  // per-path CCs, up to 256 paths (bit per path)
        bool punished_g = false;
        for (uint32_t q = 0; q < 4; ++q)
            for (uint32_t lb = h->live[q]; lb; lb &= lb - 1) {
                const uint32_t mid = q * 32 + __ffs(lb) - 1;
                const TxMsg m = load_msg(g, mid);
                for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
                    const uint32_t ci = w0 + x.lane;
                    bool ex = false;
                    if (ci < m.nchunks) {
                        const uint64_t e = m.chunk_base + ci;
                        const uint32_t fl = x.d.c_fl[e];
                        ex = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP)) && x.d.c_dead[e] <= now;
                    }
                    for (unsigned b = __ballot_sync(0xffffffffu, ex); b; b &= b - 1) {
                        const uint32_t cj = w0 + __ffs(b) - 1;
                        const int p = x.d.c_path[m.chunk_base + cj];
                        bool first;
                        if (x.d.per_path) {
                            const uint64_t bit = 1ull << (p & 63);
                            first = p < 256 ? !(punished[p >> 6] & bit) : true;
                            if (p < 256) punished[p >> 6] |= bit;
                            if (p >= 256 && x.lane == 0) atomicOr(x.d.status, CN_TX_STATUS_CAPACITY);
                        } else {
                            first = !punished_g;
                            punished_g = true;
                        }
                        if (first) {
                            __syncwarp();
                            if (x.lane == 0) cc_on_rto(x.d, *x.cc(k, p), now);
                            __syncwarp();
                        }
                        x.queue_rtx(now, k, m, mid, cj);
                    }
                }
            }
    }
    x.maybe_send_rts(k, now);  // :1166 (receiver-driven only)
    x.arm_rto(k, now);         // :1167
    pump_all(x, now);          // :1168
}

// conn_to (:84-137): the connection opens at its first send_message; its
// home engine is the least-loaded one at that moment (ties: lowest id)
__device__ void open_conn(Tx& x, int k) {
    int home = 0;
    for (uint32_t e = 1; e < x.d.engines; ++e)
        if (x.eng[e].gauge < x.eng[home].gauge) home = static_cast<int>(e);
    __syncwarp();
    if (x.lane == 0) {
        x.H(k)->home = home;
        x.H(k)->opened = 1;
    }
    __syncwarp();
}

// send_message (:144-196) + dispatch (:198-218)
__device__ void submit(Tx& x, int k, int64_t now, const cn_tx_submit& s) {
    CHot* h = x.H(k);
    if (!h->opened) open_conn(x, k);
    TxConnG* g = x.G(k);
    if (s.len == 0 || g->n_free == 0) {  // len 0 throws in the reference; flagged here
        __syncwarp();
        if (x.lane == 0) {
            g->backpressured += 1;
            if (s.len == 0) atomicOr(x.d.status, CN_TX_STATUS_EMPTY_MSG);
        }
        __syncwarp();
        return;
    }
    const uint32_t mid = g->free_ids[g->n_free - 1];
    const uint64_t seq = g->next_seq;
    wr(g->next_seq, seq + 1, x.lane);
    int pick = h->home;  // dispatch (:198-209)
    if (x.d.conn_split) {
        pick = 0;
        for (uint32_t e = 1; e < x.d.engines; ++e)
            if (x.eng[e].gauge < x.eng[pick].gauge) pick = static_cast<int>(e);
    }
    Eng& E = x.eng[pick];
    if (static_cast<uint32_t>(E.inflight_msgs) >= x.d.max_inflight) {
        wr(g->backpressured, g->backpressured + 1, x.lane);
        return;
    }
    // the connection's share of the chunk pool is a ring: a message takes
    // nc contiguous entries (the ring's end is skipped when too short) and
    // frees them when it finishes (msg_finished, :831-847); the tail is the
    // oldest live message
    const uint64_t nc = (s.len + x.d.cb - 1) / x.d.cb;
    const uint64_t pc = x.d.conn_pool;
    const uint64_t hd = g->p_head;
    uint64_t tl = hd;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if ((h->live[q] >> x.lane) & 1u) {
            const uint64_t ps = g->p_start[q * 32 + x.lane];
            tl = ps < tl ? ps : tl;
        }
    for (int o = 16; o; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, tl, o);
        tl = y < tl ? y : tl;
    }
    const uint64_t pp = hd % pc;
    const uint64_t start = pp + nc > pc ? hd + (pc - pp) : hd;
    if (nc > pc || start + nc - tl > pc) {
        if (x.lane == 0) atomicOr(x.d.status, CN_TX_STATUS_CAPACITY);
        return;
    }
    const uint64_t base = static_cast<uint64_t>(h->conn) * pc + start % pc;
    for (uint64_t j = x.lane; j < nc; j += 32) {  // a reused range starts unsent
        x.d.c_fl[base + j] = 0;
        x.d.c_q[base + j] = 0;
    }
    TxMsg m;
    memset(&m, 0, sizeof m);
    m.seq = seq;
    m.tag = s.tag;
    m.len = s.len;
    m.chunk_base = base;
    m.live = 0;  // live after dispatch (:163)
    m.in_factory = 1;
    m.engine = static_cast<uint32_t>(pick);
    store_msg(g, mid, m, x.lane);
    __syncwarp();
    if (x.lane == 0) {
        g->p_head = start + nc;
        g->p_start[mid] = start;
        E.inflight_msgs += 1;
        E.dispatched += 1;
        E.gauge += static_cast<int64_t>(s.len);
        uint32_t t = E.fq_head + E.fq_count;
        if (t >= x.d.fq_cap) t -= x.d.fq_cap;
        x.eng_fq(pick)[t] = (static_cast<uint32_t>(k) << 8) | mid;
        E.fq_count += 1;
    }
    __syncwarp();
    // dispatch's RTS check (:216) runs before the message is live, so its
    // bytes are not pending yet
    x.maybe_send_rts(k, now);
    m.live = 1;
    store_msg(g, mid, m, x.lane);
    __syncwarp();
    if (x.lane == 0) {
        h->live[mid >> 5] |= 1u << (mid & 31);
        g->n_free -= 1;
        g->msgs_sent += 1;
        h->unchunked += static_cast<int64_t>(s.len);
    }
    __syncwarp();
    pump(x, pick, now);  // :166
}

// handle_credit (:1061-1074): bank the grant up to the cap, clear the
// outstanding RTS, pump every engine, and ask again if needed
__device__ void handle_credit(Tx& x, int k, int64_t now, uint64_t bytes) {
    CHot* h = x.H(k);
    const int64_t cap = x.d.credit_cap;
    int64_t cr = h->credit;
    if (cr < cap) {
        const int64_t v = cr + static_cast<int64_t>(bytes);
        cr = v < cap ? v : cap;
    }
    __syncwarp();
    if (x.lane == 0) {
        h->credit = cr;
        h->rts_outstanding = 0;
    }
    __syncwarp();
    pump_all(x, now);
    x.maybe_send_rts(k, now);
}

// an RTS retry event (:1046-1052)
__device__ void rts_retry(Tx& x, int k, int64_t now) {
    CHot* h = x.H(k);
    const bool again = h->rts_outstanding && !h->rts_acked;
    __syncwarp();
    if (x.lane == 0) {
        h->retry_head = (h->retry_head + 1) % kRetryMax;
        h->retry_n -= 1;
        if (again) h->rts_outstanding = 0;
    }
    __syncwarp();
    if (again) x.maybe_send_rts(k, now);
}

// Fires the events the run itself scheduled -- RTO timers, deferred pumps
// and RTS retries -- that precede an input event at time t (inclusive =
// false) or the horizon t (inclusive = true), in the event queue's
// (time, seq) order: input events were all queued first, so they win ties.
__device__ void run_deferred(Tx& x, int64_t t, bool inclusive) {
    const uint32_t nk = x.hh->n_conns, ne = x.d.engines;
    for (;;) {
        // lane-parallel candidates: connection timers / retries, engine pumps
        long long bt = LLONG_MAX;
        uint32_t bs = 0xFFFFFFFFu, bid = 0xFFFFFFFFu;  // id: kind << 24 | index
        auto consider = [&](int64_t at, uint32_t seq, uint32_t id) {
            if (inclusive ? at > t : at >= t) return;
            if (at < bt || (at == bt && seq < bs)) {
                bt = at;
                bs = seq;
                bid = id;
            }
        };
        for (uint32_t k = x.lane; k < nk; k += 32) {
            const CHot* h = x.H(static_cast<int>(k));
            if (h->timer_armed)
                for (uint32_t i = 0; i < h->tmr_n; ++i) consider(h->tmr_t[i], h->tmr_seq[i], (0u << 24) | k);
            if (h->retry_n) consider(h->retry_t[h->retry_head], h->retry_seq[h->retry_head], (2u << 24) | k);
        }
        for (uint32_t e = x.lane; e < ne; e += 32)
            if (x.eng[e].pump_pending) consider(x.eng[e].pump_at, x.eng[e].pump_seq, (1u << 24) | e);
        for (int o = 16; o > 0; o >>= 1) {
            const long long ot = __shfl_xor_sync(0xffffffffu, bt, o);
            const uint32_t os = __shfl_xor_sync(0xffffffffu, bs, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bid, o);
            if (ot < bt || (ot == bt && os < bs)) {
                bt = ot;
                bs = os;
                bid = oi;
            }
        }
        CN_UNIFORM(x.d, bid);
        CN_UNIFORM(x.d, bt);
        if (bid == 0xFFFFFFFFu) return;
        const uint32_t kind = bid >> 24, idx = bid & 0xFFFFFF;
        if (kind == 0) {
            rto_fire(x, static_cast<int>(idx), bt);
        } else if (kind == 1) {
            wr(x.eng[idx].pump_pending, 0u, x.lane);
            pump(x, static_cast<int>(idx), bt);
        } else {
            rts_retry(x, static_cast<int>(idx), bt);
        }
    }
}

// Shared memory per warp: the host blob, then one blob per connection of
// the host (laid out by cn_tx_create).
__global__ void __launch_bounds__(128, 1) k_tx_run(const TxDev* __restrict__ dp, uint32_t warps_per_block,
                                                   uint32_t smem_per_warp, const uint32_t* __restrict__ ev_off,
                                                   const uint64_t* __restrict__ events,
                                                   const cn_tx_submit* __restrict__ submits,
                                                   const cn_ack_rec* __restrict__ acks, int64_t end_time,
                                                   cn_tx_rec* __restrict__ log, cn_tx_stats* __restrict__ stats) {
    extern __shared__ __align__(16) uint8_t smem[];
    const TxDev& d = *dp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t host = blockIdx.x * warps_per_block + w;
    if (host >= d.n_hosts) return;
    uint8_t* base = smem + static_cast<size_t>(w) * smem_per_warp;
    const uint32_t nk = d.host_nconns[host];
    // load the host's blobs (16-byte words)
    {
        const uint4* src = reinterpret_cast<const uint4*>(d.host_blob + static_cast<size_t>(host) * d.host_bytes);
        uint4* dst = reinterpret_cast<uint4*>(base);
        for (uint32_t i = lane; i < d.host_bytes / 16; i += 32) dst[i] = src[i];
        for (uint32_t k = 0; k < nk; ++k) {
            const uint32_t c = d.host_conns[static_cast<size_t>(host) * d.mcph + k];
            const uint4* s2 = reinterpret_cast<const uint4*>(d.conn_blob + static_cast<size_t>(c) * d.conn_bytes);
            uint4* d2 = reinterpret_cast<uint4*>(base + d.host_bytes + static_cast<size_t>(k) * d.conn_bytes);
            for (uint32_t i = lane; i < d.conn_bytes / 16; i += 32) d2[i] = s2[i];
        }
    }
    __syncwarp();
    Tx x{d,
         host,
         lane,
         reinterpret_cast<HostHdr*>(base),
         reinterpret_cast<Eng*>(base + sizeof(HostHdr)),
         base + d.host_bytes,
         d.ring + static_cast<size_t>(host) * d.engines * d.ring_cap,
         d.fq + static_cast<size_t>(host) * d.engines * d.fq_cap,
         log + static_cast<size_t>(host) * d.log_cap};
    for (uint32_t j = ev_off[host]; j < ev_off[host + 1]; ++j) {
        const uint64_t ev = events[j];
        const uint32_t type = static_cast<uint32_t>(ev >> 62);
        const uint32_t conn = static_cast<uint32_t>((ev >> 40) & 0x3FFFFF);
        const uint64_t idx = ev & ((1ull << 40) - 1);
        const int64_t t = type == 0 ? submits[idx].t : acks[idx].aux;
        CN_UNIFORM(d, ev);
        run_deferred(x, t, false);
        if (conn >= d.n_conns) {
            if (lane == 0) atomicOr(d.status, CN_TX_STATUS_INTERNAL);
            continue;
        }
        const int k = static_cast<int>(d.conn_local[conn]);
        if (type == 0) {
            submit(x, k, t, submits[idx]);
            continue;
        }
        if (!x.H(k)->opened) continue;  // conn_by_dst lookup fails: dropped (:851-852)
        const cn_ack_rec a = acks[idx];
        if (a.flags & CN_ACK_NACK) {
            handle_nack(x, k, t, a);
        } else if (a.flags & CN_ACK_CREDIT) {
            handle_credit(x, k, t, a.sack[0]);
        } else if (a.flags & CN_ACK_RTS_ACK) {
            wr(x.H(k)->rts_acked, 1u, lane);  // handle_packet rts_ack (:587-592)
        } else {
            handle_ack(x, k, t, a);
        }
    }
    run_deferred(x, end_time, true);
    __syncwarp();
    // stats and persist
    for (uint32_t k = 0; k < nk; ++k) {
        const CHot* h = x.H(static_cast<int>(k));
        if (lane == 0) {
            const TxConnG* g = d.conns + h->conn;
            const Cc& c0 = *x.cc(static_cast<int>(k), 0);
            cn_tx_stats st;
            st.chunks_sent = h->chunks_sent;
            st.chunk_rtx = h->chunk_rtx;
            st.fast_rtx = h->fast_rtx;
            st.rtos = h->rtos;
            st.msgs_sent = g->msgs_sent;
            st.msgs_completed = h->msgs_completed;
            st.backpressured = g->backpressured;
            st.n_log = x.hh->log_n;
            st.srtt = c0.srtt;
            st.rttvar = c0.rttvar;
            st.backoff = h->backoff;
            int32_t live = 0;
            for (int q = 0; q < 4; ++q) live += __popc(h->live[q]);
            st.live_msgs = live;
            st.cwnd_bytes = c0.cwnd;
            st.inflight = h->total_inflight;
            st.cwnd_pkts = c0.w;
            st.rts_sent = h->rts_sent;
            st.decreases = c0.decreases;
            stats[h->conn] = st;
        }
    }
    {
        uint4* dst = reinterpret_cast<uint4*>(d.host_blob + static_cast<size_t>(host) * d.host_bytes);
        const uint4* src = reinterpret_cast<const uint4*>(base);
        for (uint32_t i = lane; i < d.host_bytes / 16; i += 32) dst[i] = src[i];
        for (uint32_t k = 0; k < nk; ++k) {
            const uint32_t c = d.host_conns[static_cast<size_t>(host) * d.mcph + k];
            uint4* d2 = reinterpret_cast<uint4*>(d.conn_blob + static_cast<size_t>(c) * d.conn_bytes);
            const uint4* s2 = reinterpret_cast<const uint4*>(base + d.host_bytes + static_cast<size_t>(k) * d.conn_bytes);
            for (uint32_t i = lane; i < d.conn_bytes / 16; i += 32) d2[i] = s2[i];
        }
    }
}

// Initialises every connection's persistent blob, global state and
// RngStream("transport.conn", stream_index0 + c) (std::mt19937_64 seeding);
// one block per connection.
__global__ void k_tx_init(TxDev d, uint32_t c0, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                          const int32_t* __restrict__ np, uint64_t name_hash, uint64_t seed, int64_t index0) {
    const uint32_t c = c0 + blockIdx.x;
    if (c >= d.n_conns) return;
    TxConnG* g = d.conns + c;
    uint8_t* b = d.conn_blob + static_cast<size_t>(c) * d.conn_bytes;
    for (uint32_t i = threadIdx.x; i < sizeof(TxConnG) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(g)[i] = 0;
    for (uint32_t i = threadIdx.x; i < d.conn_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b)[i] = 0;
    __syncthreads();
    double* rtt = reinterpret_cast<double*>(b + d.o_rtt);
    for (uint32_t p = threadIdx.x; p < d.max_paths; p += blockDim.x) rtt[p] = d.base_rtt;  // lb.hpp:17-18
    Cc* cc = reinterpret_cast<Cc*>(b + d.o_cc);
    for (uint32_t i = threadIdx.x; i < d.n_cc; i += blockDim.x) {  // make_cc (cc.cpp:160-167)
        Cc& x = cc[i];
        x.w = d.init_cwnd;
        x.ssthresh = __longlong_as_double(0x7ff0000000000000ll);
        x.epoch_start = -1;
        x.last_decrease = kNeverDecreased;
        x.cwnd = cc_cwnd(d, x);
    }
    if (threadIdx.x == 0) {
        g->next_seq = 1;
        g->last_rewind_psn = ~0ull;
        g->src = src[c];
        g->dst = dst[c];
        g->conn_id = static_cast<int32_t>(c & 0xFF);
        for (int i = 0; i < 128; ++i) g->free_ids[i] = static_cast<uint8_t>(127 - i);  // :127-129
        g->n_free = 128;
        CHot* h = reinterpret_cast<CHot*>(b);
        h->backoff = 1;
        h->n_paths = np[c];
        h->conn = static_cast<int32_t>(c);
        h->credit = d.initial_credit;  // conn_to (:131-133)
        h->mt_idx = kMtN;
        uint64_t* mt = reinterpret_cast<uint64_t*>(b + d.o_mt);
        uint64_t prev = splitmix64_d(splitmix64_d(seed ^ name_hash) + static_cast<uint64_t>(index0 + c));
        mt[0] = prev;
        for (int i = 1; i < kMtN; ++i) {
            prev = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
            mt[i] = prev;
        }
    }
}

__global__ void k_libm_eval(int mode, const double* __restrict__ in, double* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = mode == 0 ? libm_cbrt(in[i]) : libm_pow3(in[i]);
}

}  // namespace cnb

using namespace cnb;

struct cn_tx {
    TxDev d;
    TxDev* d_dev = nullptr;  // device copy read by k_tx_run
    uint32_t max_conns = 0;
    std::vector<uint32_t> nconns;   // per host
    std::vector<uint32_t> host_of;  // per connection
    std::vector<uint32_t> loc;      // per connection
    std::map<int32_t, uint32_t> hid;  // src id -> host
    uint32_t max_k = 1;
    uint64_t seed = 0;
    int64_t stream_index0 = 0;
    int32_t *d_src = nullptr, *d_dst = nullptr, *d_np = nullptr;  // staging for k_tx_init
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
    c->engines = 1;
}

static uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Allocates an engine for up to max_conns connections, at most mcph per host.
static int tx_alloc(const cn_tx_config* cfg, uint32_t max_conns, uint32_t mcph, cn_tx** out) {
    if (!cfg || !out || max_conns == 0 || max_conns > (1u << 22) || cfg->chunk_bytes == 0 || cfg->rto_min <= 0 ||
        cfg->max_paths == 0 || cfg->max_paths > 1024 || cfg->lb_policy < 0 || cfg->lb_policy > 2 ||
        !(cfg->policy >= CN_POLICY_DEFAULT && cfg->policy <= CN_POLICY_TEST_OUT_OF_RANGE
#ifdef CN_TX_USER_POLICY_HEADER
          || cfg->policy == CN_POLICY_USER
#endif
          ) ||
        (cfg->cc_algo != CN_CC_NONE && cfg->cc_algo != CN_CC_SWIFT && cfg->cc_algo != CN_CC_CUBIC) ||
        cfg->drr_quantum == 0 || cfg->mss <= 0 || !(cfg->init_cwnd_pkts > 0) || cfg->cap_bytes < 0 ||
        cfg->engines < 1 || cfg->engines > kMaxEngines || cfg->cc_scope < 0 || cfg->cc_scope > 1) {
        set_error("cn_tx_create: bad config (rto_min resolved > 0, max_paths <= 1024, engines 1..16, "
                  "cc none / cubic / swift, scope global / per_path)");
        return CN_E_INVALID;
    }
    if (cfg->ordered && (cfg->max_paths != 1 || cfg->engines != 1 || cfg->conn_split)) {
        set_error("cn_tx_create: ordered delivery needs a single path and a single engine (transport.cpp:21-26)");
        return CN_E_LOGIC;
    }
    if (cfg->cc_scope == 1 && cfg->max_paths > 256) {
        set_error("cn_tx_create: per-path CC scope supports up to 256 paths");
        return CN_E_UNSUPPORTED;
    }
    if (mcph > 255) {
        set_error("cn_tx_create: more than 255 connections from one host");
        return CN_E_UNSUPPORTED;
    }
    *out = nullptr;
    cn_tx* t = new (std::nothrow) cn_tx();
    if (!t) return CN_E_CAPACITY;
    memset(&t->d, 0, sizeof t->d);
    TxDev& d = t->d;
    t->max_conns = max_conns;
    d.n_conns = 0;
    d.n_hosts = 0;
    d.max_paths = cfg->max_paths;
    d.mcph = mcph;
    d.engines = static_cast<uint32_t>(cfg->engines);
    d.conn_split = cfg->conn_split ? 1 : 0;
    d.per_path = cfg->cc_scope == 1 ? 1 : 0;
    d.n_cc = d.per_path ? cfg->max_paths : 1;
    d.cb = cfg->chunk_bytes;
    d.max_pl = cfg->max_payload ? cfg->max_payload : CN_MAX_PAYLOAD;
    d.dupack = cfg->dupack_threshold;
    d.avoid_prev = cfg->rtx_avoid_prev_path ? 1 : 0;
    d.lbp = static_cast<uint32_t>(cfg->lb_policy);
    d.max_inflight = cfg->max_inflight_msgs;
    d.log_cap = cfg->log_cap;
    d.cc_algo = cfg->cc_algo;
    d.ecn_as_loss = cfg->ecn_as_loss ? 1 : 0;
    d.quantum = cfg->drr_quantum;
    d.rto_min = cfg->rto_min;
    d.rto_max = cfg->rto_max > 0 ? cfg->rto_max : 64 * cfg->rto_min;  // transport.cpp:36
    d.commit_ahead = cfg->commit_ahead;
    d.swift_target = cfg->swift_target_ns;
    d.mss = cfg->mss;
    d.cap_bytes = cfg->cap_bytes;
    d.init_cwnd = cfg->init_cwnd_pkts;
    d.base_rtt = cfg->base_rtt_ns;
    d.rd = cfg->receiver_driven ? 1 : 0;
    d.ordered = cfg->ordered ? 1 : 0;
    d.pol = cfg->policy;
    d.so_cap = cfg->ordered ? (cfg->sent_order_cap ? cfg->sent_order_cap : 1u << 16) : 1;
    d.credit_cap = static_cast<int64_t>(cfg->credit_bank_quanta) * cfg->credit_quantum;
    d.initial_credit = cfg->initial_credit;
    // cap_pkts_ (cc.cpp:41-42, :111-113)
    d.cap_pkts = cfg->cap_bytes > 0 ? static_cast<double>(cfg->cap_bytes) / static_cast<double>(cfg->mss)
                                    : __builtin_huge_val();
    d.pool_cap = cfg->chunk_pool;
    d.conn_pool = cfg->chunk_pool / max_conns;
    // blob layouts
    d.host_bytes = align16(static_cast<uint32_t>(sizeof(HostHdr) + sizeof(Eng) * d.engines));
    const uint32_t mp = cfg->max_paths;
    uint32_t o = align16(sizeof(CHot));
    d.o_mt = o;
    o += kMtN * 8;
    d.o_rtt = o;
    o += 8 * mp;
    d.o_ecn = o;
    o += 8 * mp;
    d.o_infl = o;
    o += 8 * mp;
    d.o_def = o;
    o += 8 * mp;
    d.o_cc = o;
    o += static_cast<uint32_t>(sizeof(Cc)) * d.n_cc;
    d.o_txq = o;
    o += 4 * mp;
    d.o_rtxq = o;
    o += 4 * mp;
    d.o_inr = o;
    o += mp;
    d.conn_bytes = align16(o);
    if (mcph == 0) {  // as many connections per host as one SM's shared memory holds (<= 16)
        const size_t fit = (227 * 1024 - d.host_bytes) / d.conn_bytes;
        mcph = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(16, fit)));
        d.mcph = mcph;
    }
    d.ring_cap = mcph * cfg->max_paths;
    d.fq_cap = mcph * 128;
    const size_t per_warp = d.host_bytes + static_cast<size_t>(mcph) * d.conn_bytes;
    if (per_warp > 227 * 1024) {
        delete t;
        set_error("cn_tx_create: a host's state (" + std::to_string(per_warp) +
                  " B: connections x paths) exceeds one SM's shared memory");
        return CN_E_UNSUPPORTED;
    }
    t->seed = cfg->seed;
    t->stream_index0 = cfg->stream_index0;
    const uint64_t pool = cfg->chunk_pool;
    const uint32_t mh = max_conns;  // at most one host per connection
    bool ok = cudaMalloc(&d.conns, sizeof(TxConnG) * max_conns) == cudaSuccess &&
              cudaMalloc(&d.host_blob, static_cast<size_t>(d.host_bytes) * mh) == cudaSuccess &&
              cudaMalloc(&d.conn_blob, static_cast<size_t>(d.conn_bytes) * max_conns) == cudaSuccess &&
              cudaMalloc(&d.host_conns, 4ull * mh * mcph) == cudaSuccess &&
              cudaMalloc(&d.host_nconns, 4ull * mh) == cudaSuccess &&
              cudaMalloc(&d.conn_local, 4ull * max_conns) == cudaSuccess &&
              cudaMalloc(&d.ring, 4ull * mh * d.engines * d.ring_cap) == cudaSuccess &&
              cudaMalloc(&d.fq, 4ull * mh * d.engines * d.fq_cap) == cudaSuccess &&
              cudaMalloc(&d.c_path, pool * 4) == cudaSuccess && cudaMalloc(&d.c_txt, pool * 8) == cudaSuccess &&
              cudaMalloc(&d.c_dead, pool * 8) == cudaSuccess && cudaMalloc(&d.c_att, pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_fl, pool * 4) == cudaSuccess && cudaMalloc(&d.c_dup, pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_q, pool * 4) == cudaSuccess && cudaMalloc(&d.c_psn, pool * 8) == cudaSuccess &&
              cudaMalloc(&d.so_ref, static_cast<uint64_t>(max_conns) * d.so_cap * 4) == cudaSuccess &&
              cudaMalloc(&d.gq_ref, static_cast<uint64_t>(max_conns) * d.so_cap * 4) == cudaSuccess &&
              cudaMalloc(&d.gq_from, static_cast<uint64_t>(max_conns) * d.so_cap * 8) == cudaSuccess &&
              cudaMalloc(&d.status, 4) == cudaSuccess && cudaMalloc(&t->d_dev, sizeof(TxDev)) == cudaSuccess &&
              cudaMalloc(&t->d_src, 4ull * max_conns) == cudaSuccess &&
              cudaMalloc(&t->d_dst, 4ull * max_conns) == cudaSuccess &&
              cudaMalloc(&t->d_np, 4ull * max_conns) == cudaSuccess;
    if (!ok) {
        set_error("cn_tx_create: out of device memory");
        cn_tx_destroy(t);
        return CN_E_CAPACITY;
    }
    cudaMemset(d.status, 0, 4);
    cudaMemset(d.c_q, 0, pool * 4);
    cudaMemset(d.c_fl, 0, pool * 4);
    cudaMemset(d.c_path, 0, pool * 4);
    cudaMemset(d.host_nconns, 0, 4ull * mh);
    cudaMemset(d.host_blob, 0, static_cast<size_t>(d.host_bytes) * mh);
    cudaFuncSetAttribute(k_tx_run, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    *out = t;
    return CN_OK;
}

// conn_to's bookkeeping on the host side: connection index = open order,
// its host = the engine-sharing unit of its src
static int tx_register(cn_tx* t, int32_t src, int32_t dst, int32_t n_paths, uint32_t* out_c) {
    TxDev& d = t->d;
    if (d.n_conns >= t->max_conns) {
        set_error("cn_tx_open: max connections reached");
        return CN_E_CAPACITY;
    }
    if (n_paths < 1 || static_cast<uint32_t>(n_paths) > d.max_paths) {
        set_error("cn_tx_open: n_paths outside [1, max_paths]");
        return CN_E_INVALID;
    }
    auto it = t->hid.find(src);
    uint32_t h;
    if (it == t->hid.end()) {
        h = d.n_hosts;
        t->hid[src] = h;
        t->nconns.push_back(0);
        d.n_hosts += 1;
    } else {
        h = it->second;
    }
    if (t->nconns[h] >= d.mcph) {
        set_error("cn_tx_open: host " + std::to_string(src) + " has max_conns_per_host connections already");
        return CN_E_CAPACITY;
    }
    const uint32_t c = d.n_conns++;
    t->host_of.push_back(h);
    t->loc.push_back(t->nconns[h]);
    t->nconns[h] += 1;
    t->max_k = std::max(t->max_k, t->nconns[h]);
    (void)dst;
    *out_c = c;
    return CN_OK;
}

// uploads the host tables, initialises connections [c0, c0 + n) and the descriptor
static int tx_commit(cn_tx* t, uint32_t c0, uint32_t n, const int32_t* src, const int32_t* dst, const int32_t* np) {
    TxDev& d = t->d;
    for (uint32_t j = 0; j < n; ++j) {
        const uint32_t c = c0 + j, h = t->host_of[c];
        CNB_CUDA(cudaMemcpy(d.host_conns + static_cast<size_t>(h) * d.mcph + t->loc[c], &c, 4, cudaMemcpyHostToDevice));
        CNB_CUDA(cudaMemcpy(d.conn_local + c, &t->loc[c], 4, cudaMemcpyHostToDevice));
    }
    std::vector<uint32_t> touched;
    for (uint32_t j = 0; j < n; ++j) touched.push_back(t->host_of[c0 + j]);
    std::sort(touched.begin(), touched.end());
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    for (uint32_t h : touched) {
        CNB_CUDA(cudaMemcpy(d.host_nconns + h, &t->nconns[h], 4, cudaMemcpyHostToDevice));
        CNB_CUDA(cudaMemcpy(d.host_blob + static_cast<size_t>(h) * d.host_bytes + offsetof(HostHdr, n_conns),
                            &t->nconns[h], 4, cudaMemcpyHostToDevice));
    }
    CNB_CUDA(cudaMemcpy(t->d_src + c0, src, 4ull * n, cudaMemcpyHostToDevice));
    CNB_CUDA(cudaMemcpy(t->d_dst + c0, dst, 4ull * n, cudaMemcpyHostToDevice));
    CNB_CUDA(cudaMemcpy(t->d_np + c0, np, 4ull * n, cudaMemcpyHostToDevice));
    CNB_CUDA(cudaMemcpy(t->d_dev, &d, sizeof(TxDev), cudaMemcpyHostToDevice));
    k_tx_init<<<n, 128>>>(d, c0, t->d_src, t->d_dst, t->d_np, fnv1a64_h("transport.conn"), t->seed,
                          t->stream_index0);
    CNB_CUDA(cudaGetLastError());
    CNB_CUDA(cudaDeviceSynchronize());
    return CN_OK;
}

extern "C" int cn_tx_create(const cn_tx_config* cfg, uint32_t n_conns, const int32_t* h_src,
                            const int32_t* h_dst, const int32_t* h_n_paths, cn_tx** out) {
    if (!cfg || !out || n_conns == 0) {
        set_error("cn_tx_create: bad arguments");
        return CN_E_INVALID;
    }
    std::vector<int32_t> src(n_conns), dst(n_conns), np(n_conns);
    std::map<int32_t, uint32_t> cnt;
    uint32_t mcph = 1;
    for (uint32_t c = 0; c < n_conns; ++c) {
        src[c] = h_src ? h_src[c] : static_cast<int32_t>(c);
        dst[c] = h_dst ? h_dst[c] : 0;
        np[c] = h_n_paths ? h_n_paths[c] : static_cast<int32_t>(cfg->max_paths);
        mcph = std::max(mcph, ++cnt[src[c]]);
    }
    cn_tx* t = nullptr;
    int rc = tx_alloc(cfg, n_conns, mcph, &t);
    if (rc != CN_OK) return rc;
    for (uint32_t c = 0; c < n_conns; ++c) {
        uint32_t k;
        rc = tx_register(t, src[c], dst[c], np[c], &k);
        if (rc != CN_OK) {
            cn_tx_destroy(t);
            return rc;
        }
    }
    rc = tx_commit(t, 0, n_conns, src.data(), dst.data(), np.data());
    if (rc != CN_OK) {
        cn_tx_destroy(t);
        return rc;
    }
    *out = t;
    return CN_OK;
}

// An engine whose connections open one at a time (cn_tx_open), in the
// order the reference's conn_to creates them.
extern "C" int cn_tx_create_empty(const cn_tx_config* cfg, uint32_t max_conns, uint32_t max_conns_per_host,
                                  cn_tx** out) {
    return tx_alloc(cfg, max_conns, max_conns_per_host, out);
}

extern "C" int cn_tx_open(cn_tx* t, int32_t src, int32_t dst, int32_t n_paths) {
    if (!t) return CN_E_INVALID;
    uint32_t c;
    int rc = tx_register(t, src, dst, n_paths, &c);
    if (rc != CN_OK) return rc;
    rc = tx_commit(t, c, 1, &src, &dst, &n_paths);
    return rc != CN_OK ? rc : static_cast<int>(c);
}

extern "C" void cn_tx_destroy(cn_tx* t) {
    if (!t) return;
    cudaDeviceSynchronize();
    TxDev& d = t->d;
    void* ptrs[] = {d.conns,  d.host_blob, d.conn_blob, d.host_conns, d.host_nconns, d.conn_local, d.ring,
                    d.fq,     d.c_path,    d.c_txt,     d.c_dead,     d.c_att,       d.c_fl,       d.c_dup,
                    d.c_q,    d.c_psn,     d.so_ref,    d.gq_ref,     d.gq_from,     d.status,     t->d_dev,
                    t->d_src, t->d_dst,    t->d_np};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    delete t;
}

extern "C" uint32_t cn_tx_n_hosts(cn_tx* t) { return t ? t->d.n_hosts : 0; }
extern "C" int32_t cn_tx_conn_host(cn_tx* t, uint32_t conn) {
    return t && conn < t->d.n_conns ? static_cast<int32_t>(t->host_of[conn]) : -1;
}

extern "C" int cn_tx_run(cn_tx* t, const uint32_t* d_ev_off, const uint64_t* d_events,
                         const cn_tx_submit* d_submits, const cn_ack_rec* d_acks, int64_t end_time,
                         cn_tx_rec* d_log, cn_tx_stats* d_stats, void* stream) {
    if (!t || !d_ev_off || !d_log || !d_stats) {
        set_error("cn_tx_run: bad arguments");
        return CN_E_INVALID;
    }
    if (t->d.n_hosts == 0) return CN_OK;
    const size_t per_warp = t->d.host_bytes + static_cast<size_t>(t->max_k) * t->d.conn_bytes;
    uint32_t wpb = static_cast<uint32_t>(std::min<size_t>(4, (227 * 1024) / per_warp));
    if (wpb == 0) wpb = 1;
    const uint32_t blocks = (t->d.n_hosts + wpb - 1) / wpb;
    k_tx_run<<<blocks, wpb * 32, wpb * per_warp, static_cast<cudaStream_t>(stream)>>>(
        t->d_dev, wpb, static_cast<uint32_t>(per_warp), d_ev_off, d_events, d_submits, d_acks, end_time, d_log,
        d_stats);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

// per host log counts (HostHdr::log_n)
extern "C" int cn_tx_log_counts(cn_tx* t, uint32_t* h_out) {
    if (!t || !h_out) return CN_E_INVALID;
    for (uint32_t h = 0; h < t->d.n_hosts; ++h)
        CNB_CUDA(cudaMemcpy(h_out + h, t->d.host_blob + static_cast<size_t>(h) * t->d.host_bytes +
                                             offsetof(HostHdr, log_n),
                            4, cudaMemcpyDeviceToHost));
    return CN_OK;
}

// Drops the first `n[h]` records of each host's log (the ones a caller has
// read); the rest move to the front and stay pollable.
extern "C" int cn_tx_log_consume(cn_tx* t, cn_tx_rec* d_log, const uint32_t* h_n) {
    if (!t || !d_log || !h_n) return CN_E_INVALID;
    std::vector<uint32_t> cnt(t->d.n_hosts);
    int rc = cn_tx_log_counts(t, cnt.data());
    if (rc != CN_OK) return rc;
    cn_tx_rec* tmp = nullptr;
    for (uint32_t h = 0; h < t->d.n_hosts; ++h) {
        const uint32_t have = std::min(cnt[h], t->d.log_cap);
        const uint32_t drop = std::min(h_n[h], have);
        const uint32_t keep = have - drop;
        if (keep && drop) {
            if (!tmp) CNB_CUDA(cudaMalloc(&tmp, static_cast<size_t>(t->d.log_cap) * sizeof(cn_tx_rec)));
            cn_tx_rec* base = d_log + static_cast<size_t>(h) * t->d.log_cap;
            CNB_CUDA(cudaMemcpy(tmp, base + drop, keep * sizeof(cn_tx_rec), cudaMemcpyDeviceToDevice));
            CNB_CUDA(cudaMemcpy(base, tmp, keep * sizeof(cn_tx_rec), cudaMemcpyDeviceToDevice));
        }
        const uint32_t left = cnt[h] - drop;  // overflowed records stay counted (status bit set)
        CNB_CUDA(cudaMemcpy(t->d.host_blob + static_cast<size_t>(h) * t->d.host_bytes + offsetof(HostHdr, log_n),
                            &left, 4, cudaMemcpyHostToDevice));
    }
    if (tmp) cudaFree(tmp);
    return CN_OK;
}

extern "C" int cn_tx_log_clear(cn_tx* t, void* stream) {
    if (!t) return CN_E_INVALID;
    for (uint32_t h = 0; h < t->d.n_hosts; ++h)
        CNB_CUDA(cudaMemsetAsync(t->d.host_blob + static_cast<size_t>(h) * t->d.host_bytes + offsetof(HostHdr, log_n),
                                 0, 4, static_cast<cudaStream_t>(stream)));
    return CN_OK;
}

extern "C" int cn_tx_status(cn_tx* t, unsigned int* out) {
    if (!t || !out) return CN_E_INVALID;
    CNB_CUDA(cudaMemcpy(out, t->d.status, 4, cudaMemcpyDeviceToHost));
    return CN_OK;
}

// Debug: raw device state of connection `conn` (its blob, global state and
// the chunk state of its pool share) into a host buffer.
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
    put(d.conn_blob + static_cast<size_t>(conn) * d.conn_bytes, d.conn_bytes);
    put(d.conns + conn, sizeof(TxConnG));
    put(d.host_blob + static_cast<size_t>(t->host_of[conn]) * d.host_bytes, d.host_bytes);
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
    const TxDev& d = t->d;
    std::vector<uint8_t> b(d.conn_bytes);
    CNB_CUDA(cudaMemcpy(b.data(), d.conn_blob + static_cast<size_t>(conn) * d.conn_bytes, d.conn_bytes,
                        cudaMemcpyDeviceToHost));
    const CHot* h = reinterpret_cast<const CHot*>(b.data());
    out->credit = h->credit;
    out->unchunked = h->unchunked;
    out->n_paths = h->n_paths;
    out->opened = h->opened;
    out->home_engine = h->home;
    out->pad = 0;
    out->inflight = h->total_inflight;
    const uint32_t n = std::min<uint32_t>(max_paths, static_cast<uint32_t>(h->n_paths));
    const int64_t* infl = reinterpret_cast<const int64_t*>(b.data() + d.o_infl);
    const Cc* cc = reinterpret_cast<const Cc*>(b.data() + d.o_cc);
    if (h_path_inflight)
        for (uint32_t p = 0; p < n; ++p) h_path_inflight[p] = infl[p];
    return CN_OK;
}

// window_available (transport.cpp:1185-1191): the path's CC window minus the
// inflight it gates
extern "C" int cn_tx_window_available(cn_tx* t, uint32_t conn, int32_t path, int64_t* out) {
    if (!t || !out || conn >= t->d.n_conns) return CN_E_INVALID;
    CNB_CUDA(cudaDeviceSynchronize());
    const TxDev& d = t->d;
    std::vector<uint8_t> b(d.conn_bytes);
    CNB_CUDA(cudaMemcpy(b.data(), d.conn_blob + static_cast<size_t>(conn) * d.conn_bytes, d.conn_bytes,
                        cudaMemcpyDeviceToHost));
    const CHot* h = reinterpret_cast<const CHot*>(b.data());
    if (path < 0 || path >= h->n_paths) {
        *out = 0;
        return CN_OK;
    }
    const int64_t* infl = reinterpret_cast<const int64_t*>(b.data() + d.o_infl);
    const Cc* cc = reinterpret_cast<const Cc*>(b.data() + d.o_cc) + (d.per_path ? path : 0);
    *out = cc->cwnd - (d.per_path ? infl[path] : h->total_inflight);
    return CN_OK;
}

// Engine introspection (engine_inflight_msgs / dispatched / gauge,
// transport.cpp:1193-1203) of the host that connection `conn` belongs to
extern "C" int cn_tx_get_engine_state(cn_tx* t, uint32_t conn, int32_t engine, cn_tx_engine_state* out) {
    if (!t || !out || conn >= t->d.n_conns || engine < 0 || static_cast<uint32_t>(engine) >= t->d.engines)
        return CN_E_INVALID;
    CNB_CUDA(cudaDeviceSynchronize());
    Eng e;
    CNB_CUDA(cudaMemcpy(&e, t->d.host_blob + static_cast<size_t>(t->host_of[conn]) * t->d.host_bytes +
                                sizeof(HostHdr) + sizeof(Eng) * engine,
                        sizeof(Eng), cudaMemcpyDeviceToHost));
    out->inflight_msgs = e.inflight_msgs;
    out->ring_len = e.ring_len;
    out->dispatched = e.dispatched;
    out->gauge = e.gauge;
    out->committed_unsent = e.committed_unsent;
    return CN_OK;
}

// glibc cbrt (mode 0) / pow(x, 3) (mode 1) restated on the device
// (libm_exact.cuh): the KAT hook of the CUBIC parity tests
extern "C" int cn_libm_eval(int mode, const double* d_in, double* d_out, uint64_t n, void* stream) {
    if ((mode != 0 && mode != 1) || (n && (!d_in || !d_out))) return CN_E_INVALID;
    if (!n) return CN_OK;
    k_libm_eval<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(mode, d_in, d_out, n);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}
