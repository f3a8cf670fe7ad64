// tx.cu -- device sender engine: ack processing, loss detection and
// retransmission of the selective multipath transport (sm_100a).
//
// Restates, per connection, the reference sender's event handling
// (/root/reference/proj/src/transport.cpp):
//   send_message / dispatch         :144-218   (msg ids LIFO, :127-129)
//   pump / commit_chunks / egress   :232-431   (factory rotation, 128-chunk
//                                               window, retransmissions first)
//   send_chunk                      :433-494   (attempts, tx_time, deadline)
//   queue_rtx                       :516-542   (path via on_tx_rtx_chunk)
//   release_chunk / advance / finish:807-847
//   handle_ack                      :849-942   (cause release + RTT sample,
//                                               cumulative + SACK release,
//                                               dup hints -> fast retransmit)
//   cur_rto / arm_rto / rto_fire    :1078-1169 (backoff x2 capped at 64)
//   RttEstimator                    cc.hpp:12-35
// for the configuration the survey fixes for sender parity:
// congestion control none (OpenLoop: cwnd never gates, RTT samples still
// feed the RTO), one engine per host, DefaultPolicy.  Every send happens at
// the time of the event that triggers it, exactly as the reference's
// synchronous pump.
//
// One warp per connection consumes a time-ordered stream of events (message
// submissions, acks delivered at the sender) and fires its own RTO timer in
// between.  Control flow is warp-uniform; the chunk-window scans (cumulative
// and SACK release, duplicate hints, base advance, the RTO expiry scan) run
// one chunk per lane with ballots; path choices come from the connection's
// RngStream (rng.cuh), bit-identical to the reference.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <climits>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace cnb {

enum : uint32_t { TF_SENT = 1, TF_ACKED = 2, TF_RTXP = 4 };
constexpr int kTxWindow = 128;   // kCsnWindow (transport.cpp:14)
constexpr int kBackoffCap = 64;  // kBackoffCap (transport.cpp:15)
constexpr int kTxWarps = 4;

struct TxMsg {
    uint64_t seq, tag, len, chunked, chunk_base;
    uint32_t nchunks, base, acked, live, in_factory, pad0;
};

struct TxConn {
    int64_t srtt, rttvar, armed_at, timer_at, committed_unsent;
    uint64_t next_seq, chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_sent, msgs_completed, backpressured;
    int32_t has_sample, backoff, timer_armed, n_free, fq_head, fq_count, src, dst, conn_id,
        n_paths, live_msgs, pad0;
    uint32_t live_mask[4];  // message slots in use (bit = msg id)
    uint8_t free_ids[128];
    uint8_t fq[128];
    TxMsg msgs[128];
};

struct TxDev {
    uint32_t n_conns, cb, max_pl, dupack, avoid_prev, policy, max_inflight, log_cap;
    int64_t rto_min, rto_max, commit_ahead;
    uint64_t pool_cap;
    TxConn* conns;
    int32_t* c_path;
    int64_t* c_txt;
    int64_t* c_dead;
    int32_t* c_att;
    uint32_t* c_fl;
    int32_t* c_dup;
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
    double* rtt_s;  // PathScoreboard (lb.hpp:15-36), shared memory copy
    double* ecn_s;
    int n;          // paths of this connection
    cn_tx_rec* log;
    uint32_t log_n;
    // RttEstimator + timer + counters (warp-uniform registers)
    int64_t srtt, rttvar, armed_at, timer_at, committed_unsent;
    int has_sample, backoff, timer_armed;
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
    __device__ void arm_rto(int64_t now) {  // transport.cpp:1083-1092
        if (timer_armed) return;
        timer_armed = 1;
        armed_at = now;
        timer_at = now + cur_rto() * backoff;
    }
    __device__ int select(int prev_path) {  // DefaultPolicy (policy.hpp:80-91)
        int p = select_seq(r, d.policy, n, d.policy == 2 ? ecn_s : rtt_s, lane);
        if (prev_path >= 0 && d.avoid_prev && n > 1 && p == prev_path) p = (p + 1) % n;
        return p;
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
    // send_chunk (transport.cpp:433-494) for chunk e of message mid
    __device__ void send_chunk(int64_t now, uint32_t mid, const TxMsg& m, uint32_t ci, bool rtx) {
        uint64_t e = m.chunk_base + ci;
        int64_t dl = now + cur_rto() * backoff;
        if (lane == 0) {
            d.c_att[e] += 1;
            d.c_fl[e] = TF_SENT | (d.c_fl[e] & TF_ACKED);
            d.c_dup[e] = 0;
            d.c_txt[e] = now;
            d.c_dead[e] = dl;
        }
        uint64_t off = static_cast<uint64_t>(ci) * d.cb;
        uint64_t len = m.len - off < d.cb ? m.len - off : d.cb;
        if (rtx) {
            ++chunk_rtx;
        } else {
            ++chunks_sent;
            committed_unsent -= static_cast<int64_t>(len);
        }
        record(now, mid, ci, d.c_path[e], rtx || d.c_att[e] > 1, m.seq);
        __syncwarp();
        arm_rto(now);
    }
    // queue_rtx (transport.cpp:516-542); caller checked sent && !acked && !rtx_pending
    __device__ void queue_rtx(const TxMsg& m, uint32_t ci) {
        uint64_t e = m.chunk_base + ci;
        int prev = d.c_path[e];  // attempts > 0: prev_path = ch.path (view_of, :509)
        int p = select(prev);
        if (lane == 0) {
            d.c_fl[e] |= TF_RTXP;
            d.c_dup[e] = 0;
            d.c_path[e] = p;
        }
        __syncwarp();
    }
};

__device__ __forceinline__ TxMsg load_msg(const TxConn* C, uint32_t mid) { return C->msgs[mid]; }
__device__ __forceinline__ void store_msg(TxConn* C, uint32_t mid, const TxMsg& m, int lane) {
    if (lane == 0) C->msgs[mid] = m;
    __syncwarp();
}

// egress (transport.cpp:329-431) with an open cwnd: retransmissions first,
// then every committed, unsent chunk.  Returns the number of sends.
__device__ uint32_t egress(Tx& x, int64_t now) {
    uint32_t sent = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
            const uint32_t mid = q * 32 + __ffs(lb) - 1;
            TxMsg m = load_msg(x.C, mid);
            for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
                uint32_t ci = w0 + x.lane;
                uint32_t fl = ci < m.nchunks ? x.d.c_fl[m.chunk_base + ci] : (TF_SENT | TF_ACKED);
                bool want = pass == 0 ? ((fl & TF_RTXP) && !(fl & TF_ACKED)) : !(fl & TF_SENT);
                unsigned b = __ballot_sync(0xffffffffu, want);
                for (; b; b &= b - 1) {
                    uint32_t cj = w0 + __ffs(b) - 1;
                    x.send_chunk(now, mid, m, cj, pass == 0);
                    ++sent;
                }
            }
        }
    }
    return sent;
}

// commit_chunks (transport.cpp:244-310): one chunk per message per turn of
// the factory rotation, window-stalled at 128 unacked chunks, bounded by
// commit_ahead bytes.
__device__ void commit_chunks(Tx& x, int64_t now) {
    TxConn* C = x.C;
    int32_t head = C->fq_head, count = C->fq_count;
    uint32_t stalled = 0;
    while (count > 0 && stalled < static_cast<uint32_t>(count) && x.committed_unsent < x.d.commit_ahead) {
        uint32_t mid = C->fq[head];
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
            if (x.lane == 0) C->fq[(head + count) & 127] = static_cast<uint8_t>(mid);
            __syncwarp();
            ++count;
            ++stalled;
            continue;
        }
        uint64_t rem = m.len - m.chunked;
        uint32_t sz = rem < x.d.cb ? static_cast<uint32_t>(rem) : x.d.cb;
        uint32_t ci = m.nchunks;
        int p = x.select(-1);  // on_select_path (:281-287)
        if (x.lane == 0) {
            uint64_t e = m.chunk_base + ci;
            x.d.c_path[e] = p;
            x.d.c_fl[e] = 0;
            x.d.c_att[e] = 0;
            x.d.c_dup[e] = 0;
        }
        m.nchunks = ci + 1;
        m.chunked += sz;
        x.committed_unsent += sz;
        if (m.chunked < m.len) {
            if (x.lane == 0) C->fq[(head + count) & 127] = static_cast<uint8_t>(mid);
            __syncwarp();
            ++count;
        } else {
            m.in_factory = 0;
        }
        store_msg(C, mid, m, x.lane);
        stalled = 0;
    }
    if (x.lane == 0) {
        C->fq_head = head;
        C->fq_count = count;
    }
    __syncwarp();
}

__device__ void pump(Tx& x, int64_t now) {  // transport.cpp:232-240
    for (;;) {
        commit_chunks(x, now);
        if (egress(x, now) == 0) break;
    }
}

// try_advance_base (:825-829): first unacked chunk at or after base
__device__ uint32_t advance_base(const Tx& x, const TxMsg& m) {
    uint32_t b = m.base;
    while (b < m.nchunks) {
        uint32_t ci = b + x.lane;
        bool acked = ci < m.nchunks ? (x.d.c_fl[m.chunk_base + ci] & TF_ACKED) != 0 : false;
        unsigned un = __ballot_sync(0xffffffffu, !acked);
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

// release_chunk (:807-823) of a lane-owned chunk, rtt = 0 (no estimator or
// scoreboard effect under OpenLoop); returns whether it released.
__device__ __forceinline__ bool release_lane(const Tx& x, uint64_t e) {
    uint32_t fl = x.d.c_fl[e];
    if ((fl & TF_ACKED) || !(fl & TF_SENT)) return false;
    x.d.c_fl[e] = (fl | TF_ACKED) & ~TF_RTXP;
    return true;
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
        uint8_t rel = static_cast<uint8_t>(((a.hdr >> 9) & 0xFF) - base_csn);
        if (rel < kTxWindow && m.base + rel < nch) cause = m.base + rel;
    }
    if (cause >= 0) {  // cause chunk: the only trustworthy RTT echo (:869-887)
        uint64_t e = m.chunk_base + cause;
        uint32_t fl = x.d.c_fl[e];
        if ((fl & TF_SENT) && !(fl & TF_ACKED)) {
            int64_t rtt = 0;
            if (x.d.c_att[e] == 1 && a.echo_tx_time == x.d.c_txt[e] && now > a.echo_tx_time)
                rtt = now - a.echo_tx_time;
            bool ecn = (a.flags & CN_ACK_ECN_ECHO) != 0;
            int path = x.d.c_path[e];
            __syncwarp();
            if (x.lane == 0) x.d.c_fl[e] = (fl | TF_ACKED) & ~TF_RTXP;
            __syncwarp();
            m.acked += 1;
            if (rtt > 0) {
                x.est_sample(rtt);  // OpenLoop::on_ack (cc.cpp:23-25)
                if (x.lane == 0) {   // board.record_rtt / record_ecn (:819-822)
                    x.rtt_s[path] += (static_cast<double>(rtt) - x.rtt_s[path]) / 8.0;
                    x.ecn_s[path] += ((ecn ? 1.0 : 0.0) - x.ecn_s[path]) / 8.0;
                }
                __syncwarp();
            }
            ++newly;
        }
    }
    // cumulative bound (:890-897)
    uint32_t rcum = m.base;
    if (a.flags & CN_ACK_CUM_VALID) {
        uint8_t rel1 = static_cast<uint8_t>(static_cast<uint8_t>(a.cum_csn + 1) - base_csn);
        if (rel1 <= kTxWindow) rcum = m.base + rel1;
    } else {
        rcum = 0;
    }
    const uint32_t cend = rcum < nch ? rcum : nch;
    for (uint32_t w0 = m.base; w0 < cend; w0 += 32) {  // :898-904
        uint32_t ci = w0 + x.lane;
        bool rel = ci < cend && release_lane(x, m.chunk_base + ci);
        uint32_t c = __popc(__ballot_sync(0xffffffffu, rel));
        m.acked += c;
        newly += c;
    }
    __syncwarp();
    for (int q = 0; q < 4; ++q) {  // SACK (:905-914)
        uint32_t j = q * 32 + x.lane;
        bool bit = ((q < 2 ? a.sack[0] >> (j & 63) : a.sack[1] >> (j & 63)) & 1ull) != 0;
        uint64_t i = static_cast<uint64_t>(rcum) + j;
        bool rel = bit && i < nch && release_lane(x, m.chunk_base + i);
        uint32_t c = __popc(__ballot_sync(0xffffffffu, rel));
        m.acked += c;
        newly += c;
    }
    __syncwarp();
    // duplicate hints -> fast retransmit, ascending chunk order (:918-929)
    if (cause >= 0) {
        for (uint32_t w0 = m.base; w0 < static_cast<uint32_t>(cause); w0 += 32) {
            uint32_t ci = w0 + x.lane;
            bool trig = false;
            if (ci < static_cast<uint32_t>(cause)) {
                uint64_t e = m.chunk_base + ci;
                uint32_t fl = x.d.c_fl[e];
                if ((fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP))) {
                    int32_t dup = x.d.c_dup[e] + 1;
                    x.d.c_dup[e] = dup;
                    trig = dup >= static_cast<int32_t>(x.d.dupack);
                }
            }
            __syncwarp();
            for (unsigned b = __ballot_sync(0xffffffffu, trig); b; b &= b - 1) {
                ++x.fast_rtx;
                x.queue_rtx(m, w0 + __ffs(b) - 1);
            }
        }
    }
    m.base = advance_base(x, m);  // :931
    bool done = m.chunked >= m.len && nch > 0 && m.acked == nch && !m.in_factory;
    store_msg(C, mid, m, x.lane);
    if (done) msg_finished(x, mid);  // :932-934
    if (newly > 0) {  // :936-940
        x.backoff = 1;
        x.timer_armed = 0;
        x.arm_rto(now);
    }
    pump(x, now);  // :941
}

// rto_fire (:1094-1169), the live timer at x.timer_at
__device__ void rto_fire(Tx& x) {
    TxConn* C = x.C;
    const int64_t now = x.timer_at;
    x.timer_armed = 0;
    // scan: msg slots 0..127 x [base, n): oldest deadline (first wins) and
    // the expired set in scan order
    int64_t best = 0;
    bool have = false;
    uint32_t n_exp = 0;
    for (uint32_t q = 0; q < 4; ++q)
    for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
        const uint32_t mid = q * 32 + __ffs(lb) - 1;
        TxMsg m = load_msg(C, mid);
        for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
            uint32_t ci = w0 + x.lane;
            bool elig = false;
            int64_t dl = 0;
            if (ci < m.nchunks) {
                uint64_t e = m.chunk_base + ci;
                uint32_t fl = x.d.c_fl[e];
                elig = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP));
                dl = x.d.c_dead[e];
            }
            // min deadline with the lowest scan position winning ties
            long long v = elig ? dl : LLONG_MAX;
            long long mn = v;
            for (int o = 16; o > 0; o >>= 1) {
                long long t = __shfl_xor_sync(0xffffffffu, mn, o);
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
        return;
    }
    ++x.rtos;
    x.backoff = x.backoff * 2 < kBackoffCap ? x.backoff * 2 : kBackoffCap;
    // queue_rtx for every expired chunk in scan order (:1154-1164)
    for (uint32_t q = 0; q < 4; ++q)
    for (uint32_t lb = x.live[q]; lb; lb &= lb - 1) {
        const uint32_t mid = q * 32 + __ffs(lb) - 1;
        TxMsg m = load_msg(C, mid);
        for (uint32_t w0 = m.base; w0 < m.nchunks; w0 += 32) {
            uint32_t ci = w0 + x.lane;
            bool ex = false;
            if (ci < m.nchunks) {
                uint64_t e = m.chunk_base + ci;
                uint32_t fl = x.d.c_fl[e];
                ex = (fl & TF_SENT) && !(fl & (TF_ACKED | TF_RTXP)) && x.d.c_dead[e] <= now;
            }
            for (unsigned b = __ballot_sync(0xffffffffu, ex); b; b &= b - 1)
                x.queue_rtx(m, w0 + __ffs(b) - 1);
        }
    }
    x.arm_rto(now);  // :1167
    pump(x, now);    // :1168
}

// send_message (:144-196) + dispatch (:198-218)
__device__ void submit(Tx& x, int64_t now, const cn_tx_submit& s) {
    TxConn* C = x.C;
    if (s.len == 0 || C->n_free == 0) {  // len 0 throws in the reference; counted here
        if (x.lane == 0) C->backpressured += 1;
        __syncwarp();
        if (s.len == 0 && x.lane == 0) atomicOr(x.d.status, 1u);
        return;
    }
    uint32_t mid = C->free_ids[C->n_free - 1];
    uint64_t seq = C->next_seq;
    if (x.lane == 0) C->next_seq = seq + 1;
    __syncwarp();
    if (static_cast<uint32_t>(C->live_msgs) >= x.d.max_inflight) {
        if (x.lane == 0) C->backpressured += 1;
        __syncwarp();
        return;
    }
    uint64_t nc = (s.len + x.d.cb - 1) / x.d.cb;
    unsigned long long base = 0;
    if (x.lane == 0) base = atomicAdd(x.d.pool_top, static_cast<unsigned long long>(nc));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + nc > x.d.pool_cap) {
        if (x.lane == 0) atomicOr(x.d.status, 4u);
        return;
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
    pump(x, now);
}

__global__ void __launch_bounds__(kTxWarps * 32) k_tx_run(TxDev d, const uint32_t* __restrict__ ev_off,
                                                         const uint64_t* __restrict__ events,
                                                         const cn_tx_submit* __restrict__ submits,
                                                         const cn_ack_rec* __restrict__ acks,
                                                         int64_t end_time, cn_tx_rec* __restrict__ log,
                                                         uint32_t* __restrict__ log_n,
                                                         cn_tx_stats* __restrict__ stats) {
    extern __shared__ uint64_t sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t conn = blockIdx.x * kTxWarps + w;
    if (conn >= d.n_conns) return;
    uint64_t* mt = sm + static_cast<size_t>(w) * (2 * kMtN + 2 * d.s.max_paths);
    TxConn* C = d.conns + conn;
    Tx x{d, C, conn, lane, WarpRng{mt, mt + kMtN, 0},
         reinterpret_cast<double*>(mt + 2 * kMtN), reinterpret_cast<double*>(mt + 2 * kMtN + d.s.max_paths),
         C->n_paths, log + static_cast<uint64_t>(conn) * d.log_cap, log_n[conn]};
    // stream + boards into shared memory
    for (int k = lane; k < kMtN; k += 32) mt[k] = d.s.mt[static_cast<uint64_t>(conn) * kMtN + k];
    for (int p = lane; p < x.n; p += 32) {
        x.rtt_s[p] = d.s.rtt[static_cast<uint64_t>(conn) * d.s.max_paths + p];
        x.ecn_s[p] = d.s.ecn[static_cast<uint64_t>(conn) * d.s.max_paths + p];
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
    x.has_sample = C->has_sample;
    x.backoff = C->backoff;
    x.timer_armed = C->timer_armed;
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
        // timers scheduled during the run fire after same-time events (DES order)
        while (x.timer_armed && x.timer_at < t) rto_fire(x);
        if (type == 0) {
            cn_tx_submit s = submits[idx];
            submit(x, t, s);
        } else {
            cn_ack_rec a = acks[idx];
            handle_ack(x, t, a);
        }
    }
    while (x.timer_armed && x.timer_at <= end_time) rto_fire(x);
    // persist
    for (int k = lane; k < kMtN; k += 32) d.s.mt[static_cast<uint64_t>(conn) * kMtN + k] = mt[k];
    for (int p = lane; p < x.n; p += 32) {
        d.s.rtt[static_cast<uint64_t>(conn) * d.s.max_paths + p] = x.rtt_s[p];
        d.s.ecn[static_cast<uint64_t>(conn) * d.s.max_paths + p] = x.ecn_s[p];
    }
    if (lane == 0) {
        d.s.mt_idx[conn] = x.r.idx;
        C->srtt = x.srtt;
        C->rttvar = x.rttvar;
        C->armed_at = x.armed_at;
        C->timer_at = x.timer_at;
        C->committed_unsent = x.committed_unsent;
        C->has_sample = x.has_sample;
        C->backoff = x.backoff;
        C->timer_armed = x.timer_armed;
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
        stats[conn] = st;
    }
}

__global__ void k_tx_init(TxDev d, const int32_t* src, const int32_t* dst, const int32_t* np) {
    uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d.n_conns) return;
    TxConn* C = d.conns + c;
    memset(C, 0, sizeof(TxConn));
    C->backoff = 1;
    C->next_seq = 1;
    C->src = src ? src[c] : 0;
    C->dst = dst ? dst[c] : 0;
    C->n_paths = np ? np[c] : static_cast<int32_t>(d.s.max_paths);
    C->conn_id = static_cast<int32_t>(c & 0xFF);
    for (int i = 0; i < 128; ++i) C->free_ids[i] = static_cast<uint8_t>(127 - i);  // :127-129
    C->n_free = 128;
}

}  // namespace cnb

using namespace cnb;

struct cn_tx {
    TxDev d;
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
    c->seed = 0;
    c->stream_index0 = 0;
    c->log_cap = 1u << 16;
}

extern "C" int cn_tx_create(const cn_tx_config* cfg, uint32_t n_conns, const int32_t* h_src,
                            const int32_t* h_dst, const int32_t* h_n_paths, cn_tx** out) {
    if (!cfg || !out || n_conns == 0 || cfg->chunk_bytes == 0 || cfg->rto_min <= 0 ||
        cfg->max_paths == 0 || cfg->lb_policy < 0 || cfg->lb_policy > 2) {
        set_error("cn_tx_create: bad config (rto_min must be resolved, > 0)");
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
    d.rto_min = cfg->rto_min;
    d.rto_max = cfg->rto_max > 0 ? cfg->rto_max : 64 * cfg->rto_min;  // transport.cpp:36
    d.commit_ahead = cfg->commit_ahead;
    d.pool_cap = cfg->chunk_pool;
    d.s = *sched_dev(t->sched);
    int32_t *src = nullptr, *dst = nullptr, *np = nullptr;
    bool ok = cudaMalloc(&d.conns, sizeof(TxConn) * n_conns) == cudaSuccess &&
              cudaMalloc(&d.c_path, cfg->chunk_pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_txt, cfg->chunk_pool * 8) == cudaSuccess &&
              cudaMalloc(&d.c_dead, cfg->chunk_pool * 8) == cudaSuccess &&
              cudaMalloc(&d.c_att, cfg->chunk_pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_fl, cfg->chunk_pool * 4) == cudaSuccess &&
              cudaMalloc(&d.c_dup, cfg->chunk_pool * 4) == cudaSuccess &&
              cudaMalloc(&d.pool_top, 8) == cudaSuccess && cudaMalloc(&d.status, 4) == cudaSuccess &&
              cudaMalloc(&t->d_logn, n_conns * 4ull) == cudaSuccess &&
              cudaMalloc(&src, n_conns * 4ull) == cudaSuccess && cudaMalloc(&dst, n_conns * 4ull) == cudaSuccess &&
              cudaMalloc(&np, n_conns * 4ull) == cudaSuccess;
    if (!ok) {
        set_error("cn_tx_create: out of device memory");
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
    cudaMemset(t->d_logn, 0, n_conns * 4ull);
    k_tx_init<<<(n_conns + 127) / 128, 128>>>(d, src, dst, np);
    cudaError_t e = cudaDeviceSynchronize();
    cudaFree(src);
    cudaFree(dst);
    cudaFree(np);
    if (e != cudaSuccess) return cuda_status(e, "cn_tx_create");
    int smem = kTxWarps * (2 * kMtN + 2 * static_cast<int>(cfg->max_paths)) * 8;
    cudaFuncSetAttribute(k_tx_run, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    *out = t;
    return CN_OK;
}

extern "C" void cn_tx_destroy(cn_tx* t) {
    if (!t) return;
    cudaDeviceSynchronize();
    TxDev& d = t->d;
    void* ptrs[] = {d.conns, d.c_path, d.c_txt, d.c_dead, d.c_att, d.c_fl, d.c_dup, d.pool_top,
                    d.status, t->d_logn};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    cn_sched_destroy(t->sched);
    delete t;
}

extern "C" int cn_tx_run(cn_tx* t, const uint32_t* d_ev_off, const uint64_t* d_events,
                         const cn_tx_submit* d_submits, const cn_ack_rec* d_acks, int64_t end_time,
                         cn_tx_rec* d_log, cn_tx_stats* d_stats, void* stream) {
    if (!t || !d_ev_off || !d_log || !d_stats) {
        set_error("cn_tx_run: bad arguments");
        return CN_E_INVALID;
    }
    int smem = kTxWarps * (2 * kMtN + 2 * static_cast<int>(t->d.s.max_paths)) * 8;
    k_tx_run<<<(t->d.n_conns + kTxWarps - 1) / kTxWarps, kTxWarps * 32, smem,
               static_cast<cudaStream_t>(stream)>>>(t->d, d_ev_off, d_events, d_submits, d_acks,
                                                    end_time, d_log, t->d_logn, d_stats);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_tx_status(cn_tx* t, unsigned int* out) {
    if (!t || !out) return CN_E_INVALID;
    CNB_CUDA(cudaMemcpy(out, t->d.status, 4, cudaMemcpyDeviceToHost));
    return CN_OK;
}
