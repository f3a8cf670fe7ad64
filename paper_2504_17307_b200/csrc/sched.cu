// sched.cu -- batched multipath chunk scheduler on sm_100a.
//
// Replaces the path-choice arithmetic of the reference sender:
//   RngStream (include/chunknet/rng.hpp:29-60): std::mt19937_64 seeded with
//       splitmix64(splitmix64(seed ^ fnv1a64(name)) + index); next_below =
//       std::uniform_int_distribution<uint64_t> (libstdc++ 13
//       bits/uniform_int_dist.h:257-320: Lemire over a 128-bit product)
//   PathScoreboard (include/chunknet/lb.hpp:15-36): rtt/ecn EWMA, gain 1/8
//   select_path (src/lb.cpp:7-27): oblivious / power-of-two choices
//   DefaultPolicy::on_select_path / on_tx_rtx_chunk (policy.hpp:80-91)
//
// One warp owns one connection's stream.  The Mersenne twist runs in two
// data-parallel halves (k < 156 reads only old words; k >= 156 reads words
// the first half already produced), tempering is per word, and a run of
// decisions is evaluated 32 at a time: with no Lemire rejection decision j
// consumes draws 2j, 2j+1 (P2) or j (oblivious), so lanes index the
// tempered block directly.  A draw with low64 < range (probability
// range/2^64) sends the warp to an exact lane-0 sequential path for that
// group, so the output is bit-identical to the sequential reference.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace cnb {

// Decisions for one connection per warp.  req[k] = prev_path for a
// retransmission (DefaultPolicy::on_tx_rtx_chunk), -1 for a fresh chunk.
__global__ void __launch_bounds__(256) k_select(SchedDev d, int policy, int avoid_prev,
                                                const uint32_t* __restrict__ conns,
                                                const uint32_t* __restrict__ offsets,
                                                const int32_t* __restrict__ req,
                                                int32_t* __restrict__ out, uint32_t n_groups,
                                                uint32_t uniform_count) {
    extern __shared__ uint64_t sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t grp = blockIdx.x * (blockDim.x >> 5) + w;
    if (grp >= n_groups) return;
    const uint32_t conn = conns ? conns[grp] : grp;
    uint64_t* mt = sm + static_cast<size_t>(w) * (2 * kMtN + d.max_paths);
    double* score = reinterpret_cast<double*>(mt + 2 * kMtN);
    WarpRng r{mt, mt + kMtN, 0};
    const uint64_t* gmt = d.mt + static_cast<uint64_t>(conn) * kMtN;
    for (int k = lane; k < kMtN; k += 32) mt[k] = gmt[k];
    const int n = d.n_paths[conn];
    const double* gs = (policy == 2 ? d.ecn : d.rtt) + static_cast<uint64_t>(conn) * d.max_paths;
    for (int p = lane; p < n; p += 32) score[p] = gs[p];
    r.idx = d.mt_idx[conn];
    __syncwarp();
    // the tempered outputs of the current block are not stored: regenerate
    // from the raw state (tempering is a pure function of the word)
    for (int k = lane; k < kMtN; k += 32) r.out[k] = temper(mt[k]);
    __syncwarp();
    const uint64_t o0 = offsets ? offsets[grp] : static_cast<uint64_t>(grp) * uniform_count;
    const uint32_t cnt = offsets ? offsets[grp + 1] - offsets[grp] : uniform_count;
    const int draws = n == 1 ? 0 : (policy == 0 ? 1 : 2);
    const uint64_t n1 = static_cast<uint64_t>(n), n2 = static_cast<uint64_t>(n > 1 ? n - 1 : 1);
    uint32_t k = 0;
    while (k < cnt) {
        uint32_t m = cnt - k < 32 ? cnt - k : 32;  // decisions in this group
        if (draws == 0) {
            if (lane < m) out[o0 + k + lane] = 0;
            k += m;
            continue;
        }
        const uint32_t avail = (kMtN - r.idx) / draws;  // whole decisions left in this block
        if (avail == 0) {
            if (r.idx >= kMtN) {
                refill(r, lane);
            } else {  // a decision straddles the twist: exact sequential step
                int32_t pv = req ? req[o0 + k] : -1;
                int p = select_seq(r, policy, n, score, lane);
                if (avoid_prev && pv >= 0 && n > 1 && p == pv) p = (p + 1) % n;
                if (lane == 0) out[o0 + k] = p;
                k += 1;
            }
            continue;
        }
        if (m > avail) m = avail;
        // parallel: lane j takes draws idx + draws*j (+1)
        bool rej = false;
        int p = 0;
        if (lane < m) {
            uint64_t u1 = r.out[r.idx + draws * lane];
            uint64_t lo1 = u1 * n1;
            int a = static_cast<int>(__umul64hi(u1, n1));
            rej = lo1 < n1;
            if (draws == 1) {
                p = a;
            } else {
                uint64_t u2 = r.out[r.idx + 2 * lane + 1];
                uint64_t lo2 = u2 * n2;
                int b = static_cast<int>(__umul64hi(u2, n2));
                rej = rej || lo2 < n2;
                if (b >= a) b++;
                p = pick_p2(a, b, score);
            }
        }
        unsigned rm = __ballot_sync(0xffffffffu, rej);
        uint32_t good = rm ? static_cast<uint32_t>(__ffs(rm) - 1) : m;  // decisions before the first candidate rejection
        if (lane < good) {
            int32_t pv = req ? req[o0 + k + lane] : -1;
            if (avoid_prev && pv >= 0 && n > 1 && p == pv) p = (p + 1) % n;
            out[o0 + k + lane] = p;
        }
        r.idx += draws * good;
        k += good;
        if (good < m) {  // exact sequential step through a possible rejection
            int32_t pv = req ? req[o0 + k] : -1;
            int q = select_seq(r, policy, n, score, lane);
            if (avoid_prev && pv >= 0 && n > 1 && q == pv) q = (q + 1) % n;
            if (lane == 0) out[o0 + k] = q;
            k += 1;
        }
        __syncwarp();
    }
    // persist the stream
    uint64_t* wmt = d.mt + static_cast<uint64_t>(conn) * kMtN;
    for (int x = lane; x < kMtN; x += 32) wmt[x] = mt[x];
    if (lane == 0) d.mt_idx[conn] = r.idx;
}

// Raw stream outputs / next_below sequences (parity + tooling), one warp.
__global__ void k_draws(SchedDev d, uint32_t conn, int mode, const uint64_t* __restrict__ ns,
                        uint64_t* __restrict__ out, uint64_t count) {
    __shared__ uint64_t sm[2 * kMtN];
    const int lane = threadIdx.x;
    WarpRng r{sm, sm + kMtN, 0};
    for (int k = lane; k < kMtN; k += 32) sm[k] = d.mt[static_cast<uint64_t>(conn) * kMtN + k];
    r.idx = d.mt_idx[conn];
    __syncwarp();
    for (int k = lane; k < kMtN; k += 32) r.out[k] = temper(sm[k]);
    __syncwarp();
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t v = mode == 0 ? next_u64_lane0(r, lane) : next_below_warp(r, ns[i], lane);
        if (lane == 0) out[i] = v;
    }
    for (int k = lane; k < kMtN; k += 32) d.mt[static_cast<uint64_t>(conn) * kMtN + k] = sm[k];
    if (lane == 0) d.mt_idx[conn] = r.idx;
}

// PathScoreboard::record_rtt / record_ecn (lb.hpp:23-28) for a list of
// samples, applied in list order per connection (one thread per connection
// scanning its samples: EWMA updates do not commute).
__global__ void k_record(SchedDev d, const uint32_t* __restrict__ conn, const int32_t* __restrict__ path,
                         const int64_t* __restrict__ rtt, const uint8_t* __restrict__ ecn,
                         const uint32_t* __restrict__ offsets, uint32_t n_groups) {
    uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= n_groups) return;
    for (uint32_t k = offsets[gi]; k < offsets[gi + 1]; ++k) {
        uint64_t x = static_cast<uint64_t>(conn[k]) * d.max_paths + path[k];
        double r = d.rtt[x];
        r += (static_cast<double>(rtt[k]) - r) / 8.0;  // exact: /8 is a power of two
        d.rtt[x] = r;
        double e = d.ecn[x];
        e += ((ecn[k] ? 1.0 : 0.0) - e) / 8.0;
        d.ecn[x] = e;
    }
}

}  // namespace cnb

using namespace cnb;

struct cn_sched {
    SchedDev d;
    int max_paths;
};

namespace cnb {
SchedDev* sched_dev(cn_sched* s) { return &s->d; }
}  // namespace cnb

extern "C" int cn_sched_create(uint32_t n_conns, uint32_t max_paths, const int32_t* h_n_paths,
                               double base_rtt_ns, uint64_t seed, const char* stream_name,
                               int64_t index0, cn_sched** out) {
    if (!out || n_conns == 0 || max_paths == 0 || max_paths > 1024) {
        set_error("cn_sched_create: bad arguments");
        return CN_E_INVALID;
    }
    *out = nullptr;
    cn_sched* s = new (std::nothrow) cn_sched();
    if (!s) return CN_E_CAPACITY;
    SchedDev& d = s->d;
    memset(&d, 0, sizeof d);
    d.n_conns = n_conns;
    d.max_paths = max_paths;
    s->max_paths = static_cast<int>(max_paths);
    std::vector<int32_t> np(n_conns, static_cast<int32_t>(max_paths));
    if (h_n_paths)
        for (uint32_t c = 0; c < n_conns; ++c) {
            if (h_n_paths[c] < 1 || static_cast<uint32_t>(h_n_paths[c]) > max_paths) {
                delete s;
                set_error("cn_sched_create: n_paths outside [1, max_paths]");
                return CN_E_INVALID;
            }
            np[c] = h_n_paths[c];
        }
    size_t boards = static_cast<size_t>(n_conns) * max_paths;
    if (cudaMalloc(&d.mt, static_cast<size_t>(n_conns) * kMtN * 8) != cudaSuccess ||
        cudaMalloc(&d.mt_idx, n_conns * 4ull) != cudaSuccess ||
        cudaMalloc(&d.rtt, boards * 8) != cudaSuccess || cudaMalloc(&d.ecn, boards * 8) != cudaSuccess ||
        cudaMalloc(&d.n_paths, n_conns * 4ull) != cudaSuccess) {
        cudaFree(d.mt);
        cudaFree(d.mt_idx);
        cudaFree(d.rtt);
        cudaFree(d.ecn);
        cudaFree(d.n_paths);
        delete s;
        return cuda_status(cudaErrorMemoryAllocation, "cn_sched_create");
    }
    // PathScoreboard(n_paths, base_rtt_ns): rtt prior = base rtt, ecn = 0
    std::vector<double> prior(boards, base_rtt_ns);
    cudaMemcpy(d.rtt, prior.data(), boards * 8, cudaMemcpyHostToDevice);
    cudaMemset(d.ecn, 0, boards * 8);
    cudaMemcpy(d.n_paths, np.data(), n_conns * 4ull, cudaMemcpyHostToDevice);
    uint64_t nh = fnv1a64_h(stream_name ? stream_name : "transport.conn");
    k_mt_seed<<<(n_conns + 127) / 128, 128>>>(d, nh, seed, index0 < 0 ? 0 : static_cast<uint64_t>(index0),
                                             index0 < 0 ? 0 : 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_status(e, "cn_sched_create: seed");
    int smem = (2 * kMtN + static_cast<int>(max_paths)) * 8 * 8;
    cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    *out = s;
    return CN_OK;
}

extern "C" void cn_sched_destroy(cn_sched* s) {
    if (!s) return;
    cudaDeviceSynchronize();
    cudaFree(s->d.mt);
    cudaFree(s->d.mt_idx);
    cudaFree(s->d.rtt);
    cudaFree(s->d.ecn);
    cudaFree(s->d.n_paths);
    delete s;
}

extern "C" int cn_sched_boards(cn_sched* s, double** d_rtt, double** d_ecn) {
    if (!s) return CN_E_INVALID;
    if (d_rtt) *d_rtt = s->d.rtt;
    if (d_ecn) *d_ecn = s->d.ecn;
    return s->max_paths;
}

extern "C" int cn_sched_select(cn_sched* s, int policy, int rtx_avoid_prev_path,
                               const uint32_t* d_conns, const uint32_t* d_offsets,
                               const int32_t* d_prev_paths, uint32_t n_groups,
                               uint32_t uniform_count, int32_t* d_out, void* stream) {
    if (!s || !d_out || policy < 0 || policy > 2) {
        set_error("cn_sched_select: bad arguments");
        return CN_E_INVALID;
    }
    if (!d_conns && n_groups > s->d.n_conns) {
        set_error("cn_sched_select: more groups than connections");
        return CN_E_INVALID;
    }
    if (n_groups == 0) return CN_OK;
    int smem = (2 * kMtN + s->max_paths) * 8 * 8;
    k_select<<<(n_groups + 7) / 8, 256, smem, static_cast<cudaStream_t>(stream)>>>(
        s->d, policy, rtx_avoid_prev_path, d_conns, d_offsets, d_prev_paths, d_out, n_groups,
        uniform_count);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_sched_draws(cn_sched* s, uint32_t conn, const uint64_t* d_ns, uint64_t count,
                              uint64_t* d_out, void* stream) {
    if (!s || conn >= s->d.n_conns || !d_out) {
        set_error("cn_sched_draws: bad arguments");
        return CN_E_INVALID;
    }
    k_draws<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(s->d, conn, d_ns ? 1 : 0, d_ns, d_out,
                                                             count);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_sched_record(cn_sched* s, const uint32_t* d_conn, const int32_t* d_path,
                               const int64_t* d_rtt, const uint8_t* d_ecn, const uint32_t* d_offsets,
                               uint32_t n_groups, void* stream) {
    if (!s) return CN_E_INVALID;
    if (n_groups == 0) return CN_OK;
    k_record<<<(n_groups + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        s->d, d_conn, d_path, d_rtt, d_ecn, d_offsets, n_groups);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}
