// rng.cuh -- device restatement of chunknet::RngStream (rng.hpp:29-60) and
// select_path (lb.cpp:7-27), shared by the scheduler and the tx engine.
// std::mt19937_64 with a warp-cooperative twist; libstdc++ 13
// uniform_int_distribution<uint64_t> (Lemire, uniform_int_dist.h:257-320).
#pragma once
#include <stdint.h>

#include "chunknet_b200.h"

namespace cnb {

constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xb5026f5aa96619e9ull;
constexpr uint64_t kUpper = ~0ull << 31, kLower = ~kUpper;

struct SchedDev;

struct SchedDev {
    uint32_t n_conns, max_paths;
    uint64_t* mt;        // [n_conns][312] raw state
    uint32_t* mt_idx;    // [n_conns] next word index (312 = twist needed)
    double* rtt;         // [n_conns][max_paths] PathScoreboard::rtt_
    double* ecn;         // [n_conns][max_paths] PathScoreboard::ecn_
    int32_t* n_paths;    // [n_conns]
};

__host__ __device__ inline uint64_t splitmix64_d(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline uint64_t fnv1a64_h(const char* s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = reinterpret_cast<const unsigned char*>(s); *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    return h;
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= z >> 43;
    return z;
}

// std::mt19937_64::seed (sequential recurrence), one thread per stream.
static __global__ void k_mt_seed(SchedDev d, uint64_t name_hash, uint64_t seed, uint64_t index0,
                          int indexed) {
    uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d.n_conns) return;
    uint64_t s = splitmix64_d(seed ^ name_hash);
    if (indexed) s = splitmix64_d(s + index0 + c);
    uint64_t* mt = d.mt + static_cast<uint64_t>(c) * kMtN;
    uint64_t prev = s;
    mt[0] = s;
    for (int i = 1; i < kMtN; ++i) {
        prev = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
        mt[i] = prev;
    }
    d.mt_idx[c] = kMtN;
}

// Warp-cooperative twist of a 312-word state held in shared memory.
__device__ __forceinline__ void warp_twist(uint64_t* mt, int lane) {
    // first half reads old words only; iterations are warp-uniform so the
    // read-before-write barrier is legal (no divergent __syncwarp)
    for (int k0 = 0; k0 < kMtM; k0 += 32) {
        const int k = k0 + lane;
        uint64_t v = 0;
        if (k < kMtM) {
            uint64_t y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
            v = mt[k + kMtM] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
        }
        __syncwarp();
        if (k < kMtM) mt[k] = v;
    }
    __syncwarp();
    // second half: mt[k+1] is old for k < 311 (mt[0] is new for k = 311),
    // mt[k-156] is new.  Read everything before writing.
    uint64_t vals[5];
    int cnt = 0;
    for (int k = kMtM + lane; k < kMtN; k += 32) {
        uint64_t nxt = mt[(k + 1) % kMtN];
        uint64_t y = (mt[k] & kUpper) | (nxt & kLower);
        vals[cnt++] = mt[k - kMtM] ^ (y >> 1) ^ ((y & 1) ? kMtA : 0);
    }
    __syncwarp();
    cnt = 0;
    for (int k = kMtM + lane; k < kMtN; k += 32) mt[k] = vals[cnt++];
    __syncwarp();
}

struct WarpRng {
    uint64_t* mt;   // shared [312] raw state
    uint64_t* out;  // shared [312] tempered outputs of the current block
    uint32_t idx;   // next output index (312 = exhausted)
};

__device__ __forceinline__ void refill(WarpRng& r, int lane) {
    warp_twist(r.mt, lane);
    for (int k = lane; k < kMtN; k += 32) r.out[k] = temper(r.mt[k]);
    __syncwarp();
    r.idx = 0;
}

__device__ __forceinline__ uint64_t next_u64_lane0(WarpRng& r, int lane) {
    // caller: whole warp converged; every lane gets the value
    if (r.idx >= kMtN) refill(r, lane);
    uint64_t v = r.out[r.idx];
    r.idx++;
    return v;
}

// libstdc++ uniform_int_distribution<uint64_t>(0, n-1) on a 64-bit engine
// (uniform_int_dist.h:296-320): Lemire _S_nd with a 128-bit product;
// n-1 == 2^64-1 takes the raw draw.  Whole warp, identical result per lane.
__device__ __forceinline__ uint64_t next_below_warp(WarpRng& r, uint64_t n, int lane) {
    uint64_t urange = n - 1;
    if (urange == ~0ull) return next_u64_lane0(r, lane);
    uint64_t range = urange + 1;
    uint64_t u = next_u64_lane0(r, lane);
    uint64_t lo = u * range, hi = __umul64hi(u, range);
    if (lo < range) {
        uint64_t threshold = (0 - range) % range;
        while (lo < threshold) {
            u = next_u64_lane0(r, lane);
            lo = u * range;
            hi = __umul64hi(u, range);
        }
    }
    return hi;
}

__device__ __forceinline__ int pick_p2(int a, int b, const double* s) {
    if (a > b) {
        int t = a;
        a = b;
        b = t;
    }
    return s[b] < s[a] ? b : a;
}

// select_path (lb.cpp:7-27) sequentially (warp-uniform), exact.
__device__ __forceinline__ int select_seq(WarpRng& r, int policy, int n, const double* s, int lane) {
    if (n == 1) return 0;
    if (policy == 0) return static_cast<int>(next_below_warp(r, static_cast<uint64_t>(n), lane));
    int a = static_cast<int>(next_below_warp(r, static_cast<uint64_t>(n), lane));
    int b = static_cast<int>(next_below_warp(r, static_cast<uint64_t>(n - 1), lane));
    if (b >= a) b++;
    return pick_p2(a, b, s);
}

// the SchedDev inside a cn_sched handle (defined in sched.cu)
SchedDev* sched_dev(cn_sched* s);

}  // namespace cnb
