// common.cuh -- shared device helpers for the chunknet B200 hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "chunknet_b200.h"

#define CNB_STR2(x) #x
#define CNB_STR(x) CNB_STR2(x)

namespace cnb {

constexpr uint32_t kInf = 0xFFFFFFFFu;
constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kTomb = ~0ull - 1;

void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

#define CNB_CUDA(call)                                                  \
    do {                                                                \
        cudaError_t cnb_e_ = (call);                                    \
        if (cnb_e_ != cudaSuccess) return ::cnb::cuda_status(cnb_e_, #call); \
    } while (0)

// 64-bit mixer for table hashing (splitmix64 finaliser).
__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Open-addressing find-or-insert (linear probing, lock-free CAS).  Returns
// the slot or kInf when full; *inserted set for the unique winner.
__device__ inline uint32_t table_insert(unsigned long long* keys, uint32_t mask,
                                        uint64_t key, bool* inserted) {
    uint32_t h = static_cast<uint32_t>(mix64(key)) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&keys[h]);
        if (k == key) return h;
        if (k == kEmpty) {
            unsigned long long old = atomicCAS(&keys[h], kEmpty, key);
            if (old == kEmpty) {
                *inserted = true;
                return h;
            }
            if (old == key) return h;
        }
        h = (h + 1) & mask;
    }
    return kInf;
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization starts while its
// predecessor in the stream still runs; pdl_wait() blocks until that
// predecessor has completed and its writes are visible (a no-op without the
// attribute); pdl_launch() lets the successor start (the ack path's launch
// latencies overlap the kernel before).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// acquire / release and volatile accesses for the cross-block handshakes
// (decoupled look-back, published table values)
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__host__ __device__ inline uint32_t enc_hdr(uint32_t conn, uint32_t msg, uint32_t csn,
                                            uint32_t last, uint32_t rsvd) {
    return (conn << 24) | (msg << 17) | (csn << 9) | (last << 8) | rsvd;
}

}  // namespace cnb
