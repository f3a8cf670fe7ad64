// coll.cu -- send-side packetization and the multi-GPU plumbing of the
// ring collectives (sm_100a).
//
//   cn_packetize   Transport::send_chunk's per-packet loop (src/transport.cpp
//                  :433-494) for every chunk of a message at once: the 64-B
//                  header records (cn_pkt_hdr) a receiver consumes.  Chunking
//                  is DefaultPolicy::on_chunk_size (policy.hpp:75-78):
//                  min(remaining, chunk_bytes); packets of max_payload bytes.
//   cn_ipc_*       CUDA IPC mappings of a peer rank's buffers (NVLink P2P).
//   cn_flag_*      device-side progress flags between neighbouring ranks:
//                  a signal is a system-scope release store into the peer's
//                  memory, a wait is a bounded acquire spin in the local one
//                  (each rank owns its GPU, so waiting kernels never share
//                  an SM with the kernel they wait for).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>

#include "common.cuh"

namespace cnb {

__global__ void k_packetize(cn_pkt_hdr* __restrict__ out, uint64_t len, uint32_t cb, uint32_t max_pl,
                            uint32_t ppc, uint64_t nchunks, uint64_t n_pkts, int32_t src, int32_t dst,
                            uint32_t conn_id, uint32_t msg_id, uint64_t msg_seq, uint64_t tag,
                            int64_t tx_time, const int32_t* __restrict__ paths, int32_t path0,
                            uint32_t flags) {
    uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (p >= n_pkts) return;
    uint64_t c = p / ppc;
    uint32_t s = static_cast<uint32_t>(p % ppc);
    if (c >= nchunks) {  // only the last chunk can be short: fold the overflow into it
        c = nchunks - 1;
        s = static_cast<uint32_t>(p - c * ppc);
    }
    const uint64_t off = c * cb;
    const uint64_t rem = len - off;
    const uint32_t clen = rem < cb ? static_cast<uint32_t>(rem) : cb;
    const uint32_t po = s * max_pl;
    const uint32_t pl = clen - po < max_pl ? clen - po : max_pl;
    cn_pkt_hdr h;
    h.src = src;
    h.dst = dst;
    h.path_id = paths ? paths[c] : path0;
    h.hdr = enc_hdr(conn_id & 0xFF, msg_id & 0x7F, static_cast<uint32_t>(c & 0xFF),
                    c + 1 == nchunks ? 1u : 0u, 0);
    h.chunk_offset = off;
    h.chunk_len = clen;
    h.payload_len = static_cast<uint16_t>(pl);
    h.seq_in_chunk = static_cast<uint8_t>(s);
    h.flags = static_cast<uint8_t>(flags);
    h.tx_time = tx_time;
    h.msg_seq = msg_seq;
    h.msg_tag = tag;
    h.msg_len = len;
    out[p] = h;
}

__global__ void k_flag_signal(unsigned long long* a, unsigned long long* b, unsigned long long v) {
    __threadfence_system();  // data written by this stream's earlier kernels
    if (a) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
    if (b) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(b), "l"(v) : "memory");
}

__global__ void k_flag_wait(const unsigned long long* a, const unsigned long long* b,
                            unsigned long long v, unsigned long long max_spins, unsigned int* err) {
    unsigned long long spins = 0;
    for (;;) {
        unsigned long long x = ~0ull, y = ~0ull;
        if (a) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(a) : "memory");
        if (b) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(y) : "l"(b) : "memory");
        if (x >= v && y >= v) break;
        if (++spins > max_spins) {
            atomicOr(err, 1u);
            break;
        }
        __nanosleep(100);
    }
    __threadfence_system();
}

__global__ void k_flag_post(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

__global__ void k_flag_wait_signal(const unsigned long long* wa, unsigned long long va,
                                   const unsigned long long* wb, unsigned long long vb, unsigned long long* sg,
                                   unsigned long long vs, unsigned long long max_spins, unsigned int* err) {
    unsigned long long spins = 0;
    for (;;) {
        unsigned long long x = ~0ull, y = ~0ull;
        if (wa) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(wa) : "memory");
        if (wb) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(y) : "l"(wb) : "memory");
        if (x >= va && y >= vb) break;
        if (++spins > max_spins) {
            atomicOr(err, 1u);
            break;
        }
        __nanosleep(100);
    }
    if (sg)  // a consumption notice: it publishes nothing this stream wrote
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(sg), "l"(vs) : "memory");
    else
        __threadfence_system();
}

__device__ __forceinline__ long long ctr_target(const unsigned long long* it, unsigned long long per_iter,
                                                long long off) {
    return static_cast<long long>(*reinterpret_cast<const volatile unsigned long long*>(it) * per_iter) + off;
}

__global__ void k_ctr_wait(const unsigned long long* f, const unsigned long long* it, unsigned long long per_iter,
                           long long off, unsigned long long max_spins, unsigned int* err) {
    const long long v = ctr_target(it, per_iter, off);
    if (v <= 0) return;
    unsigned long long spins = 0;
    for (;;) {
        unsigned long long x;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
        if (static_cast<long long>(x) >= v) break;
        if (++spins > max_spins) {
            atomicOr(err, 1u);
            break;
        }
        __nanosleep(64);
    }
    __threadfence_system();
}

__global__ void k_ctr_signal(unsigned long long* f, const unsigned long long* it, unsigned long long per_iter,
                             long long off) {
    const long long v = ctr_target(it, per_iter, off);
    __threadfence_system();  // everything this stream wrote before
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(static_cast<unsigned long long>(v))
                 : "memory");
}

__global__ void k_ctr_advance(unsigned long long* it) { *it += 1; }

// SM-driven bulk copy (16-byte vectors, 4 in flight per thread): with a peer
// destination these are NVLink posted writes, a second "wire" beside the
// copy engines.
__global__ void __launch_bounds__(512) k_copy_sm(int4* __restrict__ dst, const int4* __restrict__ src,
                                                 uint64_t nv, unsigned long long* flag, unsigned long long value,
                                                 unsigned int* ctr) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {
        int4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
             e = __ldcs(src + i + 3 * stride);
        dst[i] = a;
        dst[i + stride] = b;
        dst[i + 2 * stride] = c;
        dst[i + 3 * stride] = e;
    }
    for (; i < nv; i += stride) dst[i] = __ldcs(src + i);
    if (flag) {  // the last block to finish raises the flag (its peers' stores fenced first)
        __shared__ bool last;
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence_system();
            *ctr = 0;  // for the next copy on this stream
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
        }
    }
}

}  // namespace cnb

using namespace cnb;

// Progress kernels run at the greatest stream priority: they are single
// threads that gate copy-engine transfers, so they must not queue behind the
// receive path's short-lived scatter blocks for an SM slot.
template <typename... KArgs, typename... Args>
static cudaError_t launch_hi(void (*k)(KArgs...), void* stream, Args... args) {
    static int prio = [] {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        return greatest;
    }();
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = prio;
    lc.gridDim = dim3(1);
    lc.blockDim = dim3(1);
    lc.stream = static_cast<cudaStream_t>(stream);
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, k, args...);
}

extern "C" int cn_ctr_wait(const unsigned long long* d_flag, const unsigned long long* d_iter, uint64_t per_iter,
                           int64_t offset, uint64_t max_spins, unsigned int* d_err, void* stream) {
    if (!d_flag || !d_iter || !d_err) return CN_E_INVALID;
    CNB_CUDA(launch_hi(k_ctr_wait, stream, d_flag, d_iter, static_cast<unsigned long long>(per_iter),
                       static_cast<long long>(offset), static_cast<unsigned long long>(max_spins), d_err));
    return CN_OK;
}

extern "C" int cn_ctr_signal(unsigned long long* d_flag, const unsigned long long* d_iter, uint64_t per_iter,
                             int64_t offset, void* stream) {
    if (!d_flag || !d_iter) return CN_E_INVALID;
    CNB_CUDA(launch_hi(k_ctr_signal, stream, d_flag, d_iter, static_cast<unsigned long long>(per_iter),
                       static_cast<long long>(offset)));
    return CN_OK;
}

extern "C" int cn_ctr_advance(unsigned long long* d_iter, void* stream) {
    if (!d_iter) return CN_E_INVALID;
    CNB_CUDA(launch_hi(k_ctr_advance, stream, d_iter));
    return CN_OK;
}

extern "C" int cn_copy_sm(void* d_dst, const void* d_src, uint64_t bytes, uint32_t blocks, void* stream) {
    if (!bytes) return CN_OK;
    if (!d_dst || !d_src || ((reinterpret_cast<uintptr_t>(d_dst) | reinterpret_cast<uintptr_t>(d_src) | bytes) & 15)) {
        set_error("cn_copy_sm: pointers and size must be 16-byte aligned");
        return CN_E_INVALID;
    }
    k_copy_sm<<<blocks ? blocks : 148, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<int4*>(d_dst), static_cast<const int4*>(d_src), bytes >> 4, nullptr, 0, nullptr);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_copy_sm_signal(void* d_dst, const void* d_src, uint64_t bytes, uint32_t blocks,
                                 unsigned long long* d_flag, uint64_t value, unsigned int* d_ctr, void* stream) {
    if (!d_dst || !d_src || !d_flag || !d_ctr || !bytes ||
        ((reinterpret_cast<uintptr_t>(d_dst) | reinterpret_cast<uintptr_t>(d_src) | bytes) & 15)) {
        set_error("cn_copy_sm_signal: non-empty, 16-byte aligned copy and a flag and counter required");
        return CN_E_INVALID;
    }
    k_copy_sm<<<blocks ? blocks : 148, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<int4*>(d_dst), static_cast<const int4*>(d_src), bytes >> 4, d_flag, value, d_ctr);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_copy_async(void* d_dst, const void* d_src, uint64_t bytes, void* stream) {
    if (!bytes) return CN_OK;
    if (!d_dst || !d_src) return CN_E_INVALID;
    CNB_CUDA(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
    return CN_OK;
}

extern "C" uint64_t cn_packet_count(uint64_t len, uint32_t chunk_bytes, uint32_t max_payload) {
    if (!len || !chunk_bytes || !max_payload) return 0;
    uint64_t nch = (len + chunk_bytes - 1) / chunk_bytes;
    uint32_t ppc = (chunk_bytes + max_payload - 1) / max_payload;
    uint64_t last = len - (nch - 1) * chunk_bytes;
    return (nch - 1) * ppc + (last + max_payload - 1) / max_payload;
}

extern "C" int cn_packetize(const cn_packetize_args* a, cn_pkt_hdr* d_out, void* stream) {
    if (!a || !d_out || a->len == 0 || a->chunk_bytes == 0) {
        set_error("cn_packetize: empty message or bad arguments (send_message throws, transport.cpp:145)");
        return CN_E_INVALID;
    }
    if (a->msg_id > 127) {
        set_error("cn_packetize: msg_id must fit 7 bits");
        return CN_E_FIELD_RANGE;
    }
    uint32_t max_pl = a->max_payload ? a->max_payload : CN_MAX_PAYLOAD;
    uint32_t ppc = (a->chunk_bytes + max_pl - 1) / max_pl;
    if (ppc > CN_MAX_PKTS_PER_CHUNK) {
        set_error("cn_packetize: more than 32 packets per chunk");
        return CN_E_INVALID;
    }
    uint64_t nch = (a->len + a->chunk_bytes - 1) / a->chunk_bytes;
    uint64_t n = cn_packet_count(a->len, a->chunk_bytes, max_pl);
    k_packetize<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_out, a->len, a->chunk_bytes, max_pl, ppc, nch, n, a->src, a->dst, a->conn_id, a->msg_id,
        a->msg_seq, a->tag, a->tx_time, a->d_chunk_paths, a->path, a->is_rtx ? CN_PKT_RTX : 0);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_dev_alloc(uint64_t bytes, void** d_ptr) {
    if (!d_ptr || !bytes) return CN_E_INVALID;
    CNB_CUDA(cudaMalloc(d_ptr, bytes));
    CNB_CUDA(cudaMemset(*d_ptr, 0, bytes));
    return CN_OK;
}

extern "C" int cn_dev_free(void* d_ptr) {
    if (d_ptr) CNB_CUDA(cudaFree(d_ptr));
    return CN_OK;
}

extern "C" int cn_ipc_get_handle(void* d_ptr, void* out64) {
    if (!d_ptr || !out64) return CN_E_INVALID;
    cudaIpcMemHandle_t h;
    CNB_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
    memcpy(out64, &h, sizeof h);
    return CN_OK;
}

extern "C" int cn_ipc_open(const void* handle64, void** d_ptr) {
    if (!handle64 || !d_ptr) return CN_E_INVALID;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    CNB_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return CN_OK;
}

extern "C" int cn_ipc_close(void* d_ptr) {
    if (!d_ptr) return CN_E_INVALID;
    CNB_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return CN_OK;
}

extern "C" int cn_flag_signal(unsigned long long* d_a, unsigned long long* d_b, uint64_t value,
                              void* stream) {
    k_flag_signal<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, value);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_flag_post(unsigned long long* d_a, uint64_t value, void* stream) {
    if (!d_a) return CN_E_INVALID;
    k_flag_post<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_a, value);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_flag_wait_signal(const unsigned long long* d_wa, uint64_t va, const unsigned long long* d_wb,
                                   uint64_t vb, unsigned long long* d_s, uint64_t vs, uint64_t max_spins,
                                   unsigned int* d_err, void* stream) {
    if (!d_err) return CN_E_INVALID;
    k_flag_wait_signal<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_wa, va, d_wb, vb, d_s, vs, max_spins,
                                                                        d_err);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_flag_wait(const unsigned long long* d_a, const unsigned long long* d_b,
                            uint64_t value, uint64_t max_spins, unsigned int* d_err, void* stream) {
    if (!d_err) return CN_E_INVALID;
    k_flag_wait<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, value, max_spins, d_err);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}
