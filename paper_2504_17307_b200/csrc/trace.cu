// trace.cu -- the reference's packet trace format on the device (sm_100a).
//
// experiment.cpp:18-40 (trace_line) writes one TSV line per network trace
// event (network.hpp:30-35 TraceEvent):
//     <t>\t<event>\t<link_id>\t<src>><dst>:<path_id>\t<csn>\t<kind>[,rtx][,ecn][,trim][,last]\n
// Here a batch of cn_trace_rec records is formatted in parallel: each
// thread renders its line (printf's %PRId64 / %d / %u digits), block sums
// of the line lengths are scanned, and every thread writes its bytes at its
// exclusive offset -- byte-identical to the reference's text, in record
// order.  Helpers turn receive-path records (cn_pkt_hdr deliveries,
// cn_ack_rec acks) into trace records.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace cnb {

constexpr int kTrThreads = 256;
constexpr int kTrLine = 160;  // trace_line's buffer (experiment.cpp:20) + flags

__device__ const char* const kEvName[] = {"deliver", "drop", "trim", "loss", "hdr_drop"};
__device__ const char* const kKindName[] = {"data", "ack", "nack", "credit", "rts", "rts_ack"};

struct LineBuf {
    char c[kTrLine];
    int n;
    __device__ void put(char x) {
        if (n < kTrLine) c[n] = x;
        ++n;
    }
    __device__ void str(const char* s) {
        while (*s) put(*s++);
    }
    __device__ void u64(unsigned long long v) {
        char d[20];
        int k = 0;
        do {
            d[k++] = static_cast<char>('0' + v % 10);
            v /= 10;
        } while (v);
        while (k) put(d[--k]);
    }
    __device__ void i64(long long v) {
        if (v < 0) {
            put('-');
            u64(static_cast<unsigned long long>(-(v + 1)) + 1);
        } else {
            u64(static_cast<unsigned long long>(v));
        }
    }
};

__device__ void render(const cn_trace_rec& r, LineBuf& b) {
    b.n = 0;
    b.i64(r.t);
    b.put('\t');
    b.str(r.event < 5 ? kEvName[r.event] : "?");
    b.put('\t');
    b.i64(r.link_id);
    b.put('\t');
    b.i64(r.src);
    b.put('>');
    b.i64(r.dst);
    b.put(':');
    b.i64(r.path_id);
    b.put('\t');
    b.u64(r.csn);
    b.put('\t');
    b.str(r.kind < 6 ? kKindName[r.kind] : "?");
    if (r.flags & CN_TRF_RTX) b.str(",rtx");
    if (r.flags & CN_TRF_ECN) b.str(",ecn");
    if (r.flags & CN_TRF_TRIM) b.str(",trim");
    if (r.flags & CN_TRF_LAST) b.str(",last");
    b.put('\n');
}

// block-wide exclusive sum (kTrThreads threads)
__device__ __forceinline__ unsigned long long block_excl(unsigned long long v, unsigned long long* ws,
                                                         unsigned long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long s = lane < kTrThreads / 32 ? ws[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kTrThreads / 32) ws[lane] = s;
    }
    __syncthreads();
    const unsigned long long before = (w ? ws[w - 1] : 0) + x - v;
    if (total) *total = ws[kTrThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(kTrThreads) k_trace_len(const cn_trace_rec* __restrict__ recs, uint64_t n,
                                                         unsigned long long* __restrict__ bsum) {
    __shared__ unsigned long long ws[kTrThreads / 32];
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(kTrThreads) + threadIdx.x;
    LineBuf b;
    b.n = 0;
    if (i < n) render(recs[i], b);
    unsigned long long tot = 0;
    block_excl(static_cast<unsigned long long>(b.n), ws, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of the block sums in place (one block); total -> *len
__global__ void __launch_bounds__(kTrThreads) k_trace_scan(unsigned long long* __restrict__ bsum, uint64_t nb,
                                                          uint64_t* __restrict__ len) {
    __shared__ unsigned long long ws[kTrThreads / 32];
    unsigned long long carry = 0;
    for (uint64_t b0 = 0; b0 < nb; b0 += kTrThreads) {
        const uint64_t k = b0 + threadIdx.x;
        const unsigned long long v = k < nb ? bsum[k] : 0;
        unsigned long long tot = 0;
        const unsigned long long ex = block_excl(v, ws, &tot);
        if (k < nb) bsum[k] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *len = carry;
}

__global__ void __launch_bounds__(kTrThreads) k_trace_write(const cn_trace_rec* __restrict__ recs, uint64_t n,
                                                           const unsigned long long* __restrict__ bsum,
                                                           char* __restrict__ out, uint64_t cap) {
    __shared__ unsigned long long ws[kTrThreads / 32];
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(kTrThreads) + threadIdx.x;
    LineBuf b;
    b.n = 0;
    if (i < n) render(recs[i], b);
    const unsigned long long off = bsum[blockIdx.x] + block_excl(static_cast<unsigned long long>(b.n), ws, nullptr);
    const int m = b.n < kTrLine ? b.n : kTrLine;
    if (off + m <= cap)
        for (int k = 0; k < m; ++k) out[off + k] = b.c[k];
}

__global__ void k_trace_from_packets(const cn_pkt_hdr* __restrict__ h, const int64_t* __restrict__ times,
                                     uint64_t n, int32_t event, int32_t link, cn_trace_rec* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const cn_pkt_hdr p = h[i];
    cn_trace_rec r;
    r.t = times ? times[i] : p.tx_time;
    r.link_id = link;
    r.src = p.src;
    r.dst = p.dst;
    r.path_id = p.path_id;
    r.csn = static_cast<uint8_t>((p.hdr >> 9) & 0xFF);
    r.event = static_cast<uint8_t>(event);
    r.kind = CN_PK_DATA;
    r.flags = static_cast<uint8_t>(((p.flags & CN_PKT_RTX) ? CN_TRF_RTX : 0) |
                                   ((p.flags & CN_PKT_ECN) ? CN_TRF_ECN : 0) |
                                   ((p.flags & CN_PKT_TRIMMED) ? CN_TRF_TRIM : 0) |
                                   (((p.hdr >> 8) & 1) ? CN_TRF_LAST : 0));
    out[i] = r;
}

__global__ void k_trace_from_acks(const cn_ack_rec* __restrict__ a, uint64_t n, int32_t event, int32_t link,
                                  cn_trace_rec* __restrict__ out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const cn_ack_rec k = a[i];
    cn_trace_rec r;
    r.t = k.aux;  // delivery time
    r.link_id = link;
    r.src = k.src;
    r.dst = k.dst;
    r.path_id = 0;  // send_ack leaves the packet's path_id at 0 (transport.cpp:763-792)
    r.csn = static_cast<uint8_t>((k.hdr >> 9) & 0xFF);
    r.event = static_cast<uint8_t>(event);
    r.kind = CN_PK_ACK;
    r.flags = 0;
    out[i] = r;
}

}  // namespace cnb

using namespace cnb;

extern "C" uint64_t cn_trace_tsv_bound(uint64_t n) { return n * kTrLine; }

extern "C" int cn_trace_format(const cn_trace_rec* d_recs, uint64_t n, char* d_out, uint64_t cap,
                               uint64_t* d_len, void* d_scratch, void* stream) {
    if ((n && (!d_recs || !d_scratch)) || !d_len) {
        set_error("cn_trace_format: null records, scratch or length");
        return CN_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t nb = (n + kTrThreads - 1) / kTrThreads;
    unsigned long long* bsum = static_cast<unsigned long long*>(d_scratch);
    if (nb) k_trace_len<<<static_cast<unsigned>(nb), kTrThreads, 0, s>>>(d_recs, n, bsum);
    k_trace_scan<<<1, kTrThreads, 0, s>>>(bsum, nb, d_len);
    if (nb && d_out) k_trace_write<<<static_cast<unsigned>(nb), kTrThreads, 0, s>>>(d_recs, n, bsum, d_out, cap);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" uint64_t cn_trace_scratch_bytes(uint64_t n) {
    return ((n + kTrThreads - 1) / kTrThreads + 1) * 8;
}

extern "C" int cn_trace_from_packets(const cn_pkt_hdr* d_hdrs, const int64_t* d_times, uint64_t n,
                                     int32_t event, int32_t link_id, cn_trace_rec* d_out, void* stream) {
    if (n && (!d_hdrs || !d_out)) return CN_E_INVALID;
    if (n)
        k_trace_from_packets<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_hdrs, d_times, n, event, link_id, d_out);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_trace_from_acks(const cn_ack_rec* d_acks, uint64_t n, int32_t event, int32_t link_id,
                                  cn_trace_rec* d_out, void* stream) {
    if (n && (!d_acks || !d_out)) return CN_E_INVALID;
    if (n)
        k_trace_from_acks<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_acks, n, event, link_id, d_out);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}
