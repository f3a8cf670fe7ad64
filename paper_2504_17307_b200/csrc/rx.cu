// rx.cu -- device-resident receive path of the chunknet transport (sm_100a).
//
// Replaces, for a batch of delivered data packets in arrival order, the
// reference's packet-at-a-time receive path (/root/reference/proj):
//   Transport::handle_packet / rconn_at   src/transport.cpp:546-594
//   Transport::handle_data                src/transport.cpp:596-688
//   Transport::accept_payload             src/transport.cpp:719-730
//   Transport::chunk_completed            src/transport.cpp:732-761
//   Transport::send_ack                   src/transport.cpp:763-792
//   Transport::maybe_deliver              src/transport.cpp:794-803
//
// Batched, data-parallel restatement: every packet i of a
// batch gets the time t = i+1 (0 = an earlier batch).  For every chunk
//   first[c][s] = first arrival time of packet s of chunk c   (atomicMin)
//   cpl[c]      = max_s first[c][s]  (time the chunk completes; INF if not)
//   pmax[c]     = max(cpl[cum0..c])  (prefix max per message)
// so that the cumulative cursor after packet i is #{c : pmax[c] <= t(i)}.
// Each packet's ack (if any) is then an independent snapshot: cum, the
// 128-bit SACK {cpl[cum+j] <= t}, and the echo of chunk
// cum + uint8(cause - uint8(cum)).  Ack records are compacted in arrival
// order with a two-level scan.  The payload scatter (accept_payload) is a
// warp-cooperative 16-byte vectorised copy of each first-arriving packet.
//
// Kernels per batch: classify -> alloc -> mark -> scan -> decide ->
// tilescan -> work (copy + ack + completion) -> finalize.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <new>
#include <string>

#include "common.cuh"

namespace cnb {

struct GenState {
    uint64_t len, tag, seq, chunk_base, buf_off, bytes;
    uint32_t nchunks, cum, n_init, rc, msg_id, epoch, max_touched, deliver_t;
};

struct RxCtl {
    unsigned long long pool_top;
    unsigned long long arena_top;
    uint32_t n_touched;
    uint32_t pad;
};

enum : uint32_t { CF_INIT = 1, CF_COMPLETE = 2, CF_ECN = 4, CF_RTX = 8 };
enum : uint8_t { PC_STALE = 1, PC_ACK = 2, PC_COPY = 4, PC_DELIVER = 8 };
constexpr uint32_t kStale = kInf;      // p_gen marker: stale before the batch
constexpr uint32_t kErr = kInf - 1;    // p_gen marker: rejected packet
constexpr int kTile = 256;             // decide / tilescan granularity

struct RxDev {
    uint32_t cb, max_pl, ppc, conn_mask, gen_mask, carry;
    uint64_t pool_cap, arena_cap;
    unsigned long long* rc_key;
    unsigned long long* rc_done;  // [conns*128] completed_seq
    unsigned long long* gen_key;
    GenState* gen;
    uint32_t* touched;
    uint32_t* c_first;  // [pool*ppc] batch scratch
    uint32_t* c_seen;   // [pool] persistent packet bitmask
    uint32_t* c_flags;  // [pool] persistent CF_*
    int64_t* c_txt;     // [pool] persistent echo tx_time
    int32_t* c_path;    // [pool] persistent echo path
    uint32_t* c_init;   // [pool] batch scratch: first arrival time
    uint32_t* c_cpl;    // [pool] batch scratch: completion time
    uint32_t* c_pmax;   // [pool] batch scratch: prefix max of c_cpl
    uint32_t* p_gen;    // [batch]
    uint32_t* p_pos;    // [batch] local ack pos | local completion pos << 16
    uint8_t* p_cls;     // [batch]
    uint32_t* tile_cnt; // [tiles*2]
    uint32_t* tile_off; // [tiles*2]
    RxCtl* ctl;
    uint8_t* arena;
};

__device__ __forceinline__ uint32_t chunk_len_of(const RxDev& d, uint64_t len, uint64_t c) {
    uint64_t rem = len - c * d.cb;
    return rem < d.cb ? static_cast<uint32_t>(rem) : d.cb;
}
__device__ __forceinline__ uint32_t pkts_of(const RxDev& d, uint32_t clen) {
    return (clen + d.max_pl - 1) / d.max_pl;
}

// ------------------------------------------------------------------ K1
// rconn_at (transport.cpp:546-563) + the stale-generation test
// (transport.cpp:602) + message-generation discovery (:620-626).
__global__ void k_classify(RxDev d, const cn_pkt_hdr* __restrict__ hdrs, uint32_t n,
                           uint32_t epoch, cn_rx_result* res) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const cn_pkt_hdr h = hdrs[i];
    uint32_t status = 0;
    if (h.flags & CN_PKT_TRIMMED) status |= CN_RXF_UNSUPPORTED;  // trim mode: DESIGN.md §7
    uint32_t g = kErr;
    if (static_cast<uint32_t>(h.src) >= (1u << 24) || static_cast<uint32_t>(h.dst) >= (1u << 24) ||
        h.msg_seq >= (1ull << 40) || h.msg_seq == 0) {
        status |= CN_RXF_UNSUPPORTED;
    } else {
        uint32_t conn = h.hdr >> 24, mid = (h.hdr >> 17) & 0x7F;
        uint64_t rkey = (static_cast<uint64_t>(h.dst) << 32) |
                        (static_cast<uint64_t>(h.src) << 8) | conn;
        bool ins = false;
        uint32_t rc = table_insert(d.rc_key, d.conn_mask, rkey, &ins);
        if (rc == kInf) {
            status |= CN_RXF_CAPACITY;
        } else if (h.msg_seq <= d.rc_done[rc * 128 + mid]) {
            g = kStale;
        } else {
            bool gins = false;
            g = table_insert(d.gen_key, d.gen_mask, (static_cast<uint64_t>(rc) << 40) | h.msg_seq,
                             &gins);
            if (g == kInf) {
                g = kErr;
                status |= CN_RXF_CAPACITY;
            } else {
                GenState* G = &d.gen[g];
                if (gins) {
                    G->len = h.msg_len;
                    G->tag = h.msg_tag;
                    G->seq = h.msg_seq;
                    G->chunk_base = kEmpty;
                    G->buf_off = 0;
                    G->bytes = 0;
                    G->nchunks = 0;
                    G->cum = 0;
                    G->n_init = 0;
                    G->rc = rc;
                    G->msg_id = mid;
                }
                if (atomicExch(&G->epoch, epoch) != epoch) {
                    uint32_t k = atomicAdd(&d.ctl->n_touched, 1u);
                    d.touched[k] = g;
                }
            }
        }
    }
    d.p_gen[i] = g;
    if (status) atomicOr(&res->status, status);
}

// ------------------------------------------------------------------ K2
// Lazy MsgRecv init (transport.cpp:620-626): chunk state and the message
// buffer (accept_payload's buf.resize, :723) come from bump pools.
__global__ void k_alloc(RxDev d, cn_rx_result* res) {
    uint32_t nt = d.ctl->n_touched;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nt;
         k += gridDim.x * blockDim.x) {
        GenState* G = &d.gen[d.touched[k]];
        if (G->chunk_base == kEmpty) {
            uint64_t nc = (G->len + d.cb - 1) / d.cb;
            uint32_t st = 0;
            if (G->len == 0 || nc >= (1ull << 31)) st = CN_RXF_UNSUPPORTED;
            unsigned long long base = 0, boff = 0;
            if (!st) {
                base = atomicAdd(&d.ctl->pool_top, static_cast<unsigned long long>(nc));
                if (base + nc > d.pool_cap) st = CN_RXF_CAPACITY;
            }
            if (!st && d.carry) {
                unsigned long long need = (G->len + 15) & ~15ull;
                boff = atomicAdd(&d.ctl->arena_top, need);
                if (boff + need > d.arena_cap) st = CN_RXF_CAPACITY;
            }
            if (st) {
                atomicOr(&res->status, st);
                G->nchunks = 0;  // every packet of this message is rejected
                G->chunk_base = 0;
            } else {
                G->chunk_base = base;
                G->buf_off = boff;
                G->nchunks = static_cast<uint32_t>(nc);
            }
        }
        G->max_touched = G->n_init;
        G->deliver_t = kInf;
    }
}

// ------------------------------------------------------------------ K3
// Per-packet bit (transport.cpp:676-683) as first-arrival times, chunk init
// (:639-645), and the unwrapped chunk vector size (:636-637).
__global__ void k_mark(RxDev d, const cn_pkt_hdr* __restrict__ hdrs, uint32_t n,
                       cn_rx_result* res) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t g = i < n ? d.p_gen[i] : kErr;
    uint32_t touched = 0;
    if (g < kErr) {
        const cn_pkt_hdr h = hdrs[i];
        const GenState* G = &d.gen[g];
        uint64_t nch = G->nchunks;
        uint64_t c = h.chunk_offset / d.cb;
        uint32_t s = h.seq_in_chunk;
        bool bad = nch == 0 || (h.chunk_offset % d.cb) != 0 || c >= nch || h.msg_len != G->len;
        if (!bad) {
            uint32_t clen = chunk_len_of(d, G->len, c);
            uint32_t exp = pkts_of(d, clen);
            uint32_t pl = clen - s * d.max_pl;
            pl = pl < d.max_pl ? pl : d.max_pl;
            bad = ((h.hdr >> 9) & 0xFF) != (c & 0xFF) || h.chunk_len != clen || s >= exp ||
                  h.payload_len != pl || ((h.hdr >> 8) & 1) != (c + 1 == nch ? 1u : 0u);
        }
        if (bad) {
            atomicOr(&res->status, CN_RXF_UNSUPPORTED);
            d.p_gen[i] = kErr;
        } else {
            uint64_t e = G->chunk_base + c;
            uint32_t t = i + 1;
            uint32_t fl = d.c_flags[e];
            if (!(fl & CF_COMPLETE) && !((d.c_seen[e] >> s) & 1u))
                atomicMin(&d.c_first[e * d.ppc + s], t);
            if (!(fl & CF_INIT)) atomicMin(&d.c_init[e], t);
            touched = static_cast<uint32_t>(c) + 1;
        }
    }
    // warp-aggregated atomicMax of the chunk vector size per message
    unsigned peers = __match_any_sync(__activemask(), g);
    int lane = threadIdx.x & 31;
    int leader = __ffs(peers) - 1;
    uint32_t gm = 0;
    for (unsigned p = peers; p; p &= p - 1) {
        uint32_t v = __shfl_sync(peers, touched, __ffs(p) - 1);
        gm = gm > v ? gm : v;
    }
    if (lane == leader && g < kErr && gm) atomicMax(&d.gen[g].max_touched, gm);
}

// block-wide inclusive max-scan over 256 threads
__device__ __forceinline__ uint32_t block_scan_max(uint32_t v, uint32_t* smem) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = v > x ? v : x;
    }
    if (lane == 31) smem[w] = v;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < (blockDim.x >> 5) ? smem[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = x > y ? x : y;
        }
        smem[lane] = x;
    }
    __syncthreads();
    if (w > 0) {
        uint32_t p = smem[w - 1];
        v = v > p ? v : p;
    }
    __syncthreads();
    return v;
}

// ------------------------------------------------------------------ K4
// chunk completion times and the cumulative-cursor prefix max
// (chunk_completed's `while (chunks[cum].complete) ++cum`, :736-738).
constexpr int kScanItems = 8;
__global__ void __launch_bounds__(256) k_scan(RxDev d) {
    __shared__ uint32_t smem[32];
    __shared__ uint32_t carry_s;
    uint32_t nt = d.ctl->n_touched;
    for (uint32_t k = blockIdx.x; k < nt; k += gridDim.x) {
        GenState* G = &d.gen[d.touched[k]];
        uint32_t lo = G->cum, hi = G->max_touched;
        uint64_t base = G->chunk_base;
        if (threadIdx.x == 0) {
            G->n_init = hi;
            carry_s = 0;
        }
        __syncthreads();
        for (uint32_t t0 = lo; t0 < hi; t0 += 256 * kScanItems) {
            uint32_t v[kScanItems];
            uint32_t run = 0;
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) {
                uint32_t c = t0 + threadIdx.x * kScanItems + j;
                uint32_t cpl = 0;
                if (c < hi) {
                    uint64_t e = base + c;
                    if (!(d.c_flags[e] & CF_COMPLETE)) {
                        uint32_t exp = pkts_of(d, chunk_len_of(d, G->len, c));
                        uint32_t seen = d.c_seen[e];
                        for (uint32_t s = 0; s < exp; ++s) {
                            if ((seen >> s) & 1u) continue;
                            uint32_t f = d.c_first[e * d.ppc + s];
                            cpl = cpl > f ? cpl : f;
                        }
                    }
                    d.c_cpl[e] = cpl;
                }
                run = run > cpl ? run : cpl;
                v[j] = run;
            }
            uint32_t incl = block_scan_max(run, smem);
            // exclusive prefix for this thread = max of previous threads
            uint32_t prev = __shfl_up_sync(0xffffffffu, incl, 1);
            if ((threadIdx.x & 31) == 0) prev = (threadIdx.x >> 5) ? smem[(threadIdx.x >> 5) - 1] : 0;
            uint32_t carry = carry_s;
            uint32_t pre = prev > carry ? prev : carry;
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) {
                uint32_t c = t0 + threadIdx.x * kScanItems + j;
                if (c < hi) d.c_pmax[base + c] = v[j] > pre ? v[j] : pre;
            }
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) carry_s = incl > carry ? incl : carry;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            uint32_t dt = kInf;
            if (G->nchunks && hi == G->nchunks) dt = d.c_pmax[base + hi - 1];
            G->deliver_t = dt;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t pmax_at(const RxDev& d, const GenState& G, uint64_t x) {
    if (x < G.cum) return 0;
    if (x >= G.n_init) return kInf;
    return d.c_pmax[G.chunk_base + x];
}

// ------------------------------------------------------------------ K5
// What the reference does with each packet (handle_data branches) and where
// its ack / completion lands in the ordered output streams.
__global__ void __launch_bounds__(kTile) k_decide(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                                  uint32_t n, cn_rx_result* res) {
    __shared__ uint32_t wsum[kTile / 32];
    uint32_t i = blockIdx.x * kTile + threadIdx.x;
    uint8_t cls = 0;
    uint32_t st = 0;
    if (i < n) {
        uint32_t g = d.p_gen[i];
        uint32_t t = i + 1;
        if (g == kStale) {
            cls = PC_STALE;  // transport.cpp:602-615
        } else if (g != kErr) {
            const GenState G = d.gen[g];
            if (t > G.deliver_t) {
                cls = PC_STALE;
            } else {
                const cn_pkt_hdr h = hdrs[i];
                uint64_t c = h.chunk_offset / d.cb;
                uint32_t s = h.seq_in_chunk;
                uint64_t e = G.chunk_base + c;
                uint32_t cpl = (d.c_flags[e] & CF_COMPLETE) ? 0 : d.c_cpl[e];
                if (cpl < t) {
                    cls = PC_ACK;  // complete chunk (:651-655) or behind cursor (:631-634)
                } else if (cpl == t) {
                    cls = PC_ACK | PC_COPY;  // completes its chunk (:686-687)
                    if (t == G.deliver_t) cls |= PC_DELIVER;
                } else if (!((d.c_seen[e] >> s) & 1u) && d.c_first[e * d.ppc + s] == t) {
                    cls = PC_COPY;  // new packet, chunk still open: silent
                }
                // The reference unwraps the 8-bit csn against the cursor
                // (:629-636); check it names chunk c (no aliasing).
                if (pmax_at(d, G, c) < t) {
                    if (pmax_at(d, G, c + 128) < t) st |= CN_RXF_ALIAS;
                } else if (c >= 128 && pmax_at(d, G, c - 128) >= t) {
                    st |= CN_RXF_ALIAS;
                }
            }
        }
        d.p_cls[i] = cls;
    }
    if (st) atomicOr(&res->status, st);
    // two exclusive counts (acks, completions) packed in one 32-bit scan
    uint32_t v = ((cls & (PC_STALE | PC_ACK)) ? 1u : 0u) | ((cls & PC_DELIVER) ? 1u << 16 : 0u);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < kTile / 32 ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < kTile / 32) wsum[lane] = x;
    }
    __syncthreads();
    uint32_t excl = incl - v + (w ? wsum[w - 1] : 0);
    if (i < n) d.p_pos[i] = excl;
    if (threadIdx.x == kTile - 1) {
        uint32_t tot = wsum[kTile / 32 - 1];
        d.tile_cnt[blockIdx.x * 2 + 0] = tot & 0xFFFFu;
        d.tile_cnt[blockIdx.x * 2 + 1] = tot >> 16;
    }
}

// ------------------------------------------------------------------ K5b
__global__ void __launch_bounds__(1024) k_tilescan(RxDev d, uint32_t tiles, uint32_t max_acks,
                                                   uint32_t max_cpls, cn_rx_result* res) {
    __shared__ uint32_t wsum[2][32];
    __shared__ uint32_t carry[2];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < 2) carry[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t t0 = 0; t0 < tiles; t0 += 1024) {
        uint32_t t = t0 + threadIdx.x;
        uint32_t a = t < tiles ? d.tile_cnt[2 * t] : 0;
        uint32_t b = t < tiles ? d.tile_cnt[2 * t + 1] : 0;
        uint32_t ia = a, ib = b;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t x = __shfl_up_sync(0xffffffffu, ia, o);
            uint32_t y = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += x;
                ib += y;
            }
        }
        if (lane == 31) {
            wsum[0][w] = ia;
            wsum[1][w] = ib;
        }
        __syncthreads();
        if (w == 0) {
            uint32_t x = wsum[0][lane], y = wsum[1][lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t p = __shfl_up_sync(0xffffffffu, x, o);
                uint32_t q = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) {
                    x += p;
                    y += q;
                }
            }
            wsum[0][lane] = x;
            wsum[1][lane] = y;
        }
        __syncthreads();
        uint32_t ea = carry[0] + ia - a + (w ? wsum[0][w - 1] : 0);
        uint32_t eb = carry[1] + ib - b + (w ? wsum[1][w - 1] : 0);
        if (t < tiles) {
            d.tile_off[2 * t] = ea;
            d.tile_off[2 * t + 1] = eb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry[0] += wsum[0][31];
            carry[1] += wsum[1][31];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        res->n_acks = carry[0];
        res->n_completions = carry[1];
        if (carry[0] > max_acks || carry[1] > max_cpls) atomicOr(&res->status, CN_RXF_CAPACITY);
    }
}

// warp-cooperative scatter copy (accept_payload's memcpy, :728-729)
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                          uint32_t len, int lane) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        uint32_t nv = len >> 4;
        for (uint32_t v0 = 0; v0 < nv; v0 += 32 * 8) {
            int4 r[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t v = v0 + k * 32 + lane;
                if (v < nv) r[k] = __ldcs(s4 + v);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t v = v0 + k * 32 + lane;
                if (v < nv) d4[v] = r[k];
            }
        }
        for (uint32_t b = (nv << 4) + lane; b < len; b += 32) dst[b] = src[b];
    } else {
        for (uint32_t b = lane; b < len; b += 32) dst[b] = src[b];
    }
}

// ------------------------------------------------------------------ K6
// One warp per packet: payload scatter, ack snapshot (send_ack :763-792 or
// the stale re-ack :602-615), completion record (maybe_deliver :794-803).
__global__ void __launch_bounds__(256) k_work(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                              const uint8_t* __restrict__ payload, uint64_t stride,
                                              uint32_t n, cn_ack_rec* __restrict__ acks,
                                              uint32_t max_acks, cn_completion* __restrict__ cpls,
                                              uint32_t max_cpls, cn_rx_result* res) {
    uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    uint8_t cls = d.p_cls[i];
    if (!cls) return;
    const cn_pkt_hdr h = hdrs[i];
    uint32_t t = i + 1;
    uint32_t tile = i / kTile;
    uint32_t pos = d.p_pos[i];
    uint32_t csn = (h.hdr >> 9) & 0xFF;

    if (cls & PC_STALE) {
        uint32_t a = d.tile_off[2 * tile] + (pos & 0xFFFFu);
        if (lane == 0 && a < max_acks) {
            cn_ack_rec r;
            memset(&r, 0, sizeof r);
            r.src = h.dst;
            r.dst = h.src;
            r.hdr = h.hdr;
            r.cum_csn = static_cast<uint8_t>(csn);
            r.flags = CN_ACK_CUM_VALID;
            r.pkt_index = i;
            r.msg_seq = h.msg_seq;
            acks[a] = r;
        }
        return;
    }
    const uint32_t g = d.p_gen[i];
    const GenState G = d.gen[g];
    if ((cls & PC_COPY) && d.carry) {
        uint64_t off = h.chunk_offset + static_cast<uint64_t>(h.seq_in_chunk) * d.max_pl;
        warp_copy(d.arena + G.buf_off + off, payload + static_cast<uint64_t>(i) * stride,
                  h.payload_len, lane);
    }
    if (cls & PC_ACK) {
        // cum after this packet: first x in [cum0, n_init) with pmax[x] > t
        uint32_t lo = G.cum, hi = G.n_init;
        const uint32_t* pm = d.c_pmax + G.chunk_base;
        while (hi - lo > 32) {
            uint32_t step = (hi - lo + 31) / 32;
            uint32_t p = lo + (lane + 1) * step - 1;
            bool ok = p < hi && pm[p] <= t;
            uint32_t k = __popc(__ballot_sync(0xffffffffu, ok));
            lo += k * step;
            hi = hi < lo + step ? hi : lo + step;
        }
        bool ok = lo + lane < hi && pm[lo + lane] <= t;
        uint32_t cum = lo + __popc(__ballot_sync(0xffffffffu, ok));
        // 128-bit SACK, bit j = chunk cum+j complete (:775-779)
        const uint32_t* cp = d.c_cpl + G.chunk_base;
        uint32_t sw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t x = cum + q * 32 + lane;
            sw[q] = __ballot_sync(0xffffffffu, x < G.n_init && cp[x] <= t);
        }
        // echo of chunk cum + uint8(cause - uint8(cum)) (:781-789)
        uint32_t rel = (csn - (cum & 0xFF)) & 0xFF;
        uint32_t ei = cum + rel;
        int64_t etxt = 0;
        int32_t epath = 0;
        uint32_t eecn = 0;
        if (rel < CN_CSN_WINDOW && ei < G.n_init) {
            uint64_t E = G.chunk_base + ei;
            uint32_t fl = d.c_flags[E];
            bool init = (fl & CF_INIT) || d.c_init[E] <= t;
            if (init) {
                uint32_t exp = pkts_of(d, chunk_len_of(d, G.len, ei));
                uint32_t seen = d.c_seen[E];
                uint32_t f = (static_cast<uint32_t>(lane) < exp && !((seen >> lane) & 1u))
                                 ? d.c_first[E * d.ppc + lane] : kInf;
                bool fok = f <= t;
                uint32_t fm = fok ? f : 0;
                uint32_t lastf = __reduce_max_sync(0xffffffffu, fm);
                uint32_t ecn_b = __ballot_sync(0xffffffffu,
                                               fok && (hdrs[fok ? f - 1 : 0].flags & CN_PKT_ECN));
                if (lastf) {
                    etxt = hdrs[lastf - 1].tx_time;
                    epath = hdrs[lastf - 1].path_id;
                } else {
                    etxt = d.c_txt[E];
                    epath = d.c_path[E];
                }
                eecn = (ecn_b != 0) || (fl & CF_ECN);
            }
        }
        uint32_t a = d.tile_off[2 * tile] + (pos & 0xFFFFu);
        if (lane == 0 && a < max_acks) {
            cn_ack_rec r;
            memset(&r, 0, sizeof r);
            r.src = h.dst;
            r.dst = h.src;
            r.hdr = enc_hdr(h.hdr >> 24, G.msg_id, csn, 0, 0);
            r.echo_path_id = epath;
            r.cum_csn = static_cast<uint8_t>((cum - 1) & 0xFF);
            r.flags = (cum > 0 ? CN_ACK_CUM_VALID : 0) | (eecn ? CN_ACK_ECN_ECHO : 0);
            r.pkt_index = i;
            r.msg_seq = G.seq;
            r.sack[0] = sw[0] | (static_cast<uint64_t>(sw[1]) << 32);
            r.sack[1] = sw[2] | (static_cast<uint64_t>(sw[3]) << 32);
            r.echo_tx_time = etxt;
            acks[a] = r;
        }
    }
    if ((cls & PC_DELIVER) && lane == 0) {
        uint32_t a = d.tile_off[2 * tile + 1] + (pos >> 16);
        if (a < max_cpls) {
            cn_completion c;
            memset(&c, 0, sizeof c);
            c.tag = G.tag;
            c.src = h.src;
            c.dst = h.dst;
            c.len = G.len;
            c.msg_seq = G.seq;
            c.pkt_index = i;
            c.msg_id = G.msg_id;
            c.buf_offset = d.carry ? G.buf_off : ~0ull;
            c.bytes = G.len;  // every byte accepted exactly once
            cpls[a] = c;
        }
    }
    if (cls & PC_COPY) {
        unsigned m = __activemask();
        if (lane == __ffs(m) - 1) {
            atomicAdd(&res->n_copied, 1u);
            atomicAdd(reinterpret_cast<unsigned long long*>(&res->bytes_copied),
                      static_cast<unsigned long long>(h.payload_len));
        }
    }
}

// ------------------------------------------------------------------ K7
// Fold batch scratch into persistent per-chunk state, advance cum, retire
// delivered messages (completed_seq, :801).
__global__ void __launch_bounds__(256) k_finalize(RxDev d, const cn_pkt_hdr* __restrict__ hdrs) {
    __shared__ uint32_t cnt_s;
    uint32_t nt = d.ctl->n_touched;
    for (uint32_t k = blockIdx.x; k < nt; k += gridDim.x) {
        uint32_t g = d.touched[k];
        GenState* G = &d.gen[g];
        uint32_t lo = G->cum, hi = G->n_init;
        uint64_t base = G->chunk_base;
        if (threadIdx.x == 0) cnt_s = 0;
        __syncthreads();
        uint32_t cnt = 0;
        for (uint32_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
            uint64_t e = base + c;
            uint32_t fl = d.c_flags[e];
            if (!(fl & CF_COMPLETE)) {
                uint32_t exp = pkts_of(d, chunk_len_of(d, G->len, c));
                uint32_t seen = d.c_seen[e];
                uint32_t lastf = 0;
                for (uint32_t s = 0; s < exp; ++s) {
                    uint32_t* fp = &d.c_first[e * d.ppc + s];
                    uint32_t f = *fp;
                    if (f == kInf) continue;
                    seen |= 1u << s;
                    lastf = lastf > f ? lastf : f;
                    uint8_t pf = hdrs[f - 1].flags;
                    if (pf & CN_PKT_ECN) fl |= CF_ECN;
                    if (pf & CN_PKT_RTX) fl |= CF_RTX;
                    *fp = kInf;
                }
                d.c_seen[e] = seen;
                if (lastf) {
                    d.c_txt[e] = hdrs[lastf - 1].tx_time;
                    d.c_path[e] = hdrs[lastf - 1].path_id;
                }
                if (d.c_cpl[e] != kInf) fl |= CF_COMPLETE;
            }
            if (d.c_init[e] != kInf) {
                fl |= CF_INIT;
                d.c_init[e] = kInf;
            }
            d.c_flags[e] = fl;
            if (d.c_pmax[e] != kInf) ++cnt;
            d.c_cpl[e] = kInf;
            d.c_pmax[e] = kInf;
        }
        if (cnt) atomicAdd(&cnt_s, cnt);
        __syncthreads();
        if (threadIdx.x == 0) {
            G->cum = lo + cnt_s;
            if (G->deliver_t != kInf) {
                atomicMax(&d.rc_done[G->rc * 128 + G->msg_id],
                          static_cast<unsigned long long>(G->seq));
                d.gen_key[g] = kTomb;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ reset
__global__ void k_reset(RxDev d, int full) {
    uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t nconn = static_cast<uint64_t>(d.conn_mask) + 1, ngen = static_cast<uint64_t>(d.gen_mask) + 1;
    for (uint64_t x = tid; x < nconn; x += stride) d.rc_key[x] = kEmpty;
    for (uint64_t x = tid; x < nconn * 128; x += stride) d.rc_done[x] = 0;
    for (uint64_t x = tid; x < ngen; x += stride) {
        d.gen_key[x] = kEmpty;
        d.gen[x].epoch = 0;
    }
    uint64_t top = full ? d.pool_cap : d.ctl->pool_top;
    if (top > d.pool_cap) top = d.pool_cap;
    for (uint64_t x = tid; x < top; x += stride) {
        d.c_seen[x] = 0;
        d.c_flags[x] = 0;
        d.c_txt[x] = 0;
        d.c_path[x] = 0;
        d.c_init[x] = kInf;
        d.c_cpl[x] = kInf;
        d.c_pmax[x] = kInf;
    }
    for (uint64_t x = tid; x < top * d.ppc; x += stride) d.c_first[x] = kInf;
}

__global__ void k_reset_ctl(RxDev d) {
    d.ctl->pool_top = 0;
    d.ctl->arena_top = 0;
    d.ctl->n_touched = 0;
}

__global__ void k_begin(RxDev d, cn_rx_result* res) {
    d.ctl->n_touched = 0;
    res->n_acks = 0;
    res->n_completions = 0;
    res->status = 0;
    res->n_copied = 0;
    res->bytes_copied = 0;
}

}  // namespace cnb

using namespace cnb;

#include <vector>

constexpr int kRxKernels = 9;  // begin classify alloc mark scan decide tilescan work finalize
static const char* kRxKernelNames[kRxKernels] = {"begin", "classify", "alloc", "mark", "scan",
                                                 "decide", "tilescan", "work", "finalize"};

struct cn_rx {
    cn_rx_config cfg;
    RxDev d;
    uint32_t epoch = 0;
    uint32_t max_tiles = 0;
    int launches = 0;
    int sms = 148;
    // optional per-kernel timing with CUDA events on the launch stream
    bool profiling = false;
    std::vector<std::vector<cudaEvent_t>> pending, spare;
    double acc_ms[kRxKernels] = {0};
    uint64_t acc_n = 0;
};

static void prof_mark(cn_rx* rx, std::vector<cudaEvent_t>* ev, cudaStream_t s) {
    if (!ev) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev->push_back(e);
}

static uint32_t pow2_at_least(uint64_t x) {
    uint32_t p = 1;
    while (p < x && p < (1u << 30)) p <<= 1;
    return p;
}

extern "C" void cn_rx_config_default(cn_rx_config* cfg) {
    cfg->chunk_bytes = 32768;
    cfg->max_payload = CN_MAX_PAYLOAD;
    cfg->max_conns = 1024;
    cfg->max_msgs = 4096;
    cfg->chunk_pool = 1ull << 22;
    cfg->arena_bytes = 1ull << 30;
    cfg->max_batch = 1u << 20;
    cfg->carry_payload = 1;
}

static void rx_free(cn_rx* rx) {
    RxDev& d = rx->d;
    void* ptrs[] = {d.rc_key, d.rc_done, d.gen_key, d.gen, d.touched, d.c_first, d.c_seen,
                    d.c_flags, d.c_txt, d.c_path, d.c_init, d.c_cpl, d.c_pmax, d.p_gen,
                    d.p_pos, d.p_cls, d.tile_cnt, d.tile_off, d.ctl, d.arena};
    for (void* p : ptrs)
        if (p) cudaFree(p);
}

extern "C" int cn_rx_create(const cn_rx_config* cfg_in, cn_rx** out) {
    if (!out) {
        set_error("cn_rx_create: null out");
        return CN_E_INVALID;
    }
    *out = nullptr;
    cn_rx_config cfg;
    cn_rx_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (cfg.max_payload == 0) cfg.max_payload = CN_MAX_PAYLOAD;
    if (cfg.chunk_bytes == 0) {
        set_error("cn_rx_create: chunk_bytes must be >= 1");
        return CN_E_INVALID;
    }
    uint32_t ppc = (cfg.chunk_bytes + cfg.max_payload - 1) / cfg.max_payload;
    if (ppc > CN_MAX_PKTS_PER_CHUNK) {
        set_error("cn_rx_create: chunk needs more than 32 packets (config.cpp:286-287)");
        return CN_E_INVALID;
    }
    if (cfg.max_batch == 0 || cfg.max_batch > (1u << 28) || cfg.max_conns == 0 ||
        cfg.max_msgs == 0 || cfg.chunk_pool == 0) {
        set_error("cn_rx_create: bad capacity");
        return CN_E_INVALID;
    }
    cn_rx* rx = new (std::nothrow) cn_rx();
    if (!rx) return CN_E_CAPACITY;
    rx->cfg = cfg;
    RxDev& d = rx->d;
    memset(&d, 0, sizeof d);
    d.cb = cfg.chunk_bytes;
    d.max_pl = cfg.max_payload;
    d.ppc = ppc;
    d.carry = cfg.carry_payload ? 1 : 0;
    uint32_t nconn = pow2_at_least(cfg.max_conns), ngen = pow2_at_least(2ull * cfg.max_msgs);
    d.conn_mask = nconn - 1;
    d.gen_mask = ngen - 1;
    d.pool_cap = cfg.chunk_pool;
    d.arena_cap = cfg.carry_payload ? cfg.arena_bytes : 0;
    uint64_t B = cfg.max_batch;
    rx->max_tiles = static_cast<uint32_t>((B + kTile - 1) / kTile);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&rx->sms, cudaDevAttrMultiProcessorCount, dev);
#define ALLOC(ptr, bytes)                                         \
    do {                                                          \
        cudaError_t e_ = cudaMalloc(&(ptr), (bytes));             \
        if (e_ != cudaSuccess) {                                  \
            rx_free(rx);                                          \
            delete rx;                                            \
            return cuda_status(e_, "cn_rx_create: cudaMalloc " #ptr); \
        }                                                         \
    } while (0)
    ALLOC(d.rc_key, nconn * 8ull);
    ALLOC(d.rc_done, nconn * 128ull * 8);
    ALLOC(d.gen_key, ngen * 8ull);
    ALLOC(d.gen, ngen * sizeof(GenState));
    ALLOC(d.touched, ngen * 4ull);
    ALLOC(d.c_first, cfg.chunk_pool * ppc * 4);
    ALLOC(d.c_seen, cfg.chunk_pool * 4);
    ALLOC(d.c_flags, cfg.chunk_pool * 4);
    ALLOC(d.c_txt, cfg.chunk_pool * 8);
    ALLOC(d.c_path, cfg.chunk_pool * 4);
    ALLOC(d.c_init, cfg.chunk_pool * 4);
    ALLOC(d.c_cpl, cfg.chunk_pool * 4);
    ALLOC(d.c_pmax, cfg.chunk_pool * 4);
    ALLOC(d.p_gen, B * 4);
    ALLOC(d.p_pos, B * 4);
    ALLOC(d.p_cls, B);
    ALLOC(d.tile_cnt, rx->max_tiles * 8ull);
    ALLOC(d.tile_off, rx->max_tiles * 8ull);
    ALLOC(d.ctl, sizeof(RxCtl));
    if (d.carry) ALLOC(d.arena, cfg.arena_bytes);
#undef ALLOC
    cudaMemset(d.gen, 0, ngen * sizeof(GenState));
    k_reset<<<rx->sms * 4, 256>>>(d, 1);
    k_reset_ctl<<<1, 1>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        rx_free(rx);
        delete rx;
        return cuda_status(e, "cn_rx_create: init");
    }
    *out = rx;
    return CN_OK;
}

extern "C" void cn_rx_destroy(cn_rx* rx) {
    if (!rx) return;
    cudaDeviceSynchronize();
    rx_free(rx);
    delete rx;
}

extern "C" int cn_rx_reset(cn_rx* rx, void* stream) {
    if (!rx) {
        set_error("cn_rx_reset: null handle");
        return CN_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_reset<<<rx->sms * 4, 256, 0, s>>>(rx->d, 0);
    k_reset_ctl<<<1, 1, 0, s>>>(rx->d);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" void* cn_rx_arena(cn_rx* rx) { return rx ? rx->d.arena : nullptr; }
extern "C" int cn_rx_last_launches(const cn_rx* rx) { return rx ? rx->launches : 0; }

extern "C" int cn_rx_batch(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const void* d_payload,
                           uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks,
                           uint32_t max_acks, cn_completion* d_completions,
                           uint32_t max_completions, cn_rx_result* d_result, void* stream) {
    if (!rx || !d_result) {
        set_error("cn_rx_batch: null handle/result");
        return CN_E_INVALID;
    }
    if (n > rx->cfg.max_batch) {
        set_error("cn_rx_batch: n exceeds max_batch");
        return CN_E_CAPACITY;
    }
    if (n > 0 && !d_hdrs) {
        set_error("cn_rx_batch: null headers");
        return CN_E_INVALID;
    }
    if (rx->d.carry && n > 0 && (!d_payload || payload_stride < rx->d.max_pl)) {
        set_error("cn_rx_batch: carry_payload needs a payload staging buffer with stride >= max_payload");
        return CN_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const RxDev& d = rx->d;
    ++rx->epoch;
    if (rx->epoch == 0) rx->epoch = 1;
    std::vector<cudaEvent_t>* ev = nullptr;
    if (rx->profiling && n > 0) {
        rx->pending.emplace_back();
        ev = &rx->pending.back();
    }
    prof_mark(rx, ev, s);
    k_begin<<<1, 1, 0, s>>>(d, d_result);
    prof_mark(rx, ev, s);
    rx->launches = 1;
    if (n > 0) {
        uint32_t pb = (n + 255) / 256;
        uint32_t gb = n < 2u * rx->sms ? n : 2u * rx->sms;
        uint32_t tiles = (n + kTile - 1) / kTile;
        const uint8_t* pl = static_cast<const uint8_t*>(d_payload);
        k_classify<<<pb, 256, 0, s>>>(d, d_hdrs, n, rx->epoch, d_result);
        prof_mark(rx, ev, s);
        k_alloc<<<(gb + 255) / 256, 256, 0, s>>>(d, d_result);
        prof_mark(rx, ev, s);
        k_mark<<<pb, 256, 0, s>>>(d, d_hdrs, n, d_result);
        prof_mark(rx, ev, s);
        k_scan<<<gb, 256, 0, s>>>(d);
        prof_mark(rx, ev, s);
        k_decide<<<tiles, kTile, 0, s>>>(d, d_hdrs, n, d_result);
        prof_mark(rx, ev, s);
        k_tilescan<<<1, 1024, 0, s>>>(d, tiles, max_acks, max_completions, d_result);
        prof_mark(rx, ev, s);
        k_work<<<(n + 7) / 8, 256, 0, s>>>(d, d_hdrs, pl, payload_stride, n, d_acks, max_acks,
                                           d_completions, max_completions, d_result);
        prof_mark(rx, ev, s);
        k_finalize<<<gb, 256, 0, s>>>(d, d_hdrs);
        prof_mark(rx, ev, s);
        rx->launches += 8;
    }
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_rx_set_profiling(cn_rx* rx, int enable) {
    if (!rx) return CN_E_INVALID;
    rx->profiling = enable != 0;
    return CN_OK;
}

// Synchronises pending profiled batches and returns the accumulated
// per-kernel milliseconds (kRxKernels entries) and the batch count.
extern "C" int cn_rx_profile(cn_rx* rx, double* ms, int max, uint64_t* batches, int reset) {
    if (!rx) return CN_E_INVALID;
    for (auto& ev : rx->pending) {
        cudaEventSynchronize(ev.back());
        for (size_t k = 0; k + 1 < ev.size() && k < (size_t)kRxKernels; ++k) {
            float t = 0;
            cudaEventElapsedTime(&t, ev[k], ev[k + 1]);
            rx->acc_ms[k] += t;
        }
        for (auto e : ev) cudaEventDestroy(e);
        rx->acc_n++;
    }
    rx->pending.clear();
    for (int k = 0; k < max && k < kRxKernels; ++k) ms[k] = rx->acc_ms[k];
    if (batches) *batches = rx->acc_n;
    if (reset) {
        for (auto& a : rx->acc_ms) a = 0;
        rx->acc_n = 0;
    }
    return kRxKernels;
}

extern "C" const char* cn_rx_kernel_name(int k) {
    return (k >= 0 && k < kRxKernels) ? kRxKernelNames[k] : "";
}
