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
// Batched, data-parallel restatement: packet i of a batch
// gets the time t = i+1 (0 = an earlier batch).  Per chunk c of a message
//   first[c][s] = first arrival time of packet s of chunk c   (atomicMin)
//   cpl[c]      = max_s first[c][s]  (time the chunk completes; INF if not)
//   pmax[c]     = max(cpl[cum0..c])  (prefix max per message)
// so the cumulative cursor right after packet i is #{c : pmax[c] <= t(i)}.
// Each packet's ack is then an independent snapshot: cum, the 128-bit SACK
// {cpl[cum+j] <= t}, and the echo of chunk cum + uint8(cause - uint8(cum)).
//
// Five kernels per batch, all graph-capturable (no host state per batch):
//   k_ingest   thread/packet: rconn + generation lookup (lock-free hash),
//              lazy message allocation, stale test, first-arrival marking
//   k_copy     warp/packet: the payload scatter of first arrivals (HBM-bound)
//   k_scan     block/message: chunk completion times + prefix max
//   k_acks     block/32-packet tile: decide, warp-parallel decoupled
//              look-back for the ordered ack/completion streams, ack
//              snapshots (SACK by ballot) and completion records
//   k_finalize block/message: fold batch scratch into persistent chunk
//              state, advance cum, retire delivered messages; last block
//              publishes the batch result and arms the next batch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace cnb {

struct GenState {
    uint64_t len, tag, seq, chunk_base, buf_off;  // buf_off: arena offset, ~0 if posted
    uint8_t* buf;                                  // absolute destination of the message
    unsigned long long touch;  // (epoch << 32) | (max chunk touched + 1) in that epoch
    uint32_t nchunks, cum, n_init, rc, msg_id, epoch, deliver_t, slot;  // slot: gen_key index
    uint32_t lo_batch, tiles_done, cum_add, born;  // born: the epoch (batch) that created it
};

// Ring allocator over `cap` positions (chunk-pool entries, or 512-B arena
// blocks): monotonic head/tail counters; storage is 2 x cap so a message's
// range is contiguous without padding; retired positions (mod cap) are bits
// a k_finalize block sweeps the tail over -- the reference frees MsgRecv
// state and buffer at delivery (:794-803).
struct RingCtl {
    unsigned long long head, tail;
};

struct RxCtl {
    RingCtl pool, arena;
    unsigned long long pool_snap, bytes_copied;
    uint32_t n_touched, epoch, tile_ticket, fin_done, status, n_copied, n_acks, n_cpls;
    uint32_t ingest_done, scan_ticket, fin_ticket, n_scan_tiles;
    uint32_t n_trim, pad_t;
    // the per-kernel batch plan: builder ticket, release flag (= epoch)
    uint32_t plan_ticket_scan, plan_ticket_fin, plan_ready_scan, plan_ready_fin;
    // c_first and the scatter's per-packet descriptors come in three parts,
    // batch k using part par = k mod 3: the scatter of batch k may still run
    // while batch k + 1's ack path does (pipelined receivers), so
    // k_finalize(k) clears the part of batch k - 2 -- the tiles it dirtied,
    // listed in dirty[(par + 1) % 3] -- for batch k + 1
    uint32_t par, n_dirty[3], n_dirty_next;
    uint32_t n_aret[3];  // arena ranges of messages delivered in the batch of that part
    // the scatter learns its batch's part through a queue k_ingest pushes
    // (graph replays fix kernel arguments): cq[cq_out & 3], popped by the
    // last block of each k_copy
    uint32_t cq[4], cq_in, cq_out, cq_done, pad_q;
    // message states: a free ring of GenState indices; the (rconn, msg_seq)
    // table maps keys to them, tombstones are compacted by a rebuild
    unsigned long long gfree_head, gfree_tail;
    uint32_t n_tomb, pad_g;
    // ring tail advance (ring_scan): head snapshots the next batch's scan
    // covers, least live offsets found, armed once a scan ran
    unsigned long long pool_hsnap, arena_hsnap;
    uint32_t adv_pool, adv_arena, adv_armed, pad_a;
    uint32_t ret_ticket, ret_done;  // k_finalize's retirement units
    // the global batch plan's slice look-back: (epoch << 32) | slice sum,
    // (epoch << 32) | inclusive prefix; [0] k_scan, [1] k_finalize
    unsigned long long plan_agg[2][16], plan_inc[2][16];
};

enum : uint32_t { CF_INIT = 1, CF_COMPLETE = 2, CF_ECN = 4, CF_RTX = 8, CF_NACKED = 16 };
constexpr uint32_t CF_NACKSET = 0x100;  // c_newfl scratch: a trimmed header after the last new packet
enum : uint8_t { PC_STALE = 1, PC_ACK = 2, PC_COPY = 4, PC_DELIVER = 8, PC_NACK = 16 };
constexpr uint32_t kTrimMax = 16384;  // trimmed headers per batch (sorted in one block, 128 KB smem)
constexpr uint32_t kStale = kInf;    // p_gen marker: stale before the batch
constexpr uint32_t kErr = kInf - 1;  // p_gen marker: rejected packet
constexpr int kAckTileMax = 128;     // packets per k_acks tile (large batches)
constexpr int kAckTileMin = 32;      // ... small batches
#ifndef CN_ACK_WARPS
#define CN_ACK_WARPS 8
#endif
constexpr int kAckWarps = CN_ACK_WARPS;  // 256 threads: 4 decide warps, 8 ack builders
constexpr int kScanThreads = 256;     // chunks per scan/finalize tile
#ifndef CN_COPY_UNROLL
#define CN_COPY_UNROLL 8
#endif
#ifndef CN_COPY_MINB
#define CN_COPY_MINB 1
#endif
constexpr int kCopyUnroll = CN_COPY_UNROLL;  // 16-byte vectors in flight per lane
constexpr uint64_t kArenaUnit = 512;  // arena allocation granule (bytes)
#ifndef CN_ARENA_REL_BLOCKS
#define CN_ARENA_REL_BLOCKS 8192
#endif
constexpr uint32_t kArenaRelBlocks = CN_ARENA_REL_BLOCKS;  // arena blocks per release entry: a large message's release spreads over blocks
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62;

struct RxDev {
    uint32_t cb, max_pl, ppc, conn_mask, gen_mask, carry, reduce, elem, post_mask;
    uint32_t ack_tile;  // packets per k_acks tile this batch (32 or 128)
    uint32_t plan_cap;  // touched messages per batch the scan / finalize plan holds (dynamic smem)
    uint32_t scan_blocks;  // leading k_ingest blocks that scan the rings' retirement bits
    uint32_t max_batch;
    unsigned long long* post_key;  // [posts] message tag (posted destinations)
    unsigned long long* post_val;  // [posts] device pointer
    unsigned long long* post_len;  // [posts] bytes
    uint64_t pool_cap, arena_cap;
    unsigned long long* rc_key;
    unsigned long long* rc_done;  // [conns*128] completed_seq (transport.hpp:223)
    unsigned long long* gen_key;  // [ngen] (rconn << 40) | msg_seq, kEmpty, kTomb
    uint32_t* gen_val;            // [ngen] GenState index of the key, kInf until published
    uint32_t* gen_free;           // [ngen] free ring of GenState indices
    unsigned long long* gen_tmp;  // [ngen] rebuild scratch: (key, index) pairs
    GenState* gen;
    uint32_t* touched;
    uint32_t* c_first;  // [2][pool*ppc] batch scratch (first arrival), half = batch parity
    uint64_t first_part;             // pool*ppc
    unsigned long long* dirty;       // [3][dirty_cap] finalize tiles: (first chunk << 9) | count
    uint32_t dirty_cap;
    uint32_t* pool_bits;             // [pool_cap/32] retired chunk-pool positions
    uint32_t* arena_bits;            // [arena_blocks/32] retired arena blocks
    uint64_t arena_blocks;           // arena_cap / kArenaUnit
    unsigned long long* aret;        // [3][plan_cap] (first block << 31) | blocks, released a batch later
    uint32_t* c_seen;   // [pool] persistent packet bitmask (ChunkRx::pkts_seen)
    uint32_t* c_flags;  // [pool] persistent CF_*
    int64_t* c_txt;     // [pool] persistent ChunkRx::tx_time
    int32_t* c_path;    // [pool] persistent ChunkRx::path
    uint32_t* c_init;   // [pool] batch scratch: first arrival time
    uint32_t* c_cpl;    // [pool] batch scratch: completion time
    uint32_t* c_pmax;   // [pool] batch scratch: prefix max of c_cpl
    uint32_t* c_newb;   // [pool] batch scratch: bits of new packets
    uint32_t* c_last;   // [pool] batch scratch: last new packet time
    uint32_t* c_newfl;  // [pool] batch scratch: ECN/RTX of new packets
    uint32_t* p_gen;    // [batch]
    unsigned long long* p_dst;  // [3][batch] scatter destination of a candidate first arrival, 0 = none
    uint32_t* p_fi;             // [3][batch] its c_first index (chunk entry * ppc + seq)
    uint8_t* p_nack;    // [batch] trimmed header that emits a NACK
    // ordered reliability (go-back-N receive filter)
    uint32_t ordered;
    const uint64_t* psn;      // [batch] conn_psn of the current batch
    // [batch] per-packet message data (Packet::msg_data, transport.hpp:88-91,
    // transport.cpp:486): packet i's payload at msgdata[i] + its message offset
    const unsigned long long* msgdata;
    // [batch] packed payloads (cn_rx_batch_packed): packet i's payload at payload + poff[i]
    const unsigned long long* poff;
    uint8_t* p_gbn;           // [batch] 0 pass on, 1 drop, 2 drop with a NACK
    uint64_t* p_gbn_psn;      // [batch] nack_psn of a NACK
    uint64_t* gbn_expected;   // [rconn] RecvConn::expected_psn
    uint8_t* gbn_nacked;      // [rconn] RecvConn::gap_nacked
    uint32_t* trim_list;  // [kTrimMax] trimmed headers of the batch (packet index)
    uint32_t* plan_F;     // [plan_cap + 1] flattened chunk offset of each touched message
    uint32_t* plan_t0;    // [tiles + 1] first message of each 256-chunk tile
    unsigned long long* tile_state;  // [ack tiles] decoupled look-back (ack order)
    unsigned long long* scan_state;  // [scan tiles] segmented look-back (prefix max)
    RxCtl* ctl;
    uint8_t* arena;
    // kept last: inserting it among the fields above reordered k_copy's
    // parameter loads and cost the scatter 3% on large batches (measured)
    uint32_t aret_cap;  // arena-release entries per part (a message: one per kArenaRelBlocks)
};

// One thread.  Ring positions [h, h + n) by one atomicAdd (no retry loop:
// a batch of a thousand new messages must not serialise on the head), laid
// out at physical [h % cap, h % cap + n) of arrays sized 2 x cap, so a range
// never wraps.  Over capacity: false -- CN_RXF_CAPACITY, fatal for the
// receiver until cn_rx_reset, as an exhausted pool always was.
__device__ inline bool ring_alloc(RingCtl* r, uint64_t cap, uint64_t n, uint64_t* pos) {
    if (n == 0 || n > cap) return false;
    const unsigned long long h = atomicAdd(&r->head, static_cast<unsigned long long>(n));
    if (h + n - ld_volatile_u64(&r->tail) > cap) return false;
    *pos = h % cap;
    return true;
}

// Lap-parity retirement bits.  Ring position p (monotonic) lies in lap
// p / cap and is retired in that lap iff its bit equals (lap + 1) & 1: a
// release toggles the bit (every position is allocated and released exactly
// once per lap), so bits are never cleared and the tail advance is a
// read-only scan any number of blocks share.  Returns, per warp, the least
// offset from the tail of a live position in [tail, hsnap) into *out
// (atomicMin; untouched if all retired).  Spare k_ingest blocks run it
// beside the packet blocks: they see every release of earlier batches, the
// tail moves in k_finalize -- off the critical path.
__device__ __forceinline__ uint32_t span_mask(uint32_t a, uint32_t b) {  // bits [a, b), 0 <= a < b <= 32
    return (b == 32 ? ~0u : (1u << b) - 1u) & (~0u << a);
}
__device__ void ring_scan(const RingCtl* r, unsigned long long hsnap, uint64_t cap, const uint32_t* bits,
                          uint32_t* out, uint32_t worker, uint32_t workers) {
    const uint64_t t = ld_volatile_u64(&r->tail);
    const uint64_t n = hsnap > t ? hsnap - t : 0;
    uint32_t best = ~0u;
    if (n) {
        const uint64_t tq = t % cap, L0 = t / cap;
        const uint32_t eh = ((L0 + 1) & 1) ? ~0u : 0u, el = ~eh;  // retired values of laps L0, L0 + 1
        const uint64_t nw = (cap + 31) >> 5;
        for (uint64_t w = worker; w < nw; w += workers) {
            const uint64_t q0 = w << 5;
            const uint32_t lim = cap - q0 < 32 ? static_cast<uint32_t>(cap - q0) : 32u;
            uint32_t hi = 0, lo = 0;  // valid bits of lap L0 (q >= tq) and of lap L0 + 1 (q < tq)
            {
                const uint64_t a = q0 > tq ? q0 : tq, b0 = q0 + lim, b1 = tq + n;
                const uint64_t b = b0 < b1 ? b0 : b1;
                if (a < b) hi = span_mask(static_cast<uint32_t>(a - q0), static_cast<uint32_t>(b - q0));
            }
            if (n > cap - tq) {
                uint64_t b = q0 + lim;
                if (b > tq) b = tq;
                if (b > n - (cap - tq)) b = n - (cap - tq);
                if (q0 < b) lo = span_mask(0, static_cast<uint32_t>(b - q0));
            }
            if (!(hi | lo)) continue;
            const uint32_t v = bits[w];
            const uint32_t lh = (v ^ eh) & hi, ll = (v ^ el) & lo;  // live positions
            uint64_t off = ~0ull;
            if (lh) off = q0 + __ffs(lh) - 1 - tq;
            else if (ll) off = cap - tq + q0 + __ffs(ll) - 1;
            if (off < best) best = static_cast<uint32_t>(off);
        }
    }
    best = __reduce_min_sync(0xffffffffu, best);
    if ((threadIdx.x & 31) == 0 && best != ~0u) atomicMin(out, best);
}
// k_finalize's last block: the tail moves over the retired prefix
__device__ __forceinline__ void ring_move_tail(RingCtl* r, unsigned long long hsnap, uint32_t off) {
    const uint64_t n = hsnap > r->tail ? hsnap - r->tail : 0;
    r->tail += off < n ? off : n;
}

// Debug builds (make EXTRA=-DCN_RX_TIMING): %globaltimer marks at phase
// boundaries of the receive kernels (min over blocks for starts, max for
// ends), read and cleared by cn_rx_debug_timing (tools/, not the product).
#ifdef CN_RX_TIMING
__device__ unsigned long long g_tm[64];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TM_END(slot_)                                         \
    do {                                                      \
        if (threadIdx.x == 0) atomicMax(&g_tm[slot_], gtime()); \
    } while (0)
#define TM_START(slot_)                                       \
    do {                                                      \
        if (threadIdx.x == 0) atomicMin(&g_tm[slot_], gtime()); \
    } while (0)
constexpr int kTileTm = 8192;
__device__ unsigned long long g_ing_tm[5][64];  // k_ingest packet blocks 0..63: start, conn, gen, end, first-load
#define TM_ING(k_, b_)                                                    \
    do {                                                                  \
        if (threadIdx.x == 0 && (b_) < 64) g_ing_tm[k_][b_] = gtime();   \
    } while (0)
__device__ unsigned long long g_tile_tm[4][kTileTm];  // k_acks per tile: start, decided, built, written
#define TM_TILE(k_, tile_)                                                   \
    do {                                                                     \
        if (threadIdx.x == 0 && (tile_) < kTileTm) g_tile_tm[k_][tile_] = gtime(); \
    } while (0)
#else
#define TM_TILE(k_, tile_) \
    do {                   \
    } while (0)
#define TM_ING(k_, b_) \
    do {               \
    } while (0)
#define TM_END(slot_) \
    do {              \
    } while (0)
#define TM_START(slot_) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ uint32_t* first_of(const RxDev& d, uint32_t par) {
    return d.c_first + par * d.first_part;
}

__device__ __forceinline__ uint32_t chunk_len_of(const RxDev& d, uint64_t len, uint64_t c) {
    uint64_t rem = len - c * d.cb;
    return rem < d.cb ? static_cast<uint32_t>(rem) : d.cb;
}
__device__ __forceinline__ uint32_t pkts_of(const RxDev& d, uint32_t clen) {
    return (clen + d.max_pl - 1) / d.max_pl;
}

// ------------------------------------------------------------ go-back-N
// handle_data_ordered (transport.cpp:690-717): per receive connection, a
// packet at the expected sequence advances it and goes on to handle_data;
// one past it (or a trimmed one at it) is dropped with a NACK naming the
// expected sequence, once until the gap closes; a trimmed one below it is
// dropped; a full one below it goes on (a duplicate).  A per-connection
// sequential scan: warp w owns the connections whose table slot is
// congruent to w and walks the batch in arrival order, 32 packets at a time.
__global__ void __launch_bounds__(256) k_gbn(RxDev d, const cn_pkt_hdr* __restrict__ hdrs, uint32_t n) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w0 = 0; w0 < n; w0 += 32) {
        const uint32_t i = w0 + lane;
        uint32_t rc = kInf;
        if (i < n) {
            const cn_pkt_hdr& h = hdrs[i];
            const uint64_t rkey = (static_cast<uint64_t>(h.dst) << 32) | (static_cast<uint64_t>(h.src) << 8) |
                                  (h.hdr >> 24);
            bool ins = false;
            rc = table_insert(d.rc_key, d.conn_mask, rkey, &ins);
        }
        for (unsigned m = __ballot_sync(0xffffffffu, rc != kInf && rc % nw == gw); m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            if (lane == j) {
                const uint64_t p = d.psn[i];
                const bool trimmed = (hdrs[i].flags & CN_PKT_TRIMMED) != 0;
                uint64_t e = d.gbn_expected[rc];
                uint8_t g = d.gbn_nacked[rc];
                uint8_t out = 0;
                if (p > e || (trimmed && p == e)) {
                    out = 1;
                    if (!g) {
                        g = 1;
                        out = 2;
                        d.p_gbn_psn[i] = e;
                    }
                } else if (trimmed) {
                    out = 1;
                } else if (p == e) {
                    ++e;
                    g = 0;
                }
                d.gbn_expected[rc] = e;
                d.gbn_nacked[rc] = g;
                d.p_gbn[i] = out;
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------ ingest
// rconn_at (transport.cpp:546-563), the stale-generation test (:602), lazy
// MsgRecv init (:620-626) with its chunk vector and buffer (:637, :723),
// chunk init (:639-645) and the per-packet bit (:676-683) recorded as a
// first-arrival time.
//
// Table work is block-aggregated: a batch carries few distinct connections
// and message generations, and every packet of a generation reads the same
// table slot and GenState line -- thousands of same-line L2 requests that
// serialise on one slice.  So lanes first dedupe keys in the warp
// (match_any), warp leaders dedupe them again in a shared-memory map, and
// only one thread per distinct key and block touches the global tables;
// results are broadcast through shared memory.
constexpr int kIngestThreads = 256;  // one packet per thread
constexpr int kIngMap = 512;         // shared map slots (power of two, >= 2 x threads)
constexpr unsigned long long kMapEmpty = ~0ull;

// Inserts key into the block map; returns its slot and whether this thread
// owns it (first inserter).
__device__ __forceinline__ uint32_t map_insert(unsigned long long* keys, uint64_t key, bool* own) {
    uint32_t h = static_cast<uint32_t>(mix64(key)) & (kIngMap - 1);
    for (;;) {
        unsigned long long k = keys[h];
        if (k == key) {
            *own = false;
            return h;
        }
        if (k == kMapEmpty) {
            unsigned long long old = atomicCAS(&keys[h], kMapEmpty, key);
            if (old == kMapEmpty) {
                *own = true;
                return h;
            }
            if (old == key) {
                *own = false;
                return h;
            }
        }
        h = (h + 1) & (kIngMap - 1);
    }
}

__global__ void __launch_bounds__(kIngestThreads) k_ingest(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                                           uint32_t n) {
    __shared__ unsigned long long m_key[kIngMap];
    __shared__ unsigned long long m_cbase[kIngMap], m_glen[kIngMap], m_buf[kIngMap];
    __shared__ uint8_t m_fresh[kIngMap];  // generation created in this batch: its chunk state is initial
    __shared__ uint32_t m_val[kIngMap], m_nch[kIngMap], m_touch[kIngMap];
    __shared__ uint32_t s_status;
    const int lane = threadIdx.x & 31;
    pdl_launch();  // k_scan may launch now (it waits for this grid)
    TM_START(10);
    if (blockIdx.x < d.scan_blocks) {  // the first blocks scan the rings (ring_scan)
        const uint32_t worker = blockIdx.x * kIngestThreads + threadIdx.x;
        const uint32_t workers = d.scan_blocks * kIngestThreads;
        RxCtl* C = d.ctl;
        ring_scan(&C->pool, C->pool_hsnap, d.pool_cap, d.pool_bits, &C->adv_pool, worker, workers);
        if (d.arena_blocks)
            ring_scan(&C->arena, C->arena_hsnap, d.arena_blocks, d.arena_bits, &C->adv_arena, worker, workers);
        if (worker == 0) C->adv_armed = 1;
        return;
    }
    const uint32_t i = (blockIdx.x - d.scan_blocks) * blockDim.x + threadIdx.x;
    const uint32_t pblk = blockIdx.x - d.scan_blocks;
    TM_ING(0, pblk);
    const uint32_t epoch = d.ctl->epoch;
    const uint32_t par = d.ctl->par;
    // the rings' tails move only in k_finalize: read them with the header, off
    // the inserters' dependent chain
    const unsigned long long ptail = ld_volatile_u64(&d.ctl->pool.tail);
    const unsigned long long atail = ld_volatile_u64(&d.ctl->arena.tail);
    const uint32_t tiles = (n + d.ack_tile - 1) / d.ack_tile;
    if (i < tiles) d.tile_state[i] = 0;
    if (i == 0 && d.carry) {  // the scatter of this batch reads part par
        RxCtl* C = d.ctl;
        C->cq[C->cq_in & 3] = par;
        C->cq_in += 1;
    }
    for (int k = threadIdx.x; k < kIngMap; k += kIngestThreads) {
        m_key[k] = kMapEmpty;
        m_touch[k] = 0;
    }
    if (threadIdx.x == 0) s_status = 0;
    uint32_t status = 0;
    uint32_t g = kErr;
    uint32_t touch = 0;
    unsigned long long cdst = 0;  // scatter descriptor (0: nothing to copy)
    uint32_t cfi = 0;
    cn_pkt_hdr h;
    bool ok = i < n;
    if (ok && d.ordered && d.p_gbn[i]) ok = false;  // dropped by the go-back-N filter
    if (ok) {
        h = hdrs[i];
        if (static_cast<uint32_t>(h.src) >= (1u << 24) ||
            static_cast<uint32_t>(h.dst) >= (1u << 24) || h.msg_seq >= (1ull << 40) ||
            h.msg_seq == 0) {
            status |= CN_RXF_UNSUPPORTED;
            ok = false;
        }
    } else {
        memset(&h, 0, sizeof h);
    }
    const uint32_t mid = (h.hdr >> 17) & 0x7F;
    __syncthreads();
    TM_ING(4, pblk);
    // ---- connection (dst, src, conn_id)
    const uint64_t rkey = (static_cast<uint64_t>(h.dst) << 32) | (static_cast<uint64_t>(h.src) << 8) |
                          (h.hdr >> 24);
    uint32_t rslot = 0;
    {
        const unsigned pr = __match_any_sync(0xffffffffu, ok ? rkey : (0xF000000000000000ull | lane));
        const int lr = __ffs(pr) - 1;
        bool own = false;
        if (ok && lane == lr) rslot = map_insert(m_key, rkey, &own);
        rslot = __shfl_sync(0xffffffffu, rslot, lr);
        __syncthreads();
        if (own) {
            bool ins = false;
            m_val[rslot] = table_insert(d.rc_key, d.conn_mask, rkey, &ins);
            m_nch[rslot] = ins;  // a connection new this batch: completed_seq is all 0
        }
        __syncthreads();
    }
    uint32_t rc = ok ? m_val[rslot] : kInf;
    if (ok && rc == kInf) {
        status |= CN_RXF_CAPACITY;
        ok = false;
    }
    if (ok && !m_nch[rslot] && h.msg_seq <= d.rc_done[rc * 128 + mid]) {
        g = kStale;  // transport.cpp:602
        ok = false;
    }
    TM_END(11);
    TM_ING(1, pblk);
    // ---- message generation (rconn, msg_seq)
    for (int k = threadIdx.x; k < kIngMap; k += kIngestThreads) m_key[k] = kMapEmpty;
    __syncthreads();
    const uint64_t gkey = (static_cast<uint64_t>(rc) << 40) | h.msg_seq;
    const unsigned pg = __match_any_sync(0xffffffffu, ok ? gkey : (0xF000000000000000ull | lane));
    const int lg = __ffs(pg) - 1;
    uint32_t gslot = 0;
    bool gown = false;
    if (ok && lane == lg) gslot = map_insert(m_key, gkey, &gown);
    gslot = __shfl_sync(0xffffffffu, gslot, lg);
    __syncthreads();
    // the generation's table slot; the unique inserter of a new generation
    // allocates its state (GenState index, touched-list slot, chunk-pool
    // range, arena range when no posted destinations exist) -- the shared
    // counters claimed once per warp for all of its inserters
    bool gins = false;
    uint32_t gslot_t = kInf;
    if (gown) gslot_t = table_insert(d.gen_key, d.gen_mask, gkey, &gins);
    gins = gins && gslot_t != kInf;
    uint64_t a_nc = 0, a_nb = 0;
    uint32_t a_st = 0;
    bool a_early = false;
    if (gins) {
        a_nc = (h.msg_len + d.cb - 1) / d.cb;
        a_nb = (h.msg_len + kArenaUnit - 1) / kArenaUnit;
        if (h.msg_len == 0 || a_nc >= (1ull << 31) || (d.reduce && (h.msg_len % d.elem))) a_st = CN_RXF_UNSUPPORTED;
        a_early = !a_st && d.carry && !d.post_mask && d.arena_blocks;
    }
    unsigned long long a_gi = 0, a_ph = 0, a_ah = 0;
    uint32_t a_tk = 0;
    {
        const unsigned ib = __ballot_sync(0xffffffffu, gins);
        if (ib) {
            const uint64_t pnc = gins && !a_st ? a_nc : 0, pnb = a_early ? a_nb : 0;
            uint64_t inc_c = pnc, inc_b = pnb;  // inclusive warp prefix sums
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t yc = __shfl_up_sync(0xffffffffu, inc_c, o), yb = __shfl_up_sync(0xffffffffu, inc_b, o);
                if (lane >= o) {
                    inc_c += yc;
                    inc_b += yb;
                }
            }
            unsigned long long gi0 = 0, ph0 = 0, ah0 = 0;
            uint32_t tk0 = 0;
            if (lane == 31) {
                const uint32_t cnt = __popc(ib);
                gi0 = atomicAdd(&d.ctl->gfree_head, static_cast<unsigned long long>(cnt));
                // a new generation is touched by this batch
                tk0 = atomicAdd(&d.ctl->n_touched, cnt);
                if (inc_c) ph0 = atomicAdd(&d.ctl->pool.head, static_cast<unsigned long long>(inc_c));
                if (inc_b) ah0 = atomicAdd(&d.ctl->arena.head, static_cast<unsigned long long>(inc_b));
            }
            gi0 = __shfl_sync(0xffffffffu, gi0, 31);
            tk0 = __shfl_sync(0xffffffffu, tk0, 31);
            ph0 = __shfl_sync(0xffffffffu, ph0, 31);
            ah0 = __shfl_sync(0xffffffffu, ah0, 31);
            const uint32_t rank = __popc(ib & ((1u << lane) - 1));
            a_gi = gi0 + rank;
            a_tk = tk0 + rank;
            a_ph = ph0 + (inc_c - pnc);
            a_ah = ah0 + (inc_b - pnb);
        }
    }
    if (gown) {
        uint32_t gs = kInf, nch = 0;
        unsigned long long cbase = 0, glen = 0, gbuf = 0;
        bool fresh = false;
        const uint32_t slot = gslot_t;
        if (slot != kInf) {
            GenState* G = nullptr;
            if (gins) {
                const uint64_t nc = a_nc, nb = a_nb;
                uint32_t st = a_st;
                const bool early_arena = a_early;
                const unsigned long long gi = a_gi;
                const uint32_t tk = a_tk;
                const unsigned long long ph = a_ph, ah = a_ah;
                // never empty: live keys <= table slots = GenStates
                gs = d.gen_free[gi & d.gen_mask];
                G = &d.gen[gs];
                uint64_t base = 0;
                unsigned long long boff = 0;
                // ring_alloc's capacity rule (fatal for the receiver until reset)
                if (!st && (nc > d.pool_cap || ph + nc - ptail > d.pool_cap)) st = CN_RXF_CAPACITY;
                if (!st) base = ph % d.pool_cap;
                uint8_t* buf = nullptr;
                if (!st && d.carry && d.post_mask) {  // a posted destination (cn_rx_post)
                    uint32_t hp = static_cast<uint32_t>(mix64(h.msg_tag)) & d.post_mask;
                    for (uint32_t q = 0; q <= d.post_mask; ++q) {
                        unsigned long long k = __ldcg(&d.post_key[hp]);
                        if (k == kEmpty) break;
                        if (k == h.msg_tag) {
                            if (__ldcg(&d.post_len[hp]) >= h.msg_len)
                                buf = reinterpret_cast<uint8_t*>(__ldcg(&d.post_val[hp]));
                            break;
                        }
                        hp = (hp + 1) & d.post_mask;
                    }
                    if (buf) boff = ~0ull;
                }
                if (!st && d.carry && !buf) {  // arena blocks of kArenaUnit bytes
                    uint64_t ab = 0;
                    bool ok_ = false;
                    if (early_arena) {
                        ok_ = nb <= d.arena_blocks && ah + nb - atail <= d.arena_blocks;
                        ab = ah % d.arena_blocks;
                    } else {
                        ok_ = ring_alloc(&d.ctl->arena, d.arena_blocks, nb, &ab);
                    }
                    if (ok_) {
                        boff = ab * kArenaUnit;
                        buf = d.arena + boff;
                    } else {
                        st = CN_RXF_CAPACITY;
                    }
                }
                status |= st;
                G->len = h.msg_len;
                G->tag = h.msg_tag;
                G->seq = h.msg_seq;
                G->chunk_base = st ? 0 : base;
                G->buf_off = boff;
                G->buf = buf;
                G->touch = 0;
                G->nchunks = st ? 0 : static_cast<uint32_t>(nc);
                G->cum = 0;
                G->n_init = 0;
                G->rc = rc;
                G->msg_id = mid;
                G->deliver_t = kInf;
                G->slot = slot;
                G->epoch = epoch;  // first touch is this batch
                G->born = epoch;
                G->lo_batch = 0;
                G->tiles_done = 0;
                G->cum_add = 0;
                d.touched[tk] = gs;
                st_release(&d.gen_val[slot], gs);
                nch = G->nchunks;  // this thread's own values: no read back
                cbase = G->chunk_base;
                glen = h.msg_len;
                gbuf = reinterpret_cast<unsigned long long>(buf);
                fresh = true;
            } else {
                // wait for the inserter (resident, already past its CAS)
                uint32_t spins = 0;
                while ((gs = ld_acquire(&d.gen_val[slot])) == kInf) {
                    __nanosleep(32);
                    if (++spins > (1u << 24)) {
                        status |= CN_RXF_CAPACITY;
                        break;
                    }
                }
                if (gs != kInf) G = &d.gen[gs];
            }
            if (gs != kInf && !gins) {
                nch = G->nchunks;
                cbase = G->chunk_base;
                glen = G->len;
                gbuf = reinterpret_cast<unsigned long long>(G->buf);
                fresh = G->born == epoch;
                // plain read first: only the first block of the batch pays the atomic
                if (ld_volatile_u32(&G->epoch) != epoch && atomicExch(&G->epoch, epoch) != epoch) {
                    // first touch this batch: freeze the batch's lower bound
                    // (finalize advances cum) and clear the tile counters
                    G->lo_batch = G->cum;
                    G->tiles_done = 0;
                    G->cum_add = 0;
                    uint32_t k = atomicAdd(&d.ctl->n_touched, 1u);
                    d.touched[k] = gs;
                }
            }
        } else {
            status |= CN_RXF_CAPACITY;
        }
        m_val[gslot] = gs;
        m_nch[gslot] = nch;
        m_cbase[gslot] = cbase;
        m_glen[gslot] = glen;
        m_buf[gslot] = gbuf;
        m_fresh[gslot] = fresh;
    }
    __syncthreads();
    TM_END(12);
    TM_ING(2, pblk);
    const uint32_t gs = ok ? m_val[gslot] : kInf;
    if (ok && gs != kInf) {
        const uint32_t nch = m_nch[gslot];
        const unsigned long long cbase = m_cbase[gslot], glen = m_glen[gslot];
        const uint64_t c = h.chunk_offset / d.cb;
        const uint32_t s = h.seq_in_chunk;
        bool bad = nch == 0 || (h.chunk_offset % d.cb) != 0 || c >= nch || h.msg_len != glen;
        if (!bad) {
            uint32_t clen = chunk_len_of(d, glen, c);
            uint32_t exp = pkts_of(d, clen);
            uint32_t pl = clen - s * d.max_pl;
            pl = pl < d.max_pl ? pl : d.max_pl;
            bad = ((h.hdr >> 9) & 0xFF) != (c & 0xFF) || h.chunk_len != clen || s >= exp ||
                  h.payload_len != pl || ((h.hdr >> 8) & 1) != (c + 1 == nch ? 1u : 0u) ||
                  (d.reduce && ((h.chunk_offset | pl) % d.elem));
        }
        if (bad) {
            status |= CN_RXF_UNSUPPORTED;
        } else {
            g = gs;
            const uint64_t e = cbase + c;
            const uint32_t t = i + 1;
            // a generation created in this batch has initial chunk state: no loads
            const bool fresh = m_fresh[gslot];
            const uint32_t fl = fresh ? 0u : d.c_flags[e];
            if (h.flags & CN_PKT_TRIMMED) {  // header only: chunk init, then the NACK pass (k_trim)
                const uint32_t k = atomicAdd(&d.ctl->n_trim, 1u);
                if (k < kTrimMax) d.trim_list[k] = i;
                else status |= CN_RXF_CAPACITY;
            } else if (!(fl & CF_COMPLETE) && (fresh || !((d.c_seen[e] >> s) & 1u))) {
                const uint64_t fi = e * d.ppc + s;
                atomicMin(&first_of(d, par)[fi], t);
                if (d.carry) {  // the scatter's descriptor (k_copy keeps the first arrival)
                    const uint64_t moff = h.chunk_offset + static_cast<uint64_t>(s) * d.max_pl;
                    cdst = m_buf[gslot] + moff;
                    cfi = static_cast<uint32_t>(fi);
                }
            }
            if (!(fl & CF_INIT)) atomicMin(&d.c_init[e], t);
            touch = static_cast<uint32_t>(c) + 1;
        }
    }
    if (i < n) {
        d.p_gen[i] = g;
        d.p_nack[i] = 0;
        if (d.carry) {
            d.p_dst[par * static_cast<uint64_t>(d.max_batch) + i] = cdst;
            d.p_fi[par * static_cast<uint64_t>(d.max_batch) + i] = cfi;
        }
    }
    // chunk-vector size per message (:636-637): max over the block, one
    // global atomic per generation and block
    const uint32_t gm = __reduce_max_sync(pg, touch);  // lanes of one group share pg
    if (lane == lg && gm) atomicMax(&m_touch[gslot], gm);
    status = __reduce_or_sync(0xffffffffu, status);
    if (lane == 0 && status) atomicOr(&s_status, status);
    __syncthreads();
    if (gown && m_val[gslot] != kInf && m_touch[gslot])
        atomicMax(&d.gen[m_val[gslot]].touch, (static_cast<unsigned long long>(epoch) << 32) | m_touch[gslot]);
    if (threadIdx.x == 0 && s_status) atomicOr(&d.ctl->status, s_status);
    TM_END(13);
    TM_ING(3, pblk);
}


// block-wide inclusive max-scan (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ uint32_t block_scan_max(uint32_t v, uint32_t* wsum) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = v > x ? v : x;
    }
    if (lane == 31) wsum[w] = v;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < nw ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = x > y ? x : y;
        }
        wsum[lane] = x;
    }
    __syncthreads();
    if (w > 0) {
        uint32_t p = wsum[w - 1];
        v = v > p ? v : p;
    }
    return v;
}


// -------------------------------------------------------------------- scan
// Flattened over every touched message: the batch's chunk ranges [lo, hi)
// are laid end to end and cut into tiles of 256 consecutive chunks, so a
// tile may hold the tail of one message, several whole small messages and
// the head of another (a thousand 1-chunk messages are 4 tiles, not 1,000).
// Per chunk: the completion time cpl (max first arrival over its missing
// packets), the new-packet bitmask and last new packet (for finalize), and
// the prefix max pmax that drives the cumulative cursor (chunk_completed's
// `while (complete) ++cum`, :736-738) -- a segmented max-scan inside the
// tile (reset at message boundaries) plus a decoupled look-back for the
// message that continues from earlier tiles.
constexpr uint32_t kPlanMax = 16384;  // cap of RxDev::plan_cap (touched messages per batch, planned in smem)

// The batch plan, built once per kernel (in every block's shared memory for
// up to kPlanSmem messages, else once in global memory by the grid): for
// each touched message k its chunk range [lo, hi) -- hi = the chunk vector
// size (:636-637) -- flattened as the exclusive prefix F[k] of the range
// lengths (F[nt] = total chunks), and for every 256-chunk tile t the first
// message t0[t] that has a chunk in it.  In k_scan lo = cum and hi =
// max(n_init, max touched chunk + 1); k_finalize reads the values k_scan
// stored (lo_batch, n_init; a delivered message whole), so both see the
// same flattened layout.  The large plan lives in global memory (L1 / L2
// resident): shared memory in these latency-bound kernels would shrink the
// L1 of the SMs the concurrent HBM-bound scatter streams through.  Its
// message-state loads are scattered, so one SM cannot issue them fast
// enough (~50 us for 16K messages); spread over the grid they cost a few.
__device__ __forceinline__ uint32_t plan_len(const RxDev& d, uint32_t k, uint32_t epoch, bool scan) {
    const GenState* G = &d.gen[d.touched[k]];
    uint32_t lo, hi;
    if (scan) {
        lo = G->cum;
        hi = G->n_init;
        const unsigned long long tch = G->touch;
        if ((tch >> 32) == epoch && static_cast<uint32_t>(tch) > hi) hi = static_cast<uint32_t>(tch);
    } else if (G->deliver_t != kInf) {
        // a delivered message is retired whole: its chunk range is reset and
        // handed back to the pool ring
        lo = 0;
        hi = G->nchunks;
    } else {
        lo = G->lo_batch;
        hi = G->n_init;
    }
    return hi > lo ? hi - lo : 0;
}

constexpr uint32_t kPlanSmem = 2048;  // up to this many touched messages every block plans in smem (8 KB)
constexpr uint32_t kPlanSlice = 1024;  // global plan: messages per slice (4 per thread)
constexpr uint32_t kPlanSlices = kPlanMax / kPlanSlice;
static_assert(kPlanSlices <= 16, "RxCtl::plan_agg holds 16 slices");

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block exclusive scan of one value per thread; *tot gets the block total.
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* s_w, uint32_t* tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t wpre = 0, t = 0;
    for (int q = 0; q < nw; ++q) {
        if (q < w) wpre += s_w[q];
        t += s_w[q];
    }
    *tot = t;
    return wpre + inc - v;
}

// Returns the total; F points at the plan (s_F when nt <= kPlanSmem -- each
// block builds its own copy -- else the global one).  The global plan is a
// single-pass scan spread over the grid: blocks take 1,024-message slices by
// ticket (so a slice is only ever waited on once a running block holds it),
// publish the slice sum, look back over the earlier slices for their base
// (decoupled look-back, tagged with the batch epoch so nothing is reset),
// write their offsets and tile starts and count the slice done; every block
// then waits for all slices.
__device__ uint32_t plan_batch(const RxDev& d, uint32_t nt, uint32_t epoch, bool scan, uint32_t* s_F,
                               const uint32_t** F_out) {
    __shared__ uint32_t s_w[32], s_total, s_sl, s_base;
    RxCtl* C = d.ctl;
    constexpr uint32_t kPer = kPlanSlice / kScanThreads;
    if (nt <= kPlanSmem) {
        *F_out = s_F;
        const uint32_t per = (nt + blockDim.x - 1) / blockDim.x;  // <= 8
        const uint32_t k0 = threadIdx.x * per, k1 = min(nt, k0 + per);
        uint32_t L[kPlanSmem / kScanThreads], sum = 0;
#pragma unroll
        for (uint32_t j = 0; j < kPlanSmem / kScanThreads; ++j) {
            L[j] = k0 + j < k1 ? plan_len(d, k0 + j, epoch, scan) : 0u;
            sum += L[j];
        }
        uint32_t tot;
        uint32_t F = block_excl_sum(sum, s_w, &tot);
#pragma unroll
        for (uint32_t j = 0; j < kPlanSmem / kScanThreads; ++j)
            if (k0 + j < k1) {
                s_F[k0 + j] = F;
                F += L[j];
            }
        if (threadIdx.x == 0) s_F[nt] = tot;
        __syncthreads();
        return tot;
    }
    *F_out = d.plan_F;
    TM_START(scan ? 30 : 34);
    uint32_t* ticket = scan ? &C->plan_ticket_scan : &C->plan_ticket_fin;
    uint32_t* done = scan ? &C->plan_ready_scan : &C->plan_ready_fin;
    unsigned long long* agg = C->plan_agg[scan ? 0 : 1];
    unsigned long long* incl = C->plan_inc[scan ? 0 : 1];
    const unsigned long long tag = static_cast<unsigned long long>(C->epoch) << 32;  // never 0
    const uint32_t ns = (nt + kPlanSlice - 1) / kPlanSlice;
    for (;;) {
        if (threadIdx.x == 0) s_sl = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t sl = s_sl;
        if (sl >= ns) break;
        const uint32_t kb = sl * kPlanSlice + threadIdx.x * kPer;
        uint32_t L[kPer], sum = 0;
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            L[u] = kb + u < nt ? plan_len(d, kb + u, epoch, scan) : 0u;
            sum += L[u];
        }
        uint32_t tot;
        uint32_t F = block_excl_sum(sum, s_w, &tot);
        if (threadIdx.x < 32) {  // warp 0: publish, then look back over all earlier slices at once
            const int lane = threadIdx.x;
            uint32_t base = 0;
            if (sl == 0) {
                if (lane == 0) st_release_u64(&incl[0], tag | tot);
            } else {
                if (lane == 0) st_release_u64(&agg[sl], tag | tot);
                const int q = static_cast<int>(sl) - 1 - lane;  // lane j: slice sl - 1 - j
                for (;;) {
                    unsigned long long v = 0, a = 0;
                    if (q >= 0) {
                        v = ld_acquire_u64(&incl[q]);
                        a = ld_acquire_u64(&agg[q]);
                    }
                    const bool hi = q >= 0 && (v & ~0xffffffffull) == tag;
                    const bool ha = q >= 0 && (a & ~0xffffffffull) == tag;
                    const uint32_t mi = __ballot_sync(0xffffffffu, hi), ma = __ballot_sync(0xffffffffu, ha);
                    if (mi) {  // the nearest inclusive prefix, and every aggregate before it
                        const int lim = __ffs(mi) - 1;
                        const uint32_t need = lim ? (1u << lim) - 1 : 0u;
                        if ((ma & need) == need) {
                            uint32_t x = lane < lim ? static_cast<uint32_t>(a)
                                                    : lane == lim ? static_cast<uint32_t>(v) : 0u;
                            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                            base = x;
                            break;
                        }
                    }
                    __nanosleep(32);
                }
                if (lane == 0) st_release_u64(&incl[sl], tag | (base + tot));
            }
            if (lane == 0) {
                s_base = base;
                if (sl == ns - 1) {
                    d.plan_F[nt] = base + tot;
                    d.plan_t0[(base + tot + kScanThreads - 1) / kScanThreads] = nt;  // sentinel
                }
            }
        }
        __syncthreads();
        F += s_base;
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t k = kb + u, len = L[u];
            if (k < nt) {
                d.plan_F[k] = F;
                // tiles whose first chunk falls in this message's range
                for (uint32_t t = (F + kScanThreads - 1) / kScanThreads; len && t * kScanThreads < F + len; ++t)
                    d.plan_t0[t] = k;
            }
            F += len;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(done, 1u);
    }
    TM_END(scan ? 31 : 35);
    if (threadIdx.x == 0) {
        while (ld_acquire(done) < ns) __nanosleep(64);
        s_total = ld_volatile_u32(&d.plan_F[nt]);
    }
    __syncthreads();
    TM_END(scan ? 32 : 36);
    return s_total;
}

// the message holding flattened chunk f of tile t: the last k with
// F[k] <= f (within [t0[t], t0[t+1]] for the global plan; empty ranges share
// their successor's offset and are skipped)
__device__ __forceinline__ uint32_t msg_of_flat(const RxDev& d, const uint32_t* F, uint32_t nt, uint32_t t,
                                                uint32_t f) {
    const bool small = nt <= kPlanSmem;
    uint32_t lo = small ? 0u : d.plan_t0[t], hi = small ? nt : d.plan_t0[t + 1] + 1;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (F[mid] <= f) lo = mid; else hi = mid;
    }
    return lo;
}

// Block-wide segmented inclusive max-scan: segments start where head is
// set (and at thread 0).  Returns this thread's inclusive value.
__device__ __forceinline__ uint32_t block_seg_scan_max(uint32_t v, bool head, uint32_t* s_v, uint32_t* s_h) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t h = head ? 1u : 0u;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yv = __shfl_up_sync(0xffffffffu, v, o);
        const uint32_t yh = __shfl_up_sync(0xffffffffu, h, o);
        if (lane >= o) {
            if (!h) v = v > yv ? v : yv;
            h |= yh;
        }
    }
    if (lane == 31) {
        s_v[w] = v;
        s_h[w] = h;
    }
    __syncthreads();
    if (w == 0) {  // scan the warp totals
        uint32_t x = lane < nw ? s_v[lane] : 0, xh = lane < nw ? s_h[lane] : 1;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yv = __shfl_up_sync(0xffffffffu, x, o);
            const uint32_t yh = __shfl_up_sync(0xffffffffu, xh, o);
            if (lane >= o) {
                if (!xh) x = x > yv ? x : yv;
                xh |= yh;
            }
        }
        if (lane < nw) s_v[lane] = x;
    }
    __syncthreads();
    if (w > 0 && !h) {  // no segment head in this warp up to me: the earlier warps' carry
        const uint32_t p = s_v[w - 1];
        v = v > p ? v : p;
    }
    return v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan(RxDev d) {
    __shared__ uint32_t s_v[32], s_h[32];
    __shared__ uint32_t s_ticket, s_carry, s_k0;
    pdl_wait();
    pdl_launch();
    const int lane = threadIdx.x & 31;
    const uint32_t epoch = d.ctl->epoch;
    const uint32_t nt = min(d.ctl->n_touched, d.plan_cap);
    const uint32_t ppc = d.ppc;
    TM_START(20);
    const uint32_t* __restrict__ cf = first_of(d, d.ctl->par);
    uint32_t my_n = 0;             // first arrivals (n_copied) and their bytes
    unsigned long long my_b = 0;
    __shared__ uint32_t s_F[kPlanSmem + 1];
    const uint32_t* F = nullptr;
    const uint32_t T = plan_batch(d, nt, epoch, true, s_F, &F);
    const uint32_t tiles = (T + kScanThreads - 1) / kScanThreads;
    if (blockIdx.x == 0 && threadIdx.x == 0 && d.ctl->n_touched > d.plan_cap)
        atomicOr(&d.ctl->status, CN_RXF_CAPACITY);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&d.ctl->scan_ticket, 1u);
        __syncthreads();
        const uint32_t ticket = s_ticket;
        if (ticket >= tiles) break;
        const uint32_t f0 = ticket * kScanThreads;
        const uint32_t f = f0 + threadIdx.x;
        const bool in = f < T;
        uint32_t k = 0, c = 0, cpl = 0;
        GenState* G = nullptr;
        if (in) {
            k = msg_of_flat(d, F, nt, ticket, f);
            G = &d.gen[d.touched[k]];
            c = G->cum + (f - F[k]);  // cum: the batch's lower bound (finalize moves it later)
            const uint64_t e = G->chunk_base + c;
            if (!(d.c_flags[e] & CF_COMPLETE)) {
                const uint32_t clen = chunk_len_of(d, G->len, c);
                const uint32_t exp = pkts_of(d, clen);
                const uint32_t seen = d.c_seen[e];
                uint32_t newb = 0, last = 0;
                for (uint32_t q = 0; q < exp; ++q) {
                    uint32_t fa = cf[e * ppc + q];
                    if (fa != kInf) {
                        newb |= 1u << q;
                        last = last > fa ? last : fa;
                        // a first arrival: exactly the packets k_copy scatters
                        const uint32_t rem = clen - q * d.max_pl;
                        ++my_n;
                        my_b += rem < d.max_pl ? rem : d.max_pl;
                    }
                    if ((seen >> q) & 1u) fa = 0;
                    cpl = cpl > fa ? cpl : fa;
                }
                d.c_newb[e] = newb;
                d.c_last[e] = last;
            }
            d.c_cpl[e] = cpl;
        }
        // segments: one per message present in the tile
        const bool head = in && (threadIdx.x == 0 || f == F[k]);
        const uint32_t incl = block_seg_scan_max(cpl, head, s_v, s_h);
        // the message of the tile's first chunk may continue from earlier
        // tiles (it then spans back to tile F / 256): look back for its carry
        if (threadIdx.x < 32) {
            const uint32_t fl_ = (f0 + kScanThreads <= T ? f0 + kScanThreads : T) - 1;
            const uint32_t k0 = msg_of_flat(d, F, nt, ticket, f0), kl = msg_of_flat(d, F, nt, ticket, fl_);
            const bool cont = F[k0] < f0;           // first message started before this tile
            const bool last_here = F[kl] >= f0;     // last message starts in this tile
            // the tile's last segment value: the inclusive scan at its last chunk
            const uint32_t agg = s_v[kScanThreads / 32 - 1];
            uint32_t carry = 0;
            if (last_here && lane == 0) atomicExch(&d.scan_state[ticket], kFlagIncl | agg);
            if (cont) {
                if (!last_here && lane == 0) atomicExch(&d.scan_state[ticket], kFlagAgg | agg);
                int64_t b = static_cast<int64_t>(ticket) - 1;
                const int64_t seg0 = static_cast<int64_t>(F[k0] / kScanThreads);  // the message's first tile
                for (;;) {
                    int64_t p = b - lane;
                    unsigned long long v = p >= seg0 ? ld_volatile_u64(&d.scan_state[p]) : kFlagIncl;
                    unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                    unsigned upto = inc ? ((2u << (__ffs(inc) - 1)) - 1) : 0xffffffffu;
                    unsigned waiting = __ballot_sync(0xffffffffu, (v >> 62) == 0) & upto;
                    if (waiting) {
                        __nanosleep(32);
                        continue;
                    }
                    uint32_t mine = ((upto >> lane) & 1u) ? static_cast<uint32_t>(v) : 0u;
                    mine = __reduce_max_sync(0xffffffffu, mine);
                    carry = carry > mine ? carry : mine;
                    if (inc) break;
                    b -= 32;
                }
                if (!last_here && lane == 0) {
                    __threadfence();
                    atomicExch(&d.scan_state[ticket], kFlagIncl | (agg > carry ? agg : carry));
                }
            }
            if (lane == 0) {
                s_carry = cont ? carry : 0u;
                s_k0 = k0;
            }
        }
        __syncthreads();
        if (in) {
            // the carry belongs to the tile's first message only
            const uint32_t carry = k == s_k0 ? s_carry : 0u;
            const uint32_t pm = incl > carry ? incl : carry;
            d.c_pmax[G->chunk_base + c] = pm;
            if (f + 1 == F[k + 1]) {  // the message's last chunk of the batch range
                const uint32_t hi = c + 1;
                G->deliver_t = hi == G->nchunks ? pm : kInf;
                G->n_init = hi;
            }
        }
        __syncthreads();
    }
    my_n = __reduce_add_sync(0xffffffffu, my_n);
    for (int o = 16; o; o >>= 1) my_b += __shfl_xor_sync(0xffffffffu, my_b, o);
    if (lane == 0 && my_n) {
        atomicAdd(&d.ctl->n_copied, my_n);
        atomicAdd(&d.ctl->bytes_copied, my_b);
    }
    TM_END(21);
}


// -------------------------------------------------------------------- copy
// accept_payload's scatter memcpy (:719-730) for every first-arriving packet
// (duplicates of a seen packet return before it, :677).  Pure streaming:
// one warp per packet, 16-byte vectors, all loads of a packet in flight
// before its stores.  The decision needs only the batch's first[] (final
// after k_ingest), so this kernel does not wait for the ack machinery.
//
// Reduce mode: the scatter is fused
// with the ring reduction step -- dst = dst + payload elementwise (fp32, or
// bf16 with an fp32 add rounded to nearest even), each element exactly
// once, so the result is independent of arrival order.
// Source addressing: payload + i*stride (arrival-order staging), or with
// stride 0 payload + message offset (zero-copy from the sender's message
// buffer, e.g. a peer GPU's memory over NVLink).
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (u >> 16) | 0x40u;  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return u >> 16;
}
// fp32 adds (a NaN sum is the canonical 0x7FFFFFFF), then both halves
// rounded to nearest even by one cvt (canonical NaN 0x7FFF) -- the fold's
// rules (oracle/chunknet_oracle.c)
__device__ __forceinline__ uint32_t add_bf16x2(uint32_t a, uint32_t b) {
    const float lo = __fadd_rn(bf16_lo(a), bf16_lo(b)), hi = __fadd_rn(bf16_hi(a), bf16_hi(b));
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
template <int R>
__device__ __forceinline__ int4 combine(int4 dst, int4 src) {
    if (R == 1) {
        float4 a = *reinterpret_cast<float4*>(&dst), b = *reinterpret_cast<float4*>(&src), c;
        c.x = __fadd_rn(a.x, b.x);
        c.y = __fadd_rn(a.y, b.y);
        c.z = __fadd_rn(a.z, b.z);
        c.w = __fadd_rn(a.w, b.w);
        return *reinterpret_cast<int4*>(&c);
    } else {
        int4 c;
        c.x = static_cast<int>(add_bf16x2(dst.x, src.x));
        c.y = static_cast<int>(add_bf16x2(dst.y, src.y));
        c.z = static_cast<int>(add_bf16x2(dst.z, src.z));
        c.w = static_cast<int>(add_bf16x2(dst.w, src.w));
        return c;
    }
}

template <int R>
__device__ __forceinline__ void warp_scatter(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                             uint32_t len, int lane) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        const uint32_t nv = len >> 4;
        for (uint32_t v0 = 0; v0 < nv; v0 += 32 * kCopyUnroll) {
            int4 r[kCopyUnroll];
            int4 a[R ? kCopyUnroll : 1];
#pragma unroll
            for (int k = 0; k < kCopyUnroll; ++k) {
                uint32_t v = v0 + k * 32 + lane;
                if (v < nv) {
#ifdef CN_COPY_LD_NOALLOC
                {
                    int4 t_;
                    asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(t_.x), "=r"(t_.y), "=r"(t_.z), "=r"(t_.w)
                                 : "l"(s4 + v));
                    r[k] = t_;
                }
#elif defined(CN_COPY_LD_CG)
                    r[k] = __ldcg(s4 + v);
#else
                    r[k] = __ldcs(s4 + v);
#endif
                    if (R) a[R ? k : 0] = __ldcs(d4 + v);  // global (not generic) accesses
                }
            }
#pragma unroll
            for (int k = 0; k < kCopyUnroll; ++k) {
                uint32_t v = v0 + k * 32 + lane;
                if (v < nv) {
                    // streaming stores: the message buffers must not evict the
                    // bookkeeping arrays the concurrent ack kernels walk
                    if (R) __stcs(d4 + v, combine<R ? R : 1>(a[R ? k : 0], r[k]));
                    else __stcs(d4 + v, r[k]);
                }
            }
        }
        const uint32_t tail = nv << 4;
        if (R == 0) {
            for (uint32_t b = tail + lane; b < len; b += 32) dst[b] = src[b];
        } else if (R == 1) {  // 4-byte aligned tail
            for (uint32_t b = tail + 4 * lane; b + 4 <= len; b += 128)
                *reinterpret_cast<float*>(dst + b) =
                    __fadd_rn(*reinterpret_cast<float*>(dst + b), *reinterpret_cast<const float*>(src + b));
        } else {
            for (uint32_t b = tail + 2 * lane; b + 2 <= len; b += 64) {
                uint16_t x = *reinterpret_cast<uint16_t*>(dst + b), y = *reinterpret_cast<const uint16_t*>(src + b);
                *reinterpret_cast<uint16_t*>(dst + b) =
                    static_cast<uint16_t>(bf16_rne(__fadd_rn(bf16_lo(x), bf16_lo(y))));
            }
        }
    } else if (R == 0) {
        for (uint32_t b = lane; b < len; b += 32) dst[b] = src[b];
    } else if (R == 1) {
        for (uint32_t b = 4 * lane; b + 4 <= len; b += 128) {
            float x, y;
            memcpy(&x, dst + b, 4);
            memcpy(&y, src + b, 4);
            x = __fadd_rn(x, y);
            memcpy(dst + b, &x, 4);
        }
    } else {
        for (uint32_t b = 2 * lane; b + 2 <= len; b += 64) {
            uint16_t x, y;
            memcpy(&x, dst + b, 2);
            memcpy(&y, src + b, 2);
            uint16_t z = static_cast<uint16_t>(bf16_rne(__fadd_rn(bf16_lo(x), bf16_lo(y))));
            memcpy(dst + b, &z, 2);
        }
    }
}

template <int R>
// reduce modes: 3 blocks per SM (80 registers, a few bytes spilled) beat 2
// (105 registers): fp32 0.149 -> 0.130 ms on the 4 x 64 MiB batch
__global__ void __launch_bounds__(256, R ? 3 : CN_COPY_MINB) k_copy(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                              const uint8_t* __restrict__ payload, uint64_t stride,
                                              uint32_t n) {
    const int lane = threadIdx.x & 31;
    TM_START(24);
    RxCtl* C = d.ctl;
    const uint32_t par = C->cq[C->cq_out & 3];
    const uint32_t* __restrict__ cf = first_of(d, par);
    const unsigned long long* __restrict__ pd = d.p_dst + par * static_cast<uint64_t>(d.max_batch);
    const uint32_t* __restrict__ pf = d.p_fi + par * static_cast<uint64_t>(d.max_batch);
    const unsigned long long* __restrict__ md = d.msgdata;
    const unsigned long long* __restrict__ po = d.poff;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
        // k_ingest's descriptor: only packets not seen before the batch, of
        // a live message (GenStates may be reused while a pipelined scatter
        // still runs, so the destination travels with the packet)
#ifndef CN_COPY_LAZY_HDR
        // every load but the first-arrival test's is independent: issued together
        const unsigned long long dst = pd[i];
        const uint32_t fi = pf[i];
        const unsigned long long mdv = md ? md[i] : 0;
        const cn_pkt_hdr* hp = hdrs + i;
        const uint32_t len = hp->payload_len;
        const uint64_t moff = hp->chunk_offset + static_cast<uint64_t>(hp->seq_in_chunk) * d.max_pl;
        // first arrival within the batch: c_first is final after k_ingest
        // (fi is 0 for a packet without a descriptor: a valid index)
        if (cf[fi] != i + 1 || !dst) continue;
#else
        const unsigned long long dst = pd[i];
        const uint32_t fi = pf[i];
        if (cf[fi] != i + 1 || !dst) continue;
        const unsigned long long mdv = md ? md[i] : 0;
        const cn_pkt_hdr* hp = hdrs + i;
        const uint32_t len = hp->payload_len;
        const uint64_t moff = hp->chunk_offset + static_cast<uint64_t>(hp->seq_in_chunk) * d.max_pl;
#endif
        const uint8_t* src = po    ? payload + po[i]
                             : md   ? reinterpret_cast<const uint8_t*>(mdv) + moff
                             : stride ? payload + static_cast<uint64_t>(i) * stride : payload + moff;
        if (md && !mdv) continue;  // no message data: accepted, nothing to copy (transport.cpp:722)
        warp_scatter<R>(reinterpret_cast<uint8_t*>(dst), src, len, lane);
    }
    TM_END(25);
    // the last block pops the part queue (every block has read it by now)
    if (threadIdx.x == 0 && atomicAdd(&C->cq_done, 1u) == gridDim.x - 1) {
        C->cq_done = 0;
        C->cq_out += 1;
    }
}

// What the reference does with packet i (handle_data's branches).  Every
// load that does not depend on an earlier one is issued up front: the
// kernel is latency-bound and usually shares HBM with the scatter.
__device__ __forceinline__ uint32_t pmax_ld(const RxDev& d, uint64_t cbase, uint32_t cum, uint32_t n_init,
                                            uint64_t x) {
    return x < cum ? 0u : x >= n_init ? kInf : d.c_pmax[cbase + x];
}
// The copy-mode scatter on the bulk-copy engine: persistent blocks of one
// warp, kTmaSlots lanes each owning a shared-memory slot.  Per packet the
// lane issues a bulk load of its 16-byte-multiple body into the slot (an
// mbarrier counts the bytes), prefetches its next packet's descriptor while
// the load flies, then issues the bulk store from the slot; the next load
// into the slot waits only for that store to have READ the slot.  The
// scatter thus holds 2 x 148 warps instead of thousands, and the
// latency-bound ack path beside it keeps the SMs' issue slots.  Bytes past
// the last 16-byte multiple, and packets whose source or destination is not
// 16-byte aligned (chunk sizes that are not multiples of 16), take the
// warp-cooperative vector path.
constexpr int kTmaLanes = 16;             // lanes with slots (the other 16 help with misaligned packets)
constexpr int kTmaBufs = 2;               // slots per lane: the next load flies while the current one lands
constexpr uint32_t kTmaSlotBytes = 4096;  // >= max_payload, multiple of 16
constexpr uint32_t kTmaSmem = kTmaLanes * kTmaBufs * kTmaSlotBytes;

struct TmaPkt {
    unsigned long long dst;
    const uint8_t* src;
    uint32_t len;
    bool bulk;
};

__global__ void __launch_bounds__(32) k_copy_tma(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                                 const uint8_t* __restrict__ payload, uint64_t stride,
                                                 uint32_t n) {
    extern __shared__ __align__(128) uint8_t tma_buf[];
    __shared__ __align__(8) uint64_t tma_bar[kTmaLanes * kTmaBufs];
    const int lane = threadIdx.x;
    TM_START(24);
    RxCtl* C = d.ctl;
    const uint32_t par = C->cq[C->cq_out & 3];
    const uint32_t* __restrict__ cf = first_of(d, par);
    const unsigned long long* __restrict__ pd = d.p_dst + par * static_cast<uint64_t>(d.max_batch);
    const uint32_t* __restrict__ pf = d.p_fi + par * static_cast<uint64_t>(d.max_batch);
    const bool act = lane < kTmaLanes;
    const int ln = act ? lane : 0;
    uint32_t slot[kTmaBufs], bar[kTmaBufs], phase[kTmaBufs];
#pragma unroll
    for (int q = 0; q < kTmaBufs; ++q) {
        slot[q] = smem_u32(tma_buf + (ln * kTmaBufs + q) * kTmaSlotBytes);
        bar[q] = smem_u32(&tma_bar[ln * kTmaBufs + q]);
        phase[q] = 0;
        if (act) mbar_init(bar[q], 1);
    }
    fence_mbar_init();
    __syncwarp();
    const uint64_t pol = l2_evict_first();
    // this lane's packet: k_ingest's descriptor, the first-arrival test, the header fields
    auto prep = [&](uint32_t i) {
        TmaPkt p{0, nullptr, 0, false};
        if (!act || i >= n) return p;
        const unsigned long long d0 = pd[i];
        const uint32_t fi = pf[i];
        const cn_pkt_hdr* hp = hdrs + i;
        const uint32_t l = hp->payload_len;
        const uint64_t mo = hp->chunk_offset + static_cast<uint64_t>(hp->seq_in_chunk) * d.max_pl;
        if (cf[fi] != i + 1 || !d0) return p;
        const unsigned long long mdv = d.msgdata ? d.msgdata[i] : 0;
        if (d.msgdata && !mdv) return p;  // no message data: nothing to copy
        p.dst = d0;
        p.len = l;
        p.src = d.poff      ? payload + d.poff[i]
                : d.msgdata ? reinterpret_cast<const uint8_t*>(mdv) + mo
                : stride    ? payload + static_cast<uint64_t>(i) * stride : payload + mo;
        p.bulk = (l & ~15u) && !((reinterpret_cast<uintptr_t>(p.src) | d0) & 15);
        return p;
    };
    uint32_t uses = 0;  // bulk loads issued by this lane (slot = uses % kTmaBufs)
    bool stored = false;
    auto issue = [&](const TmaPkt& p) {
        if (!p.bulk) return;
        const int q = uses % kTmaBufs;
        // the slot's previous store (kTmaBufs loads ago) must have read it: with
        // two slots that is the most recent committed store
        if (stored) bulk_wait_read0();
        mbar_arrive_expect_tx(bar[q], p.len & ~15u);
        bulk_g2s(slot[q], p.src, p.len & ~15u, bar[q], pol);
        ++uses;
    };
    const uint32_t step = gridDim.x * kTmaLanes;
    uint32_t i = blockIdx.x * kTmaLanes + lane;
    TmaPkt cur = prep(i);
    issue(cur);
    TmaPkt nxt = prep(i + step);
    for (uint32_t base = blockIdx.x * kTmaLanes; base < n; base += step) {
        // the next packet's load joins the current one in flight
        issue(nxt);
        const TmaPkt nn = prep(i + 2 * step);
        if (cur.bulk) {
            const uint32_t len16 = cur.len & ~15u;
            for (uint32_t b = len16; b < cur.len; ++b) reinterpret_cast<uint8_t*>(cur.dst)[b] = cur.src[b];
        }
        // misaligned packets (chunk sizes not a multiple of 16): the whole warp
        unsigned fb = __ballot_sync(0xffffffffu, cur.dst && !cur.bulk);
        while (fb) {
            const int l = __ffs(fb) - 1;
            fb &= fb - 1;
            const unsigned long long fd = __shfl_sync(0xffffffffu, cur.dst, l);
            const unsigned long long fs = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(cur.src), l);
            const uint32_t fl = __shfl_sync(0xffffffffu, cur.len, l);
            warp_scatter<0>(reinterpret_cast<uint8_t*>(fd), reinterpret_cast<const uint8_t*>(fs), fl, lane);
        }
        if (cur.bulk) {
            // cur's load is the one issued before nxt's
            const int q = (uses - (nxt.bulk ? 2 : 1)) % kTmaBufs;
            mbar_wait(bar[q], phase[q]);
            phase[q] ^= 1u;
            bulk_s2g(reinterpret_cast<void*>(cur.dst), slot[q], cur.len & ~15u, pol);
            bulk_commit();
            stored = true;
        }
        i += step;
        cur = nxt;
        nxt = nn;
    }
    bulk_wait_all();
    TM_END(25);
    __syncwarp();
    if (lane == 0 && atomicAdd(&C->cq_done, 1u) == gridDim.x - 1) {  // pops the part queue
        C->cq_done = 0;
        C->cq_out += 1;
    }
}

// What decide() learned about an ack-emitting packet, kept in shared memory
// for build_ack (the header, its message's state, chunk c): the ack
// snapshot then takes two dependent round trips.
struct AckCtx {
    unsigned long long cbase, seq, len;  // chunk base, msg_seq (G's; the header's if stale), msg length
    uint32_t c, cum0, n_init, hdr;       // chunk, cursor before the batch, chunk vector size, wire header
    int32_t src, dst;
    uint8_t msg_id, exp, flags, pad;     // exp = packets of chunk c; flags = header flags
};

__device__ __forceinline__ uint8_t decide(const RxDev& d, const cn_pkt_hdr* __restrict__ hdrs,
                                          uint32_t i, uint32_t* st, uint64_t* e_out, uint32_t* pmc,
                                          AckCtx* x) {
    const uint32_t g = d.p_gen[i];
    const cn_pkt_hdr* hp = hdrs + i;
    const uint64_t off = hp->chunk_offset;
    const uint32_t s = hp->seq_in_chunk;
    const uint8_t hfl = hp->flags;
    x->hdr = hp->hdr;
    x->src = hp->src;
    x->dst = hp->dst;
    x->seq = hp->msg_seq;
    x->flags = hfl;
    const uint32_t t = i + 1;
    if (d.ordered && d.p_gbn[i]) return d.p_gbn[i] == 2 ? PC_NACK : 0;  // decided by k_gbn
    if (hfl & CN_PKT_TRIMMED) return d.p_nack[i] ? PC_NACK : 0;  // decided by k_trim
    if (g == kStale) return PC_STALE;  // transport.cpp:602-615
    if (g == kErr) return 0;
    const GenState& G = d.gen[g];
    const uint32_t dt = G.deliver_t, cum = G.cum, n_init = G.n_init;
    const uint64_t cbase = G.chunk_base;
    const uint64_t c = off / d.cb;
    const uint64_t e = cbase + c;
    *e_out = e;
    const uint32_t fl = d.c_flags[e], cpl0 = d.c_cpl[e], seen = d.c_seen[e];
    const uint32_t first = d.c_first[e * d.ppc + s];
    const uint32_t pm0 = pmax_ld(d, cbase, cum, n_init, c);
    const uint32_t pm1 = pmax_ld(d, cbase, cum, n_init, c + 128);
    const uint32_t pm2 = c >= 128 ? pmax_ld(d, cbase, cum, n_init, c - 128) : 0u;
    *pmc = pm0;
    if (t > dt) return PC_STALE;
    x->cbase = cbase;
    x->seq = G.seq;
    x->len = G.len;
    x->c = static_cast<uint32_t>(c);
    x->cum0 = cum;
    x->n_init = n_init;
    x->msg_id = static_cast<uint8_t>(G.msg_id);
    x->exp = static_cast<uint8_t>(pkts_of(d, chunk_len_of(d, G.len, c)));
    uint8_t cls = 0;
    const uint32_t cpl = (fl & CF_COMPLETE) ? 0 : cpl0;
    if (cpl < t) {
        cls = PC_ACK;  // complete chunk (:651-655) or behind the cursor (:631-634)
    } else if (cpl == t) {
        cls = PC_ACK | PC_COPY;  // completes its chunk (:686-687)
        if (t == dt) cls |= PC_DELIVER;
    } else if (!((seen >> s) & 1u) && first == t) {
        cls = PC_COPY;  // new packet of an open chunk: silent
    }
    // The reference unwraps the 8-bit csn against the cursor (:629-636):
    // verify it names chunk c (no aliasing) -- DESIGN.md §3.
    if (pm0 < t) {
        if (pm1 < t) *st |= CN_RXF_ALIAS;
    } else if (c >= 128 && pm2 >= t) {
        *st |= CN_RXF_ALIAS;
    }
    return cls;
}

// -------------------------------------------------------------------- trim
// Trimmed headers (trim queue mode; handle_data :596-674): a trimmed packet
// of an open chunk emits a NACK unless the chunk is already `nacked` -- set
// by a trimmed header, cleared by every new data packet (:658-660, :679).
// Within a batch that is an order question per chunk: the header at time t
// NACKs iff no trimmed header of its chunk arrived since the chunk's last
// new packet before t (or, with none in the batch, the chunk was not left
// nacked by an earlier batch).  Trimmed headers are rare, so one block sorts
// them by (chunk, time) and decides each from its predecessor; the decision
// feeds k_acks, which orders the NACK records into the ack stream.
__global__ void __launch_bounds__(1024) k_trim(RxDev d, const cn_pkt_hdr* __restrict__ hdrs) {
    pdl_wait();
    pdl_launch();
    extern __shared__ unsigned long long key[];  // [kTrimMax]
    const uint32_t m0 = d.ctl->n_trim;
    const uint32_t m = m0 < kTrimMax ? m0 : kTrimMax;
    if (m == 0) return;
    uint32_t P = 1;
    while (P < m) P <<= 1;
    for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) {
        unsigned long long v = ~0ull;
        if (k < m) {
            const uint32_t i = d.trim_list[k];
            const uint32_t g = d.p_gen[i];
            if (g < kErr)
                v = ((d.gen[g].chunk_base + hdrs[i].chunk_offset / d.cb) << 32) | (i + 1);
        }
        key[k] = v;
    }
    __syncthreads();
    for (uint32_t sz = 2; sz <= P; sz <<= 1)  // bitonic sort, ascending
        for (uint32_t j = sz >> 1; j > 0; j >>= 1) {
            for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) {
                const uint32_t l = k ^ j;
                if (l > k) {
                    const unsigned long long a = key[k], b = key[l];
                    const bool up = (k & sz) == 0;
                    if ((a > b) == up) {
                        key[k] = b;
                        key[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    uint32_t st = 0;
    for (uint32_t k = threadIdx.x; k < m; k += blockDim.x) {
        const unsigned long long v = key[k];
        if (v == ~0ull) continue;
        const uint64_t e = v >> 32;
        const uint32_t t = static_cast<uint32_t>(v), i = t - 1;
        const uint32_t prev_t = (k > 0 && (key[k - 1] >> 32) == e) ? static_cast<uint32_t>(key[k - 1]) : 0;
        const bool last = k + 1 == m || (key[k + 1] >> 32) != e;
        const GenState& G = d.gen[d.p_gen[i]];
        const uint64_t c = e - G.chunk_base;
        const uint32_t fl = d.c_flags[e];
        // stale generation (:603), complete or behind the cursor (:629-634, :651-655): silent
        bool silent = t > G.deliver_t || ((fl & CF_COMPLETE) ? true : d.c_cpl[e] < t);
        // the csn must name chunk c (no aliasing), as in decide()
        const uint32_t pm0 = pmax_ld(d, G.chunk_base, G.cum, G.n_init, c);
        if (pm0 < t) {
            if (pmax_ld(d, G.chunk_base, G.cum, G.n_init, c + 128) < t) st |= CN_RXF_ALIAS;
        } else if (c >= 128 && pmax_ld(d, G.chunk_base, G.cum, G.n_init, c - 128) >= t) {
            st |= CN_RXF_ALIAS;
        }
        if (!silent) {
            uint32_t L = 0;  // the chunk's last new packet before t in this batch
            const uint32_t exp = pkts_of(d, chunk_len_of(d, G.len, c));
            for (uint32_t q = 0; q < exp; ++q) {
                const uint32_t f = first_of(d, d.ctl->par)[e * d.ppc + q];
                if (f < t && f > L) L = f;
            }
            const bool nacked = prev_t > L || (L == 0 && prev_t == 0 && (fl & CF_NACKED));
            if (!nacked) d.p_nack[i] = 1;
        }
        if (last && !(fl & CF_COMPLETE) && t > d.c_last[e]) atomicOr(&d.c_newfl[e], CF_NACKSET);
    }
    if (st) atomicOr(&d.ctl->status, st);
}

// -------------------------------------------------------------------- acks
// Persistent blocks pull 128-packet tiles by ticket.  Per tile: 4 warps
// decide (one lane per packet) and compact the tile's ack and completion
// packets into lists; warp 0 orders the tile's counts with a warp-parallel
// decoupled look-back while the other warps build the ack snapshots
// (send_ack :763-792, stale re-ack :602-615) round-robin, one warp per ack;
// then the records are written to their stream positions, with completion
// records (maybe_deliver :794-803).

// cum after packet t: the first x in [lo, hi) with pmax[x] > t (pmax is
// non-decreasing over [cum0, n_init)), by 32-ary bisection
__device__ __forceinline__ uint32_t first_above(const uint32_t* __restrict__ pm, uint32_t lo, uint32_t hi,
                                                uint32_t t, int lane) {
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + (lane + 1) * step - 1;
        const bool ok = p < hi && pm[p] <= t;
        const uint32_t k = __popc(__ballot_sync(0xffffffffu, ok));
        lo += k * step;
        hi = hi < lo + step ? hi : lo + step;
    }
    const bool okc = lo + lane < hi && pm[lo + lane] <= t;
    return lo + __popc(__ballot_sync(0xffffffffu, okc));
}

__device__ __forceinline__ void build_ack(const RxDev& d, const cn_pkt_hdr* __restrict__ hdrs,
                                          uint32_t i, uint8_t cls, uint32_t pmc, const AckCtx& x, int lane,
                                          cn_ack_rec* out) {
    const uint32_t t = i + 1;
    const uint32_t csn = (x.hdr >> 9) & 0xFF;
    if (cls & (PC_STALE | PC_NACK)) {  // stale re-ack (:602-615) / trimmed-header NACK (:657-674)
        if (lane == 0) {
            cn_ack_rec r;
            memset(&r, 0, sizeof r);
            r.src = x.dst;
            r.dst = x.src;
            r.hdr = x.hdr;
            r.cum_csn = static_cast<uint8_t>(csn);
            r.flags = (cls & PC_NACK) ? CN_ACK_NACK : CN_ACK_CUM_VALID;
            r.pkt_index = i;
            r.msg_seq = x.seq;
            if ((cls & PC_NACK) && d.ordered) {  // sequence-gap NACK (:695-707): nack_psn, no csn / seq
                r.cum_csn = 0;
                r.msg_seq = 0;
                r.flags = CN_ACK_NACK | CN_ACK_GBN | ((x.flags & CN_PKT_TRIMMED) ? CN_ACK_NACK_TRIM : 0);
                r.sack[0] = d.p_gbn_psn[i];
            }
            *out = r;
        }
        return;
    }
    const uint32_t cum0 = x.cum0, n_init = x.n_init;
    const uint64_t cbase = x.cbase;
    const uint32_t* pm = d.c_pmax + cbase;
    const uint32_t c = x.c;
    const uint32_t par = d.ctl->par;
    // round trip 1: the cursor's 32-chunk window beside c, and chunk c's
    // state -- the echo chunk whenever the ack carries an echo (below)
    const uint64_t Ec = cbase + c;
    uint32_t fl = d.c_flags[Ec], cinit = d.c_init[Ec], seen = d.c_seen[Ec];
    int64_t txt0 = d.c_txt[Ec];
    int32_t path0 = d.c_path[Ec];
    uint32_t f0 = static_cast<uint32_t>(lane) < x.exp ? first_of(d, par)[Ec * d.ppc + lane] : kInf;
    // cum after this packet, searched outward from the packet's own chunk c
    // (pmax[c] came from decide): usually one 32-chunk window decides it
    uint32_t cum;
    if (pmc <= t) {  // the cursor is past c: scan upward from c + 1
        const uint32_t y = c + 1 + lane;
        const bool le = y < cum0 || (y < n_init && pm[y] <= t);
        const unsigned b = __ballot_sync(0xffffffffu, le);
        cum = b != 0xffffffffu ? c + 1 + __popc(b)
                               : first_above(pm, c + 33 > cum0 ? c + 33 : cum0, n_init, t, lane);
    } else {  // the cursor is at or before c: scan downward from c
        const int64_t y = static_cast<int64_t>(c) - 32 + lane;
        const bool gt = y >= static_cast<int64_t>(cum0) && pm[y] > t;
        const unsigned b = __ballot_sync(0xffffffffu, gt);
        if ((b & 1u) && static_cast<int64_t>(c) - 32 > static_cast<int64_t>(cum0))
            cum = first_above(pm, cum0, c - 32, t, lane);
        else
            cum = b ? c - 32 + (__ffs(b) - 1) : c;
    }
    // echo of chunk cum + uint8(cause - uint8(cum)) (:781-789): with an
    // echo (offset < 128) that is chunk c itself, as the cursor moves at
    // most a window per packet; anything else reloads (kept exact)
    const uint32_t rel = (csn - (cum & 0xFF)) & 0xFF;
    const uint32_t ei = cum + rel;
    const bool echo = rel < CN_CSN_WINDOW && ei < n_init;
    uint32_t exp = x.exp;
    if (echo && ei != c) {
        const uint64_t E = cbase + ei;
        exp = pkts_of(d, chunk_len_of(d, x.len, ei));
        fl = d.c_flags[E];
        cinit = d.c_init[E];
        seen = d.c_seen[E];
        txt0 = d.c_txt[E];
        path0 = d.c_path[E];
        f0 = static_cast<uint32_t>(lane) < exp ? first_of(d, par)[E * d.ppc + lane] : kInf;
    }
    const bool live = echo && ((fl & CF_INIT) || cinit <= t);
    const uint32_t f = ((seen >> lane) & 1u) ? kInf : f0;
    const bool fok = live && f <= t;
    const uint32_t lastf = __reduce_max_sync(0xffffffffu, fok ? f : 0u);
    // round trip 2: the 128-bit SACK, bit j = chunk cum+j complete
    // (:775-779), and the headers of the echo chunk's new packets
    const uint32_t* cp = d.c_cpl + cbase;
    uint32_t cv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t y = cum + q * 32 + lane;
        cv[q] = y < n_init ? cp[y] : kInf;
    }
    const uint8_t pfl = fok ? hdrs[f - 1].flags : 0;
    int64_t etxt = 0;
    int32_t epath = 0;
    if (lastf) {
        etxt = hdrs[lastf - 1].tx_time;
        epath = hdrs[lastf - 1].path_id;
    } else if (live) {
        etxt = txt0;
        epath = path0;
    }
    uint32_t sw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sw[q] = __ballot_sync(0xffffffffu, cv[q] <= t);
    const unsigned eb = __ballot_sync(0xffffffffu, fok && (pfl & CN_PKT_ECN));
    const uint32_t eecn = live && ((eb != 0) || (fl & CF_ECN));
    if (lane == 0) {
        cn_ack_rec r;
        memset(&r, 0, sizeof r);
        r.src = x.dst;
        r.dst = x.src;
        r.hdr = enc_hdr(x.hdr >> 24, x.msg_id, csn, 0, 0);
        r.echo_path_id = epath;
        r.cum_csn = static_cast<uint8_t>((cum - 1) & 0xFF);
        r.flags = (cum > 0 ? CN_ACK_CUM_VALID : 0) | (eecn ? CN_ACK_ECN_ECHO : 0);
        r.pkt_index = i;
        r.msg_seq = x.seq;
        r.sack[0] = sw[0] | (static_cast<uint64_t>(sw[1]) << 32);
        r.sack[1] = sw[2] | (static_cast<uint64_t>(sw[3]) << 32);
        r.echo_tx_time = etxt;
        *out = r;
    }
}

// TILE packets per tile: 128 for large batches; 32 for small ones, so that a
// batch of a few thousand acks spreads over many blocks instead of making
// 8 warps per tile build 16 acks each in turn
template <int TILE>
__global__ void __launch_bounds__(kAckWarps * 32) k_acks(
    RxDev d, const cn_pkt_hdr* __restrict__ hdrs, uint32_t n, cn_ack_rec* __restrict__ acks,
    uint32_t max_acks, cn_completion* __restrict__ cpls, uint32_t max_cpls) {
    constexpr int kAckTile = TILE;
    constexpr int kDecideWarps = kAckTile / 32;
    __shared__ cn_ack_rec s_rec[kAckTile];
    __shared__ uint8_t s_cls[kAckTile];
    __shared__ uint32_t s_g[kAckTile], s_pm[kAckTile];
    __shared__ AckCtx s_ctx[kAckTile];
    __shared__ uint16_t s_alist[kAckTile], s_clist[kAckTile];
    __shared__ uint32_t s_wa[kDecideWarps], s_wc[kDecideWarps];
    __shared__ uint32_t s_tile, s_base_a, s_base_c;
    pdl_wait();
    pdl_launch();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tiles = (n + kAckTile - 1) / kAckTile;
    TM_START(22);
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&d.ctl->tile_ticket, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= tiles) break;
        TM_TILE(0, tile);
        const uint32_t i0 = tile * kAckTile;
        uint8_t cls = 0;
        unsigned ab = 0, cb = 0;
        if (warp < kDecideWarps) {
            uint32_t st = 0;
            uint64_t e = 0;
            const uint32_t j = warp * 32 + lane;
            const uint32_t i = i0 + j;
            uint32_t pmc = 0;
            AckCtx x;
            if (i < n) cls = decide(d, hdrs, i, &st, &e, &pmc, &x);
            if (cls & (PC_STALE | PC_ACK | PC_NACK)) s_ctx[j] = x;
            if (cls & PC_COPY) {  // ChunkRx::ecn / any_rtx of new packets (:680-681)
                const uint8_t pf = hdrs[i].flags;
                const uint32_t b = ((pf & CN_PKT_ECN) ? CF_ECN : 0) | ((pf & CN_PKT_RTX) ? CF_RTX : 0);
                if (b) atomicOr(&d.c_newfl[e], b);
            }
            ab = __ballot_sync(0xffffffffu, cls & (PC_STALE | PC_ACK | PC_NACK));
            cb = __ballot_sync(0xffffffffu, cls & PC_DELIVER);
            s_cls[j] = cls;
            s_pm[j] = pmc;
            if (i < n) s_g[j] = d.p_gen[i];
            if (lane == 0) {
                s_wa[warp] = __popc(ab);
                s_wc[warp] = __popc(cb);
            }
            st = __reduce_or_sync(0xffffffffu, st);
            if (lane == 0 && st) atomicOr(&d.ctl->status, st);
        }
        __syncthreads();
        TM_TILE(1, tile);
        uint32_t na = 0, nc = 0;
        for (int w = 0; w < kDecideWarps; ++w) {
            na += s_wa[w];
            nc += s_wc[w];
        }
        if (warp < kDecideWarps) {  // compact the tile's ack / completion packets
            uint32_t pa = 0, pc = 0;
            for (int w = 0; w < warp; ++w) {
                pa += s_wa[w];
                pc += s_wc[w];
            }
            const unsigned lt = (1u << lane) - 1;
            const uint16_t j = static_cast<uint16_t>(warp * 32 + lane);
            if ((ab >> lane) & 1u) s_alist[pa + __popc(ab & lt)] = j;
            if ((cb >> lane) & 1u) s_clist[pc + __popc(cb & lt)] = j;
        }
        if (warp == 0) {
            const unsigned long long agg = na | (static_cast<unsigned long long>(nc) << 31);
            unsigned long long pre = 0;
            if (tile == 0) {
                if (lane == 0) atomicExch(&d.tile_state[0], kFlagIncl | agg);
            } else {
                if (lane == 0) atomicExch(&d.tile_state[tile], kFlagAgg | agg);
                // warp-parallel look-back: lane l inspects tile (base - l)
                int64_t base = static_cast<int64_t>(tile) - 1;
                for (;;) {
                    const int64_t p = base - lane;
                    const unsigned long long v = p >= 0 ? ld_volatile_u64(&d.tile_state[p]) : kFlagIncl;
                    const unsigned incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                    const unsigned upto = incl ? ((2u << (__ffs(incl) - 1)) - 1) : 0xffffffffu;
                    const unsigned waiting = __ballot_sync(0xffffffffu, (v >> 62) == 0) & upto;
                    if (waiting) {
                        __nanosleep(32);
                        continue;
                    }
                    unsigned long long mine = ((upto >> lane) & 1u) ? (v & ~(3ull << 62)) : 0ull;
                    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
                    pre += mine;
                    if (incl) break;
                    base -= 32;
                }
                if (lane == 0) {
                    __threadfence();
                    atomicExch(&d.tile_state[tile], kFlagIncl | (agg + pre));
                }
            }
            if (lane == 0) {
                s_base_a = static_cast<uint32_t>(pre & 0x7FFFFFFFu);
                s_base_c = static_cast<uint32_t>(pre >> 31);
                if (tile == tiles - 1) {
                    const unsigned long long tot = agg + pre;
                    const uint32_t ta = static_cast<uint32_t>(tot & 0x7FFFFFFFu);
                    const uint32_t tc = static_cast<uint32_t>(tot >> 31);
                    d.ctl->n_acks = ta;
                    d.ctl->n_cpls = tc;
                    if (ta > max_acks || tc > max_cpls) atomicOr(&d.ctl->status, CN_RXF_CAPACITY);
                }
            }
        }
        __syncthreads();  // s_alist / s_clist complete
        // acks round-robin over the warps, warp 0 (busy looking back) last
        for (uint32_t k = kAckWarps - 1 - warp; k < na; k += kAckWarps) {
            const uint32_t j = s_alist[k];
            build_ack(d, hdrs, i0 + j, s_cls[j], s_pm[j], s_ctx[j], lane, &s_rec[k]);
        }
        __syncthreads();
        TM_TILE(2, tile);
        for (uint32_t k = warp; k < na; k += kAckWarps) {
            const uint32_t a = s_base_a + k;
            if (lane < 16 && a < max_acks)
                reinterpret_cast<uint32_t*>(&acks[a])[lane] = reinterpret_cast<const uint32_t*>(&s_rec[k])[lane];
        }
        for (uint32_t k = threadIdx.x; k < nc; k += kAckWarps * 32) {
            const uint32_t i = i0 + s_clist[k];
            const uint32_t a = s_base_c + k;
            if (a < max_cpls) {
                const GenState& G = d.gen[d.p_gen[i]];
                cn_completion c;
                memset(&c, 0, sizeof c);
                c.tag = G.tag;
                c.src = hdrs[i].src;
                c.dst = hdrs[i].dst;
                c.len = G.len;
                c.msg_seq = G.seq;
                c.pkt_index = i;
                c.msg_id = G.msg_id;
                c.buf_offset = d.carry ? G.buf_off : ~0ull;
                c.reserved = reinterpret_cast<uint64_t>(G.buf);  // absolute device pointer
                c.bytes = G.len;  // every byte accepted exactly once
                cpls[a] = c;
            }
        }
        __syncthreads();  // shared lists are reused by the next tile
        TM_TILE(3, tile);
    }
    TM_END(23);
}

// One arena release entry (start << 31 | blocks), a warp's lanes over its
// bit words: ring positions [a0, a0 + n0) mod arena_blocks, at most two runs.
__device__ __forceinline__ void arena_release(const RxDev& d, unsigned long long v, int lane) {
    const uint64_t a0 = v >> 31, n0 = v & 0x7FFFFFFF;
    for (int part = 0; part < 2; ++part) {
        const uint64_t a = part ? 0 : a0;
        const uint64_t e0 = a0 + n0 > d.arena_blocks ? d.arena_blocks : a0 + n0;
        const uint64_t end = part ? (a0 + n0 > d.arena_blocks ? a0 + n0 - d.arena_blocks : 0) : e0;
        for (uint64_t w = (a >> 5) + lane; (w << 5) < end; w += 32) {
            const uint64_t lo_ = (w << 5) > a ? (w << 5) : a, hi_ = (w << 5) + 32 < end ? (w << 5) + 32 : end;
            const uint32_t m = (hi_ - lo_ == 32 ? ~0u : ((1u << (hi_ - lo_)) - 1)) << (lo_ - (w << 5));
            atomicXor(&d.arena_bits[w], m);  // lap-parity release
        }
    }
}

// ---------------------------------------------------------------- finalize
// Same tiles: fold batch scratch into persistent per-chunk state
// (pkts_seen, complete, init, ecn, any_rtx, tx_time/path of the last new
// packet, :678-683).  The last tile of a message advances its cum and
// retires it if delivered (completed_seq, :801); the last block of the
// grid publishes the batch result and arms the next batch.
__global__ void __launch_bounds__(kScanThreads) k_finalize(RxDev d, const cn_pkt_hdr* __restrict__ hdrs,
                                                           cn_rx_result* res) {
    __shared__ uint32_t s_ticket;
    __shared__ bool last_block;
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_cnt[kScanThreads];  // per message segment of the tile: chunks now in the cum prefix
    pdl_wait();
    const uint32_t nt = min(d.ctl->n_touched, d.plan_cap);
    const uint32_t ppc = d.ppc;
    const uint32_t par = d.ctl->par;
    __shared__ uint32_t s_F[kPlanSmem + 1];
    const uint32_t* F = nullptr;
    const uint32_t T = plan_batch(d, nt, 0, false, s_F, &F);
    const uint32_t total = (T + kScanThreads - 1) / kScanThreads;
    TM_START(0);
    // the previous batch's first-arrival half: its scatter has finished
    // (stream order), the next batch uses it
    {
        const uint32_t nxt = par == 2 ? 0u : par + 1;  // batch k - 2's part, batch k + 1's
        uint32_t* cf1 = first_of(d, nxt);
        const unsigned long long* dl = d.dirty + nxt * static_cast<uint64_t>(d.dirty_cap);
        const uint32_t nd = d.ctl->n_dirty[nxt];
        // phases go to different blocks (tiles are taken by ticket, usually
        // by the first blocks): dirty lists from a third of the grid on,
        // arena releases from two thirds, retirement from the middle
        // a warp takes up to 32 entries (one coalesced load; fewer when the
        // list is short, so large runs spread over the grid) and clears each
        // entry's contiguous run of chunks x ppc slots across its lanes
        const int lane = threadIdx.x & 31;
        const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
        const uint32_t gw = (((blockIdx.x + gridDim.x - gridDim.x / 3) % gridDim.x) * blockDim.x + threadIdx.x) >> 5;
        const uint32_t per = min(32u, (nd + nwarps - 1) / nwarps);
        for (uint32_t j0 = gw * per; j0 < nd; j0 += nwarps * per) {
            const unsigned long long vl = j0 + lane < nd && lane < per ? dl[j0 + lane] : 0ull;
            const uint32_t m = min(per, nd - j0);
            for (uint32_t e = 0; e < m; ++e) {
                const unsigned long long v = __shfl_sync(0xffffffffu, vl, e);
                uint32_t* p0 = cf1 + (v >> 9) * ppc;
                const uint32_t nq = static_cast<uint32_t>(v & 511) * ppc;
                for (uint32_t q = lane; q < nq; q += 32) p0[q] = kInf;
            }
        }
    }
    TM_END(1);
    unsigned long long* dirty = d.dirty + par * static_cast<uint64_t>(d.dirty_cap);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&d.ctl->fin_ticket, 1u);
        s_cnt[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t ticket = s_ticket;
        if (ticket >= total) break;
        const uint32_t f0 = ticket * kScanThreads;
        const uint32_t f = f0 + threadIdx.x;
        if (threadIdx.x == 0) d.scan_state[ticket] = 0;  // re-arm the look-back state
        const bool in = f < T;
        uint32_t k = 0, c = 0, done = 0;
        bool head = false, retire = false;
        GenState* G = nullptr;
        uint64_t base = 0;
        if (in) {
            k = msg_of_flat(d, F, nt, ticket, f);
            G = &d.gen[d.touched[k]];
            retire = G->deliver_t != kInf;
            c = (retire ? 0u : G->lo_batch) + (f - F[k]);
            base = G->chunk_base;
            head = threadIdx.x == 0 || f == F[k];
        }
        {  // each run of a message in this tile: c_first cleared through the dirty list (one claim per warp)
            const unsigned hm = __ballot_sync(0xffffffffu, in && head);
            const int lane = threadIdx.x & 31;
            uint32_t j = 0;
            if (lane == 0 && hm) j = atomicAdd(&d.ctl->n_dirty_next, static_cast<uint32_t>(__popc(hm)));
            j = __shfl_sync(0xffffffffu, j, 0) + __popc(hm & ((1u << lane) - 1));
            if (in && head) {
                const uint32_t end = F[k + 1] < f0 + kScanThreads ? F[k + 1] : f0 + kScanThreads;
                if (j < d.dirty_cap) dirty[j] = ((base + c) << 9) | (end - f);
            }
        }
        if (in && retire) {
            // initial chunk state for the next owner; this batch's c_first
            // half is cleared through the dirty list (the scatter reads it)
            const uint64_t e = base + c;
            d.c_seen[e] = 0;
            d.c_flags[e] = 0;
            d.c_txt[e] = 0;
            d.c_path[e] = 0;
            d.c_init[e] = kInf;
            d.c_cpl[e] = kInf;
            d.c_pmax[e] = kInf;
            d.c_newb[e] = 0;
            d.c_last[e] = 0;
            d.c_newfl[e] = 0;
            const uint64_t rp = e >= d.pool_cap ? e - d.pool_cap : e;  // ring position
            // lap-parity release, one atomic per bit word and warp (a message's
            // chunks are consecutive: a warp's 32 usually share one word)
#ifndef CN_POOL_REL_PER_CHUNK
            const unsigned am = __activemask();
            const unsigned peers = __match_any_sync(am, static_cast<unsigned long long>(rp >> 5));
            const uint32_t m = __reduce_or_sync(peers, 1u << (rp & 31));
            if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicXor(&d.pool_bits[rp >> 5], m);
#else
            atomicXor(&d.pool_bits[rp >> 5], 1u << (rp & 31));
#endif
        } else if (in) {
            const uint64_t e = base + c;
            uint32_t fl = d.c_flags[e];
            if (!(fl & CF_COMPLETE)) {
                d.c_seen[e] |= d.c_newb[e];
                const uint32_t lf = d.c_last[e];
                if (lf) {
                    d.c_txt[e] = hdrs[lf - 1].tx_time;
                    d.c_path[e] = hdrs[lf - 1].path_id;
                }
                const uint32_t nf = d.c_newfl[e];
                fl |= nf & (CF_ECN | CF_RTX);
                if (nf & CF_NACKSET) fl |= CF_NACKED;  // cr.nacked (:658-660, cleared at :679)
                else if (d.c_newb[e]) fl &= ~CF_NACKED;
                if (d.c_cpl[e] != kInf) fl |= CF_COMPLETE;
                d.c_newb[e] = 0;
                d.c_last[e] = 0;
                d.c_newfl[e] = 0;
            }
            if (d.c_init[e] != kInf) {
                fl |= CF_INIT;
                d.c_init[e] = kInf;
            }
            d.c_flags[e] = fl;
            done = d.c_pmax[e] != kInf;
            d.c_cpl[e] = kInf;
            d.c_pmax[e] = kInf;
            if (done) atomicAdd(&s_cnt[F[k] > f0 ? F[k] - f0 : 0u], 1u);  // slot of the run's first chunk
        }
        __syncthreads();
        if (in && head && !retire) {
            // the message's tiles report their share of the new cum prefix;
            // the last one to report moves cum
            const uint32_t lo = G->lo_batch;
            const uint32_t F0 = F[k], F1 = F[k + 1];
            const uint32_t ntiles = (F1 - 1) / kScanThreads - F0 / kScanThreads + 1;
            const uint32_t cnt = s_cnt[threadIdx.x];  // the head is the run's first chunk
            if (cnt) atomicAdd(&G->cum_add, cnt);
            __threadfence();
            if (atomicAdd(&G->tiles_done, 1u) == ntiles - 1) {
                __threadfence();
                G->cum = lo + atomicAdd(&G->cum_add, 0u);
            }
        }
        __syncthreads();
    }
    TM_END(4);
    // ---- arena blocks of the previous batch's deliveries: the completion
    // handler has run (the reference hands the buffer to on_complete and
    // frees it after, :794-803)
    {
        const uint32_t prv = par == 0 ? 2u : par - 1;  // the previous batch's part
        const unsigned long long* al = d.aret + prv * static_cast<uint64_t>(d.aret_cap);
        const uint32_t na = min(d.ctl->n_aret[prv], d.aret_cap);
        const int lane = threadIdx.x & 31;
        const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
        const uint32_t gw = (((blockIdx.x + gridDim.x - 2 * (gridDim.x / 3)) % gridDim.x) * blockDim.x + threadIdx.x) >> 5;
        const uint32_t per = min(32u, (na + nwarps - 1) / nwarps);
        for (uint32_t j0 = gw * per; j0 < na; j0 += nwarps * per) {
            const unsigned long long vl = j0 + lane < na && lane < per ? al[j0 + lane] : 0ull;
            const uint32_t m = min(per, na - j0);
            for (uint32_t e = 0; e < m; ++e) arena_release(d, __shfl_sync(0xffffffffu, vl, e), lane);
        }
    }
    TM_END(5);
    // ---- delivered messages: completed_seq (:801) and retirement, in
    // units of 256 messages taken by ticket (the shared counters are claimed
    // once per warp: a batch may retire thousands of small messages)
    const uint32_t nunits = (nt + blockDim.x - 1) / blockDim.x;
    for (;;) {
        __syncthreads();  // s_ticket reuse
        if (threadIdx.x == 0) s_ticket = atomicAdd(&d.ctl->ret_ticket, 1u);
        __syncthreads();
        if (s_ticket >= nunits) break;
        const uint32_t k0 = s_ticket * blockDim.x + (threadIdx.x & ~31u);
        const uint32_t k = k0 + (threadIdx.x & 31);
        const int lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1;
        uint32_t g = 0;
        GenState* G = nullptr;
        bool ret = false, arel = false;
        if (k < nt) {
            g = d.touched[k];
            G = &d.gen[g];
            ret = G->deliver_t != kInf;
            arel = ret && G->buf_off != ~0ull && d.carry && G->nchunks;
        }
        const unsigned rb = __ballot_sync(0xffffffffu, ret), ab = __ballot_sync(0xffffffffu, arel);
        // a message's arena range is released in entries of kArenaRelBlocks
        // (inclusive warp prefix of the entry counts)
        const uint64_t ablk = arel ? (G->len + kArenaUnit - 1) / kArenaUnit : 0;
        const uint32_t npc = static_cast<uint32_t>((ablk + kArenaRelBlocks - 1) / kArenaRelBlocks);
        uint32_t inc = npc;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        unsigned long long ft = 0;
        uint32_t aj = 0;
        if (lane == 31 && rb) {
            ft = atomicAdd(&d.ctl->gfree_tail, static_cast<unsigned long long>(__popc(rb)));
            atomicAdd(&d.ctl->n_tomb, static_cast<uint32_t>(__popc(rb)));
            if (ab) aj = atomicAdd(&d.ctl->n_aret[par], inc);
        }
        ft = __shfl_sync(0xffffffffu, ft, 31);
        aj = __shfl_sync(0xffffffffu, aj, 31);
        if (ret) {
            atomicMax(&d.rc_done[G->rc * 128 + G->msg_id], static_cast<unsigned long long>(G->seq));
            if (arel) {
                const uint64_t b0 = G->buf_off / kArenaUnit;
                const uint32_t j0 = aj + (inc - npc);
                unsigned long long* out = d.aret + par * static_cast<uint64_t>(d.aret_cap) + j0;
                if (j0 + npc > d.aret_cap) atomicOr(&d.ctl->status, CN_RXF_CAPACITY);  // cannot happen (sized)
                for (uint32_t q = 0; q < npc && j0 + q < d.aret_cap; ++q) {
                    const uint64_t lo = static_cast<uint64_t>(q) * kArenaRelBlocks;
                    const uint64_t nb = ablk - lo < kArenaRelBlocks ? ablk - lo : kArenaRelBlocks;
                    // a start past the ring's end names the wrapped position (the range never wraps physically)
                    const uint64_t st = b0 + lo >= d.arena_blocks ? b0 + lo - d.arena_blocks : b0 + lo;
                    out[q] = (st << 31) | nb;
                }
            }
            d.gen_key[G->slot] = kTomb;
            d.gen_val[G->slot] = kInf;
            d.gen_free[(ft + __popc(rb & lt)) & d.gen_mask] = g;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(&d.ctl->ret_done, 1u);
    }
    TM_END(6);
    // ---- tombstone compaction once every retirement unit is done (a block
    // here only waits for units that running blocks hold), every warp a
    // 32-slot window of the message table (with a 32-slot lookahead): a
    // tombstone whose next non-tombstone slot in probe order is empty carries
    // no probe chain -- a key past it would have been placed in that empty
    // slot -- so it becomes empty.  No lookups or inserts run now (k_ingest
    // does them).  Runs past the lookahead and tombstones inside clusters of
    // live keys are left to the last block's rebuild (at 1/4 of the table).
    if (threadIdx.x == 0) {
        while (ld_acquire(&d.ctl->ret_done) < nunits) __nanosleep(64);
        s_ticket = ld_volatile_u32(&d.ctl->n_tomb);
    }
    __syncthreads();
    if (s_ticket) {
        const uint32_t size = d.gen_mask + 1;
        const uint32_t nwin = (size + 31) / 32;
        const int lane = threadIdx.x & 31;
        const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
        uint32_t cleared = 0;
        for (uint32_t w = gw; size >= 64 && w < nwin; w += nwarps) {  // (a window must not alias itself)
            const uint32_t x = (w * 32 + lane) & d.gen_mask, x2 = (w * 32 + 32 + lane) & d.gen_mask;
            const unsigned long long k = ld_volatile_u64(&d.gen_key[x]), k2 = ld_volatile_u64(&d.gen_key[x2]);
            const unsigned long long T = __ballot_sync(0xffffffffu, k == kTomb) |
                                         (static_cast<unsigned long long>(__ballot_sync(0xffffffffu, k2 == kTomb)) << 32);
            const unsigned long long E = __ballot_sync(0xffffffffu, k == kEmpty) |
                                         (static_cast<unsigned long long>(__ballot_sync(0xffffffffu, k2 == kEmpty)) << 32);
            if (!((T >> lane) & 1ull)) continue;
            const unsigned long long after = ~T & (~0ull << (lane + 1));  // non-tombstones past this slot
            if (!after) continue;  // the run outlasts the lookahead
            const int j = __ffsll(static_cast<long long>(after)) - 1;
            if ((E >> j) & 1ull) {
                d.gen_key[x] = kEmpty;
                d.gen_val[x] = kInf;
                ++cleared;
            }
        }
        cleared = __reduce_add_sync(0xffffffffu, cleared);
        if ((threadIdx.x & 31) == 0 && cleared) atomicSub(&d.ctl->n_tomb, cleared);
    }
    // ---- batch epilogue (last block)
    if (threadIdx.x == 0) {
        __threadfence();
        last_block = atomicAdd(&d.ctl->fin_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last_block) return;
    __threadfence();
    // tombstones of retired generations: once they reach 1/4 of the table,
    // rebuild it (no other kernel uses the table now: the scatter reads
    // GenStates by index, which do not move)
    if (d.ctl->n_tomb * 4 >= d.gen_mask + 1) {
        __shared__ uint32_t s_live;
        if (threadIdx.x == 0) s_live = 0;
        __syncthreads();
        for (uint32_t x0 = threadIdx.x * 4; x0 <= d.gen_mask; x0 += blockDim.x * 4) {
            unsigned long long k[4];  // independent loads in flight
#pragma unroll
            for (int q = 0; q < 4; ++q) k[q] = x0 + q <= d.gen_mask ? d.gen_key[x0 + q] : kEmpty;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (k[q] != kEmpty && k[q] != kTomb) {
                    const uint32_t j = atomicAdd(&s_live, 1u);
                    d.gen_tmp[2 * j] = k[q];
                    d.gen_tmp[2 * j + 1] = d.gen_val[x0 + q];
                }
        }
        __syncthreads();
        for (uint32_t x = threadIdx.x; x <= d.gen_mask; x += blockDim.x) {
            d.gen_key[x] = kEmpty;
            d.gen_val[x] = kInf;
        }
        __threadfence_block();
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < s_live; j += blockDim.x) {
            bool ins = false;
            const uint32_t slot = table_insert(d.gen_key, d.gen_mask, d.gen_tmp[2 * j], &ins);
            const uint32_t g = static_cast<uint32_t>(d.gen_tmp[2 * j + 1]);
            d.gen_val[slot] = g;
            d.gen[g].slot = slot;
        }
        __syncthreads();
        if (threadIdx.x == 0) d.ctl->n_tomb = 0;
    }
    if (threadIdx.x == 0) {
        RxCtl* C = d.ctl;
        res->n_acks = C->n_acks;
        res->n_completions = C->n_cpls;
        res->status = C->status;
        res->n_copied = C->n_copied;  // counted by k_scan
        res->bytes_copied = C->bytes_copied;
        C->n_copied = 0;
        C->bytes_copied = 0;
        C->n_touched = 0;
        C->n_trim = 0;
        C->tile_ticket = 0;
        C->fin_done = 0;
        C->status = 0;
        C->n_acks = 0;
        C->n_cpls = 0;
        C->scan_ticket = 0;
        C->fin_ticket = 0;
        C->plan_ticket_scan = 0;
        C->plan_ticket_fin = 0;
        C->plan_ready_scan = 0;
        C->plan_ready_fin = 0;
        C->ret_ticket = 0;
        C->ret_done = 0;
        uint32_t ep = C->epoch + 1;
        C->epoch = ep ? ep : 1;
        const uint32_t nxt = par == 2 ? 0u : par + 1, prv = par == 0 ? 2u : par - 1;
        C->n_dirty[par] = min(C->n_dirty_next, d.dirty_cap);
        C->n_dirty_next = 0;
        C->n_dirty[nxt] = 0;  // cleared by this batch
        C->n_aret[prv] = 0;   // released by this batch
        C->par = nxt;
        // physical extent used since the last reset (ranges overhang cap once the ring laps)
        C->pool_snap = C->pool.head < d.pool_cap ? C->pool.head : 2 * d.pool_cap;
        // the rings' tails over what the batch's ring scan found retired
        // (releases of earlier batches), and the next scan's extent
        if (C->adv_armed) {
            ring_move_tail(&C->pool, C->pool_hsnap, C->adv_pool);
            ring_move_tail(&C->arena, C->arena_hsnap, C->adv_arena);
        }
        C->adv_pool = ~0u;
        C->adv_arena = ~0u;
        C->adv_armed = 0;
        C->pool_hsnap = C->pool.head;
        C->arena_hsnap = C->arena.head;
    }
    TM_END(7);
}

// -------------------------------------------------------------------- reset
__global__ void k_reset(RxDev d, int full) {
    uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t nconn = static_cast<uint64_t>(d.conn_mask) + 1, ngen = static_cast<uint64_t>(d.gen_mask) + 1;
    for (uint64_t x = tid; x < nconn; x += stride) {
        d.rc_key[x] = kEmpty;
        if (d.ordered) {
            d.gbn_expected[x] = 0;
            d.gbn_nacked[x] = 0;
        }
    }
    for (uint64_t x = tid; x < nconn * 128; x += stride) d.rc_done[x] = 0;
    for (uint64_t x = tid; x < ngen; x += stride) {
        d.gen_key[x] = kEmpty;
        d.gen_val[x] = kInf;
        d.gen_free[x] = static_cast<uint32_t>(x);
        d.gen[x].epoch = 0;
        d.gen[x].touch = 0;
    }
    uint64_t top = full ? 2 * d.pool_cap : d.ctl->pool_snap;
    if (top > 2 * d.pool_cap) top = 2 * d.pool_cap;
    for (uint64_t x = tid; x < top; x += stride) {
        d.c_seen[x] = 0;
        d.c_flags[x] = 0;
        d.c_txt[x] = 0;
        d.c_path[x] = 0;
        d.c_init[x] = kInf;
        d.c_cpl[x] = kInf;
        d.c_pmax[x] = kInf;
        d.c_newb[x] = 0;
        d.c_last[x] = 0;
        d.c_newfl[x] = 0;
    }
    for (uint64_t x = tid; x < (d.pool_cap + 31) / 32; x += stride) d.pool_bits[x] = 0;
    for (uint64_t x = tid; x < (d.arena_blocks + 31) / 32; x += stride) d.arena_bits[x] = 0;
    for (uint64_t x = tid; x < top * d.ppc; x += stride) {
        d.c_first[x] = kInf;
        d.c_first[d.first_part + x] = kInf;
        d.c_first[2 * d.first_part + x] = kInf;
    }
    if (full)
        for (uint64_t x = tid; x < d.pool_cap / kScanThreads + ngen + 2; x += stride) d.scan_state[x] = 0;
    if (tid == 0) {
        d.ctl->pool.head = d.ctl->pool.tail = 0;
        d.ctl->arena.head = d.ctl->arena.tail = 0;
        for (int q = 0; q < 3; ++q) {
            d.ctl->n_dirty[q] = 0;
            d.ctl->n_aret[q] = 0;
        }
        d.ctl->n_dirty_next = 0;
        d.ctl->cq_in = d.ctl->cq_out = d.ctl->cq_done = 0;
        d.ctl->gfree_head = 0;
        d.ctl->gfree_tail = ngen;
        d.ctl->n_tomb = 0;
        d.ctl->pool_hsnap = d.ctl->arena_hsnap = 0;
        d.ctl->adv_pool = d.ctl->adv_arena = ~0u;
        d.ctl->adv_armed = 0;
    }
}

__global__ void k_ctl_init(RxDev d) {
    memset(d.ctl, 0, sizeof(RxCtl));
    d.ctl->epoch = 1;
}

}  // namespace cnb

using namespace cnb;

constexpr int kRxKernels = 5;
static const char* kRxKernelNames[kRxKernels] = {"ingest", "copy", "scan", "acks", "finalize"};

struct cn_rx {
    cn_rx_config cfg;
    RxDev d;
    uint32_t max_tiles = 0;
    int launches = 0;
    int sms = 148;
    int copy_bps = 64;  // k_copy block cap per SM (CN_COPY_BLOCKS_PER_SM overrides)
    int scan_first = 1;  // launch scan/acks before the scatter (CN_SCAN_FIRST=0 reverts)
    int copy_tma = 0;    // copy mode on the bulk-copy engine (CN_COPY_TMA=1; default: the vector path)
    int tma_bps = 1;     // its blocks per SM (CN_TMA_BPS)
    int ack_bps = 4;     // k_acks blocks per SM (CN_ACK_BPS)
    int chain_bps = 2;   // k_scan / k_finalize blocks per SM (CN_CHAIN_BPS)
    int copy_warps = 8;  // warps per copy-mode scatter block (CN_COPY_WARPS, 1..8)
    // programmatic dependent launch along the ack path (CN_PDL=1): measured
    // slower -- the early-launched waiting blocks take SM slots from the
    // scatter (pipelined step 101.6 -> 105.9 us, strict 105.2 -> 112.5 us)
    int pdl = 0;
    uint32_t small_batch = 32768;  // batches up to this many packets use 32-packet ack tiles (CN_ACK_SMALL)
    int hi_prio = 0;     // greatest stream priority: the latency-bound ack path wins SM slots
    // optional per-kernel timing with CUDA events on the launch stream
    bool profiling = false;
    cudaStream_t side = nullptr;           // k_copy overlaps the ack machinery
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // pipelined receivers (cn_rx_config::pipeline): the scatter of batch k is
    // joined into the caller's stream at the end of batch k + 1 (or by
    // cn_rx_flush); ev_copy alternates by host batch count
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};
    uint64_t batch_no = 0;
    int copy_pending = -1;  // ev_copy index of the scatter not yet joined, -1 none
    int* post_ok = nullptr;
    std::vector<std::vector<cudaEvent_t>> pending;
    double acc_ms[kRxKernels] = {0};
    uint64_t acc_n = 0;
};

static void prof_mark(std::vector<cudaEvent_t>* ev, cudaStream_t s) {
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
    cfg->ordered = 0;
    cfg->chunk_bytes = 32768;
    cfg->max_payload = CN_MAX_PAYLOAD;
    cfg->max_conns = 1024;
    cfg->max_msgs = 4096;
    cfg->chunk_pool = 1ull << 22;
    cfg->arena_bytes = 1ull << 30;
    cfg->max_batch = 1u << 20;
    cfg->carry_payload = 1;
    cfg->reduce_op = CN_REDUCE_NONE;
    cfg->max_posts = 0;
    cfg->pipeline = 0;
}

static void rx_free(cn_rx* rx) {
    RxDev& d = rx->d;
    void* ptrs[] = {d.rc_key, d.rc_done, d.gen_key, d.gen_val, d.gen_free, d.gen_tmp, d.gen, d.touched, d.c_first, d.dirty, d.pool_bits,
                    d.arena_bits, d.aret, d.c_seen,
                    d.c_flags, d.c_txt, d.c_path, d.c_init, d.c_cpl, d.c_pmax, d.c_newb,
                    d.c_last, d.c_newfl, d.p_gen, d.p_dst, d.p_fi, d.p_nack, d.trim_list, d.p_gbn, d.p_gbn_psn,
                    d.gbn_expected, d.gbn_nacked,
                    d.tile_state, d.scan_state, d.ctl, d.plan_F, d.plan_t0, d.arena, d.post_key,
                    d.post_val, d.post_len};
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
        cfg.max_conns > (1u << 20) ||
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
    d.reduce = static_cast<uint32_t>(cfg.reduce_op);
    d.elem = cfg.reduce_op == CN_REDUCE_SUM_F32 ? 4 : (cfg.reduce_op == CN_REDUCE_SUM_BF16 ? 2 : 1);
    if (cfg.reduce_op < 0 || cfg.reduce_op > 2 || (cfg.reduce_op && !cfg.carry_payload) ||
        (cfg.reduce_op && (cfg.max_payload % d.elem))) {
        delete rx;
        set_error("cn_rx_create: reduce_op needs carry_payload and element-aligned packets");
        return CN_E_INVALID;
    }
    if (cfg.max_posts) d.post_mask = pow2_at_least(2ull * cfg.max_posts) - 1;
    uint32_t nconn = pow2_at_least(cfg.max_conns), ngen = pow2_at_least(2ull * cfg.max_msgs);
    d.conn_mask = nconn - 1;
    d.gen_mask = ngen - 1;
    d.pool_cap = cfg.chunk_pool;
    d.arena_cap = cfg.carry_payload ? cfg.arena_bytes : 0;
    uint64_t B = cfg.max_batch;
    rx->max_tiles = static_cast<uint32_t>((B + kAckTileMin - 1) / kAckTileMin);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&rx->sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_trim, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTrimMax * 8));
    if (const char* e = getenv("CN_COPY_BLOCKS_PER_SM")) rx->copy_bps = atoi(e) > 0 ? atoi(e) : 64;
    if (const char* e = getenv("CN_SCAN_FIRST")) rx->scan_first = atoi(e);
    if (const char* e = getenv("CN_COPY_TMA")) rx->copy_tma = atoi(e);
    if (const char* e = getenv("CN_ACK_BPS")) rx->ack_bps = atoi(e) > 0 ? atoi(e) : 4;
    if (const char* e = getenv("CN_CHAIN_BPS")) rx->chain_bps = atoi(e) > 0 ? atoi(e) : 2;
    if (const char* e = getenv("CN_COPY_WARPS")) rx->copy_warps = std::min(8, std::max(1, atoi(e)));
    if (const char* e = getenv("CN_PDL")) rx->pdl = atoi(e);
    if (const char* e = getenv("CN_TMA_BPS")) rx->tma_bps = atoi(e) > 0 ? atoi(e) : 1;
    cudaFuncSetAttribute(k_copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
    if (const char* e = getenv("CN_ACK_SMALL")) rx->small_batch = static_cast<uint32_t>(atoi(e));
    {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        rx->hi_prio = greatest;
        if (const char* e = getenv("CN_ACK_PRIO")) rx->hi_prio = atoi(e) ? greatest : least;
    }
#define ALLOC(ptr, bytes)                                             \
    do {                                                              \
        cudaError_t e_ = cudaMalloc(&(ptr), (bytes));                 \
        if (e_ != cudaSuccess) {                                      \
            rx_free(rx);                                              \
            delete rx;                                                \
            return cuda_status(e_, "cn_rx_create: cudaMalloc " #ptr); \
        }                                                             \
    } while (0)
    ALLOC(d.rc_key, nconn * 8ull);
    ALLOC(d.rc_done, nconn * 128ull * 8);
    ALLOC(d.gen_key, ngen * 8ull);
    ALLOC(d.gen, ngen * sizeof(GenState));
    ALLOC(d.gen_val, ngen * 4ull);
    ALLOC(d.gen_free, ngen * 4ull);
    ALLOC(d.gen_tmp, ngen * 16ull);
    ALLOC(d.touched, ngen * 4ull);
    const uint64_t phys = 2 * cfg.chunk_pool;  // ring capacity + overhang
    d.first_part = phys * ppc;
    if (3 * d.first_part >= (1ull << 32)) {  // p_fi indices are 32-bit
        rx_free(rx);
        delete rx;
        set_error("cn_rx_create: chunk_pool too large (2 * chunk_pool * packets per chunk must be < 2^31)");
        return CN_E_INVALID;
    }
    ALLOC(d.c_first, 3 * d.first_part * 4);
    d.plan_cap = ngen < kPlanMax ? ngen : kPlanMax;
    if (const char* e = getenv("CN_PLAN_CAP")) d.plan_cap = std::min<uint32_t>(d.plan_cap, atoi(e) > 0 ? atoi(e) : 1);
    d.dirty_cap = static_cast<uint32_t>(cfg.chunk_pool / kScanThreads + d.plan_cap + 1);
    ALLOC(d.dirty, 3ull * d.dirty_cap * 8);
    ALLOC(d.pool_bits, (cfg.chunk_pool + 31) / 32 * 4);
    d.arena_blocks = d.arena_cap / kArenaUnit;
    if (d.pool_cap >= (1ull << 32) || d.arena_blocks >= (1ull << 32)) {  // ring offsets are 32-bit
        rx_free(rx);
        delete rx;
        set_error("cn_rx_create: chunk_pool and arena_bytes / 512 must be < 2^32");
        return CN_E_INVALID;
    }
    {  // one retirement-bit word per scan thread, both rings
        const uint64_t words = std::max<uint64_t>((d.pool_cap + 31) / 32, (d.arena_blocks + 31) / 32);
        const uint64_t b = (words + kIngestThreads - 1) / kIngestThreads;
        uint64_t cap_b = 2ull * rx->sms;
        if (const char* e = getenv("CN_SCAN_BLOCKS")) cap_b = std::max(1, atoi(e));
        d.scan_blocks = static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(b, 1), cap_b));
    }
    if (d.arena_blocks) ALLOC(d.arena_bits, (d.arena_blocks + 31) / 32 * 4);
    d.aret_cap = static_cast<uint32_t>(d.plan_cap + d.arena_blocks / kArenaRelBlocks + 1);
    ALLOC(d.aret, 3ull * d.aret_cap * 8);
    ALLOC(d.plan_F, (d.plan_cap + 1ull) * 4);
    ALLOC(d.plan_t0, (cfg.chunk_pool / kScanThreads + d.plan_cap + 4ull) * 4);
    ALLOC(d.c_seen, phys * 4);
    ALLOC(d.c_flags, phys * 4);
    ALLOC(d.c_txt, phys * 8);
    ALLOC(d.c_path, phys * 4);
    ALLOC(d.c_init, phys * 4);
    ALLOC(d.c_cpl, phys * 4);
    ALLOC(d.c_pmax, phys * 4);
    ALLOC(d.c_newb, phys * 4);
    ALLOC(d.c_last, phys * 4);
    ALLOC(d.c_newfl, phys * 4);
    ALLOC(d.p_gen, B * 4);
    d.max_batch = static_cast<uint32_t>(B);
    if (d.carry) {
        ALLOC(d.p_dst, 3 * B * 8);
        ALLOC(d.p_fi, 3 * B * 4);
    }
    ALLOC(d.p_nack, B);
    d.ordered = cfg.ordered ? 1 : 0;
    if (d.ordered) {
        ALLOC(d.p_gbn, B);
        ALLOC(d.p_gbn_psn, B * 8);
        ALLOC(d.gbn_expected, (static_cast<uint64_t>(d.conn_mask) + 1) * 8);
        ALLOC(d.gbn_nacked, static_cast<uint64_t>(d.conn_mask) + 1);
    }
    ALLOC(d.trim_list, kTrimMax * 4ull);
    ALLOC(d.tile_state, rx->max_tiles * 8ull);
    ALLOC(d.scan_state, (cfg.chunk_pool / kScanThreads + ngen + 2) * 8ull);
    ALLOC(d.ctl, sizeof(RxCtl));
    if (d.carry && cfg.arena_bytes) ALLOC(d.arena, 2 * cfg.arena_bytes);  // ring + overhang
    if (d.post_mask) {
        ALLOC(d.post_key, (d.post_mask + 1ull) * 8);
        ALLOC(d.post_val, (d.post_mask + 1ull) * 8);
        ALLOC(d.post_len, (d.post_mask + 1ull) * 8);
        cudaMemset(d.post_key, 0xFF, (d.post_mask + 1ull) * 8);
    }
#undef ALLOC
    cudaStreamCreateWithFlags(&rx->side, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&rx->ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rx->ev_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rx->ev_copy[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rx->ev_copy[1], cudaEventDisableTiming);
    cudaMemset(d.gen, 0, ngen * sizeof(GenState));
    k_ctl_init<<<1, 1>>>(d);
    k_reset<<<rx->sms * 4, 256>>>(d, 1);
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
    for (auto& ev : rx->pending)
        for (auto e : ev) cudaEventDestroy(e);
    if (rx->side) cudaStreamDestroy(rx->side);
    for (auto e : rx->ev_copy)
        if (e) cudaEventDestroy(e);
    if (rx->post_ok) cudaFree(rx->post_ok);
    if (rx->ev_fork) cudaEventDestroy(rx->ev_fork);
    if (rx->ev_join) cudaEventDestroy(rx->ev_join);
    rx_free(rx);
    delete rx;
}

extern "C" int cn_rx_reset(cn_rx* rx, void* stream) {
    if (!rx) {
        set_error("cn_rx_reset: null handle");
        return CN_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = cn_rx_flush(rx, stream);  // an outstanding pipelined scatter finishes first
    if (rc != CN_OK) return rc;
    k_reset<<<rx->sms * 4, 256, 0, s>>>(rx->d, 0);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

// Joins the outstanding scatter of a pipelined receiver into `stream`.
extern "C" int cn_rx_flush(cn_rx* rx, void* stream) {
    if (!rx) {
        set_error("cn_rx_flush: null handle");
        return CN_E_INVALID;
    }
    if (rx->copy_pending >= 0) {
        CNB_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), rx->ev_copy[rx->copy_pending], 0));
        rx->copy_pending = -1;
    }
    return CN_OK;
}

extern "C" void* cn_rx_arena(cn_rx* rx) { return rx ? rx->d.arena : nullptr; }
extern "C" uint64_t cn_rx_arena_bytes(const cn_rx* rx) { return rx && rx->d.arena ? 2 * rx->d.arena_cap : 0; }
extern "C" int cn_rx_last_launches(const cn_rx* rx) { return rx ? rx->launches : 0; }

extern "C" int cn_rx_get_usage(cn_rx* rx, cn_rx_usage* out) {
    if (!rx || !out) {
        set_error("cn_rx_get_usage: null argument");
        return CN_E_INVALID;
    }
    RingCtl r[2];
    CNB_CUDA(cudaDeviceSynchronize());
    CNB_CUDA(cudaMemcpy(r, rx->d.ctl, sizeof r, cudaMemcpyDeviceToHost));  // pool, arena lead RxCtl
    out->pool_live = r[0].head - r[0].tail;
    out->pool_cap = rx->d.pool_cap;
    out->pool_allocated = r[0].head;
    out->arena_live = r[1].head - r[1].tail;
    out->arena_blocks = rx->d.arena_blocks;
    out->arena_allocated = r[1].head;
    return CN_OK;
}

static int rx_batch_impl(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                         uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                         cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                         void* stream, const uint64_t* d_msgdata = nullptr, const uint64_t* d_poff = nullptr);

extern "C" int cn_rx_batch(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const void* d_payload,
                           uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks,
                           uint32_t max_acks, cn_completion* d_completions,
                           uint32_t max_completions, cn_rx_result* d_result, void* stream) {
    if (rx && rx->d.ordered && n > 0) {
        set_error("cn_rx_batch: ordered reliability needs conn_psn (cn_rx_batch_psn)");
        return CN_E_INVALID;
    }
    return rx_batch_impl(rx, d_hdrs, nullptr, d_payload, payload_stride, n, d_acks, max_acks, d_completions,
                         max_completions, d_result, stream);
}

// Packets carrying their message's data pointer (Packet::msg_data, the
// reference's send_message_data path): packet i's payload is read at
// d_msg_data[i] + chunk_offset + seq_in_chunk * max_payload; a 0 pointer is a
// packet without data (accepted and counted, nothing copied, :722).
extern "C" int cn_rx_batch_msgdata(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                                   const uint64_t* d_msg_data, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                                   cn_completion* d_completions, uint32_t max_completions,
                                   cn_rx_result* d_result, void* stream) {
    if (rx && (rx->d.ordered ? (n > 0 && !d_psn) : d_psn != nullptr)) {
        set_error("cn_rx_batch_msgdata: conn_psn exactly when the receiver is ordered");
        return CN_E_INVALID;
    }
    if (rx && n > 0 && !d_msg_data) {
        set_error("cn_rx_batch_msgdata: null msg_data");
        return CN_E_INVALID;
    }
    return rx_batch_impl(rx, d_hdrs, d_psn, nullptr, 0, n, d_acks, max_acks, d_completions, max_completions,
                         d_result, stream, d_msg_data);
}

// Packed payloads: packet i's payload_len bytes at d_payload + d_offset[i]
// (a NIC ring's variable-size packet buffers; no stride padding to move).
extern "C" int cn_rx_batch_packed(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                                  const uint64_t* d_offset, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                                  cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                                  void* stream) {
    if (rx && (rx->d.ordered ? (n > 0 && !d_psn) : d_psn != nullptr)) {
        set_error("cn_rx_batch_packed: conn_psn exactly when the receiver is ordered");
        return CN_E_INVALID;
    }
    if (rx && n > 0 && rx->d.carry && (!d_offset || !d_payload)) {
        set_error("cn_rx_batch_packed: null payload or offsets");
        return CN_E_INVALID;
    }
    return rx_batch_impl(rx, d_hdrs, d_psn, d_payload, 0, n, d_acks, max_acks, d_completions, max_completions,
                         d_result, stream, nullptr, d_offset);
}

extern "C" int cn_rx_batch_psn(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                               uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                               cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                               void* stream) {
    if (rx && (!rx->d.ordered || (n > 0 && !d_psn))) {
        set_error("cn_rx_batch_psn: needs a receiver created with ordered = 1 and conn_psn");
        return CN_E_INVALID;
    }
    return rx_batch_impl(rx, d_hdrs, d_psn, d_payload, payload_stride, n, d_acks, max_acks, d_completions,
                         max_completions, d_result, stream);
}

static int rx_batch_impl(cn_rx* rx, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                         uint64_t payload_stride, uint32_t n, cn_ack_rec* d_acks, uint32_t max_acks,
                         cn_completion* d_completions, uint32_t max_completions, cn_rx_result* d_result,
                         void* stream, const uint64_t* d_msgdata, const uint64_t* d_poff) {
    if (!rx || !d_result) {
        set_error("cn_rx_batch: null handle/result");
        return CN_E_INVALID;
    }
    rx->d.psn = d_psn;
    rx->d.msgdata = reinterpret_cast<const unsigned long long*>(d_msgdata);
    rx->d.poff = reinterpret_cast<const unsigned long long*>(d_poff);
    if (n > rx->cfg.max_batch) {
        set_error("cn_rx_batch: n exceeds max_batch");
        return CN_E_CAPACITY;
    }
    if (n > 0 && !d_hdrs) {
        set_error("cn_rx_batch: null headers");
        return CN_E_INVALID;
    }
    if (rx->d.carry && n > 0 && !d_msgdata && (!d_payload || (payload_stride && payload_stride < rx->d.max_pl))) {
        set_error("cn_rx_batch: carry_payload needs a payload buffer (stride 0 or >= max_payload)");
        return CN_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const RxDev& d = rx->d;
    std::vector<cudaEvent_t>* ev = nullptr;
    if (rx->profiling && n > 0) {
        int rc = cn_rx_flush(rx, stream);  // profiled batches run strictly in order
        if (rc != CN_OK) return rc;
        rx->pending.emplace_back();
        ev = &rx->pending.back();
    }
    // chunk-tile kernels: persistent grids pulling 256-chunk tiles by ticket
    uint32_t gb = static_cast<uint32_t>(rx->chain_bps) * static_cast<uint32_t>(rx->sms);
    prof_mark(ev, s);
    if (n > 0) {
        const uint8_t* pl = static_cast<const uint8_t*>(d_payload);
        const uint32_t ack_tile = n <= rx->small_batch ? kAckTileMin : kAckTileMax;
        rx->d.ack_tile = ack_tile;
        uint32_t tiles = (n + ack_tile - 1) / ack_tile;
        const uint32_t cwarps = static_cast<uint32_t>(rx->copy_warps);
        uint32_t cw = (n + cwarps - 1) / cwarps;  // one warp (packet) per copy-block warp
        // about one packet per warp: short-lived blocks, so the block
        // scheduler hands SM slots to the high-priority ack path first and
        // to the scatter as they free up (a persistent scatter grid would
        // pin half the register file for its whole duration)
        uint32_t cmax = static_cast<uint32_t>(rx->sms * rx->copy_bps);
        // the ack path at the greatest priority from its first kernel: in a
        // pipelined receiver the previous batch's scatter still fills the SMs
        auto hi = [&](dim3 grid, dim3 block, size_t smem) {
            cudaLaunchConfig_t lc = {};
            static thread_local cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = rx->hi_prio;
            lc.gridDim = grid;
            lc.blockDim = block;
            lc.dynamicSmemBytes = smem;
            lc.stream = s;
            lc.attrs = at;
            lc.numAttrs = 1;
            return lc;
        };
        if (d.ordered) {  // the go-back-N filter first
            cudaLaunchConfig_t lc = hi(dim3(4), dim3(256), 0);
            CNB_CUDA(cudaLaunchKernelEx(&lc, k_gbn, d, d_hdrs, n));
        }
        {
            cudaLaunchConfig_t lc = hi(dim3(d.scan_blocks + (n + kIngestThreads - 1) / kIngestThreads),
                                       dim3(kIngestThreads), 0);
            CNB_CUDA(cudaLaunchKernelEx(&lc, k_ingest, d, d_hdrs, n));
        }
        prof_mark(ev, s);
        // fork: the HBM-bound scatter runs beside the latency-bound ack path
        cudaStream_t cs = ev ? s : rx->side;
        if (!ev) {
            CNB_CUDA(cudaEventRecord(rx->ev_fork, s));
            CNB_CUDA(cudaStreamWaitEvent(cs, rx->ev_fork, 0));
        }
        const uint32_t cg = cw < cmax ? cw : cmax;
        auto copy = [&] {
            if (!d.carry) {  // headers only (e.g. the ring's all-gather, payload already in place)
                prof_mark(ev, s);
                return;
            }
            if (d.reduce == 1)
                k_copy<1><<<cg, 256, 0, cs>>>(d, d_hdrs, pl, payload_stride, n);
            else if (d.reduce == 2)
                k_copy<2><<<cg, 256, 0, cs>>>(d, d_hdrs, pl, payload_stride, n);
            else if (rx->copy_tma && payload_stride % 16 == 0 && d.max_pl <= kTmaSlotBytes)
                k_copy_tma<<<rx->tma_bps * rx->sms, 32, kTmaSmem, cs>>>(d, d_hdrs, pl, payload_stride, n);
            else
                k_copy<0><<<cg, 32 * cwarps, 0, cs>>>(d, d_hdrs, pl, payload_stride, n);
            prof_mark(ev, s);
        };
        const bool copy_last = rx->scan_first && !ev;  // profiling keeps the named kernel order
        // programmatic dependent launch along the ack path (not under the
        // per-kernel profiling events, which sit between the kernels)
        const bool pdl = rx->pdl && !ev;
        if (!copy_last) copy();
        {
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = rx->hi_prio;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (pdl_wait)
            at[1].val.programmaticStreamSerializationAllowed = 1;
            lc.gridDim = dim3(gb);
            lc.blockDim = dim3(kScanThreads);
            lc.stream = s;
            lc.attrs = at;
            lc.numAttrs = pdl ? 2 : 1;
            CNB_CUDA(cudaLaunchKernelEx(&lc, k_scan, d));
        }
        {  // rare work, but on the ack path: same priority, or it queues behind the scatter
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = rx->hi_prio;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (pdl_wait)
            at[1].val.programmaticStreamSerializationAllowed = 1;
            lc.gridDim = dim3(1);
            lc.blockDim = dim3(1024);
            lc.dynamicSmemBytes = kTrimMax * 8;
            lc.stream = s;
            lc.attrs = at;
            lc.numAttrs = pdl ? 2 : 1;
            CNB_CUDA(cudaLaunchKernelEx(&lc, k_trim, d, d_hdrs));
        }
        prof_mark(ev, s);
        // persistent: as many blocks as fit beside the scatter, tiles by ticket
        const uint32_t acap = static_cast<uint32_t>(rx->sms * rx->ack_bps);
        const uint32_t ag = tiles < acap ? tiles : acap;
        {
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = rx->hi_prio;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (pdl_wait)
            at[1].val.programmaticStreamSerializationAllowed = 1;
            lc.gridDim = dim3(ag);
            lc.blockDim = dim3(kAckWarps * 32);
            lc.stream = s;
            lc.attrs = at;
            lc.numAttrs = pdl ? 2 : 1;
            if (ack_tile == kAckTileMin)
                CNB_CUDA(cudaLaunchKernelEx(&lc, k_acks<kAckTileMin>, d, d_hdrs, n, d_acks, max_acks, d_completions,
                                            max_completions));
            else
                CNB_CUDA(cudaLaunchKernelEx(&lc, k_acks<kAckTileMax>, d, d_hdrs, n, d_acks, max_acks, d_completions,
                                            max_completions));
        }
        prof_mark(ev, s);
        if (copy_last) copy();
        // the fold into persistent state needs the ack path, not the scatter
        // (it clears the other c_first half): it runs beside the scatter's tail
        {
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = rx->hi_prio;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (pdl_wait)
            at[1].val.programmaticStreamSerializationAllowed = 1;
            lc.gridDim = dim3(gb);
            lc.blockDim = dim3(kScanThreads);
            lc.stream = s;
            lc.attrs = at;
            lc.numAttrs = pdl ? 2 : 1;
            CNB_CUDA(cudaLaunchKernelEx(&lc, k_finalize, d, d_hdrs, d_result));
        }
        prof_mark(ev, s);
        if (!ev && d.carry && rx->cfg.pipeline) {
            // pipelined: join the PREVIOUS batch's scatter; this one's runs on
            // beside the next batch's ingest and ack path
            const int j = static_cast<int>(rx->batch_no & 1);
            CNB_CUDA(cudaEventRecord(rx->ev_copy[j], cs));
            if (rx->copy_pending >= 0) CNB_CUDA(cudaStreamWaitEvent(s, rx->ev_copy[rx->copy_pending], 0));
            rx->copy_pending = j;
        } else if (!ev) {
            CNB_CUDA(cudaEventRecord(rx->ev_join, cs));
            CNB_CUDA(cudaStreamWaitEvent(s, rx->ev_join, 0));
        }
    } else {
        k_finalize<<<gb, kScanThreads, 0, s>>>(d, d_hdrs, d_result);
        prof_mark(ev, s);
        int rc = cn_rx_flush(rx, stream);  // an empty batch completes the pipeline
        if (rc != CN_OK) return rc;
    }
    rx->batch_no += 1;
    rx->launches = n > 0 ? (d.carry ? 6 : 5) + (d.ordered ? 1 : 0) : 1;
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

__global__ void k_post(RxDev d, uint64_t tag, uint64_t ptr, uint64_t len, int* ok) {
    uint32_t h = static_cast<uint32_t>(mix64(tag)) & d.post_mask;
    for (uint32_t q = 0; q <= d.post_mask; ++q) {
        unsigned long long old = atomicCAS(&d.post_key[h], kEmpty, tag);
        if (old == kEmpty || old == tag) {
            d.post_val[h] = ptr;
            d.post_len[h] = len;
            *ok = 1;
            return;
        }
        h = (h + 1) & d.post_mask;
    }
    *ok = 0;
}

extern "C" int cn_rx_post(cn_rx* rx, uint64_t tag, void* d_buf, uint64_t len, void* stream) {
    if (!rx || !d_buf || !rx->d.post_mask || !rx->d.carry) {
        set_error("cn_rx_post: needs carry_payload and max_posts > 0");
        return CN_E_INVALID;
    }
    if (reinterpret_cast<uintptr_t>(d_buf) & 15) {
        set_error("cn_rx_post: buffer must be 16-byte aligned");
        return CN_E_INVALID;
    }
    if (!rx->post_ok) CNB_CUDA(cudaMalloc(&rx->post_ok, sizeof(int)));
    k_post<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(rx->d, tag, reinterpret_cast<uint64_t>(d_buf),
                                                           len, rx->post_ok);
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
        for (size_t k = 0; k + 1 < ev.size() && k < static_cast<size_t>(kRxKernels); ++k) {
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

#ifdef CN_RX_TIMING
// debug builds only: the phase marks (ns, %globaltimer), then re-armed
extern "C" int cn_rx_debug_timing(unsigned long long* out, int n) {
    unsigned long long h[64];
    CNB_CUDA(cudaMemcpyFromSymbol(h, g_tm, sizeof h));
    for (int k = 0; k < n && k < 64; ++k) out[k] = h[k];
    const unsigned long long mins[] = {0, 10, 20, 22, 24, 30, 34};
    for (int k = 0; k < 64; ++k) h[k] = 0;
    for (unsigned long long k : mins) h[k] = ~0ull;
    CNB_CUDA(cudaMemcpyToSymbol(g_tm, h, sizeof h));
    return CN_OK;
}
// k_ingest per-packet-block marks: [5][64]
extern "C" int cn_rx_debug_ingest_timing(unsigned long long* out) {
    CNB_CUDA(cudaMemcpyFromSymbol(out, g_ing_tm, sizeof g_ing_tm));
    return CN_OK;
}
// k_acks per-tile marks of the last batch: [4][kTileTm] (start, decided, built, written)
extern "C" int cn_rx_debug_tile_timing(unsigned long long* out) {
    CNB_CUDA(cudaMemcpyFromSymbol(out, g_tile_tm, sizeof g_tile_tm));
    return CN_OK;
}
#endif

extern "C" const char* cn_rx_kernel_name(int k) {
    return (k >= 0 && k < kRxKernels) ? kRxKernelNames[k] : "";
}
