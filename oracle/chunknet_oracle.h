/* chunknet_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker the CUDA path is compared against.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.  Every function cites the reference file:line it
 * restates (/root/reference/proj/...).  Pinned against the compiled
 * reference (oracle/_ref) through tests/golden fixtures.
 */
#ifndef CHUNKNET_ORACLE_H
#define CHUNKNET_ORACLE_H

#include <stdint.h>

#include "chunknet_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:11-60 + libstdc++ 13 <random> ---------------------------- */
typedef struct orc_mt64 {
    uint64_t mt[312];
    int idx;
} orc_mt64;

uint64_t orc_fnv1a64(const char* s);
uint64_t orc_splitmix64(uint64_t x);
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
/* RngStream(seed, name[, index]) (rng.hpp:32-35); index < 0 = unindexed */
void orc_rng_stream(orc_mt64* g, uint64_t seed, const char* name, int64_t index);
uint64_t orc_next_below(orc_mt64* g, uint64_t n);  /* rng.hpp:40-43 */
double orc_next_double(orc_mt64* g);                /* rng.hpp:46-48 */

/* select_path (lb.cpp:7-27): policy 0 oblivious, 1 p2_rtt, 2 p2_ecn */
int orc_select_path(int policy, int n_paths, const double* rtt, const double* ecn,
                    orc_mt64* g);
/* sequence of `count` decisions on a fixed board */
void orc_select_paths(int policy, int n_paths, const double* rtt, const double* ecn,
                      uint64_t seed, const char* name, int64_t index, uint64_t count,
                      int32_t* out);

void orc_rng_u64_seq(uint64_t seed, const char* name, int64_t index, uint64_t count,
                     uint64_t* out);
void orc_next_below_seq(uint64_t seed, const char* name, int64_t index,
                        const uint64_t* ns, uint64_t count, uint64_t* out);
void orc_next_double_seq(uint64_t seed, const char* name, int64_t index, uint64_t count,
                         double* out);

/* ---- receive path (transport.cpp:546-803) ----------------------------- */
typedef struct orc_rx orc_rx;
orc_rx* orc_rx_create(uint32_t max_payload, int carry_payload);
/* ordered (go-back-N) reliability: psn[i] = conn_psn of packet i of every
 * following batch (the pointer is read during orc_rx_batch) */
void orc_rx_set_ordered(orc_rx* rx, int ordered, const uint64_t* psn);
void orc_rx_destroy(orc_rx* rx);
/* Processes n packets in order (payload of packet i at payload + i*stride).
 * Appends acks / completions; reassembled buffers are copied into arena at
 * 16-byte aligned running offsets (cn_completion::buf_offset).  Returns
 * CN_OK or a negative status (logic_error paths of the reference). */
typedef struct orc_rx_counts {
    uint64_t n_acks;
    uint64_t n_completions;
    uint64_t n_nacks;
    uint64_t arena_used;
    uint64_t pkts_accepted;
    uint64_t bytes_accepted;
} orc_rx_counts;
int orc_rx_batch(orc_rx* rx, const cn_pkt_hdr* hdrs, const uint8_t* payload,
                 uint64_t stride, uint64_t n, uint32_t index_base, cn_ack_rec* acks,
                 uint64_t max_acks, cn_completion* cpls, uint64_t max_cpls,
                 uint8_t* arena, uint64_t arena_bytes, orc_rx_counts* counts);

/* ---- helpers ----------------------------------------------------------- */
/* pattern_bytes (test_transport.cpp:63-71) */
void orc_pattern_bytes(uint64_t n, uint64_t seed, uint8_t* out);
/* staging[i*stride ..] = src_of(pkt i)[chunk_offset + seq*max_pl ..] for
 * pattern payloads (seed = msg_tag), threads >= 1 */
void orc_fill_staging(const cn_pkt_hdr* hdrs, uint64_t n, uint32_t max_pl,
                      uint8_t* staging, uint64_t stride);

/* ---- ring reduction fold (builder-defined) ----------
 * x: n_ranks arrays of `count` elements, rank-major.  Ring reduce-scatter +
 * allgather in the exact per-hop order; out: the allreduced array every
 * rank ends with (identical across ranks).  dtype 0 = fp32, 1 = bf16
 * (uint16 storage, fp32 add, round-to-nearest-even per hop). */
void orc_ring_allreduce(int dtype, int n_ranks, uint64_t count, const void* x,
                        void* out);
/* same with segment boundaries rounded down to multiples of `quantum`. */
void orc_ring_allreduce_q(int dtype, int n_ranks, uint64_t count, const void* x, void* out,
                          uint64_t quantum);

#ifdef __cplusplus
}
#endif
#endif
