/* chunknet_policy.cuh -- the transport policy plug-in of the sm_100a sender
 * engine (the reference's TransportPolicy, proj/include/chunknet/policy.hpp:
 * 39-67, installed per connection with Transport::set_policy_factory,
 * transport.hpp:80-81,95).
 *
 * The engine runs one warp per connection on the device, so a policy is not
 * a host object behind a vtable: it is a struct of static __device__ hooks
 * compiled into the engine (inlined into the warp's event loop -- no
 * indirect calls, no host round trips) and chosen per engine at run time
 * with cn_tx_config::policy.  Every lane of the connection's warp runs a
 * hook with the same arguments and must return the same value; random draws
 * (rng.next_below) are warp-collective and come from the connection's
 * RngStream("transport.conn", index), exactly as the reference's hooks draw
 * from theirs.  `state` is the connection's policy state -- the members of
 * the reference's per-connection policy instance (the factory is called
 * once per connection): 4 words, zero at engine creation.
 *
 * Hooks (a policy defines all three):
 *   select_path(view, board, rng, state)  -> path in [0, board.n_paths)
 *       TransportPolicy::on_select_path, for a fresh chunk (commit_chunks,
 *       transport.cpp:281-287)
 *   rtx_path(view, board, rng, state)     -> path, or -1 = select_path
 *       TransportPolicy::on_tx_rtx_chunk (queue_rtx, :516-542)
 *   pacing(view)                          -> 0 (the engine sends at once;
 *       a non-zero delay is a contract violation, like on_chunk_size below)
 * Chunk sizes are DefaultPolicy's (min(remaining, chunk_bytes),
 * policy.hpp:75-78): the receive path identifies chunks by offset /
 * chunk_bytes.  A path outside [0, n_paths) is the reference's logic_error
 * (transport.cpp:283-286, 528-531): the engine sets status bit
 * CN_TX_STATUS_POLICY (cn_tx_status) and sends on path 0.
 *
 * Adding a policy: write the struct (see RoundRobinPolicy below) in a header
 * and build the library with `make USER_POLICY=/abs/path/my_policy.cuh`
 * (it must define `struct CnUserPolicy`); select it with
 * cn_tx_config::policy = CN_POLICY_USER. */
#ifndef CHUNKNET_POLICY_CUH
#define CHUNKNET_POLICY_CUH

#include <stdint.h>

/* ChunkView (policy.hpp:13-26), as the engine builds it (view_of,
 * transport.cpp:496-512) */
struct cn_chunk_view {
    int32_t src, dst;
    uint32_t msg_id;
    uint32_t csn;        /* chunk index & 0xFF */
    uint64_t msg_seq, msg_len, offset;
    uint32_t len;
    int32_t last;
    int32_t attempts;    /* transmissions so far (0 for a fresh chunk) */
    int32_t prev_path;   /* path of the previous attempt, -1 if none */
    uint64_t remaining;  /* unchunked bytes left in the message */
};

/* PathScoreboard (lb.hpp:15-36): per-path EWMAs of the connection */
struct cn_path_board {
    const double* rtt_ewma;
    const double* ecn_ewma;
    int32_t n_paths;
};

namespace cn_policy {

/* Spray chunks over the paths in turn (a per-connection counter); a
 * retransmission takes the next turn and steps off its previous path. */
struct RoundRobinPolicy {
    template <class Rng>
    __device__ static int select_path(const cn_chunk_view&, const cn_path_board& b, Rng&, uint64_t* st) {
        const int p = static_cast<int>(st[0] % static_cast<uint64_t>(b.n_paths));
        st[0] += 1;
        return p;
    }
    template <class Rng>
    __device__ static int rtx_path(const cn_chunk_view& v, const cn_path_board& b, Rng&, uint64_t* st) {
        int p = static_cast<int>(st[0] % static_cast<uint64_t>(b.n_paths));
        st[0] += 1;
        if (b.n_paths > 1 && p == v.prev_path) p = (p + 1) % b.n_paths;
        return p;
    }
    __device__ static int64_t pacing(const cn_chunk_view&) { return 0; }
};

/* Single path per connection (flow-hash, the ECMP baseline): every chunk
 * and retransmission of a (src, dst) pair on one path. */
struct SinglePathPolicy {
    __device__ static int pick(const cn_chunk_view& v, const cn_path_board& b) {
        const uint64_t h = static_cast<uint64_t>(static_cast<uint32_t>(v.src)) * 2654435761ull +
                           static_cast<uint64_t>(static_cast<uint32_t>(v.dst));
        return static_cast<int>(h % static_cast<uint64_t>(b.n_paths));
    }
    template <class Rng>
    __device__ static int select_path(const cn_chunk_view& v, const cn_path_board& b, Rng&, uint64_t*) {
        return pick(v, b);
    }
    template <class Rng>
    __device__ static int rtx_path(const cn_chunk_view&, const cn_path_board&, Rng&, uint64_t*) {
        return -1;
    }
    __device__ static int64_t pacing(const cn_chunk_view&) { return 0; }
};

/* Test policy: a path out of range (the reference's "path out of range"
 * contract test, test_transport.cpp:686-703). */
struct OutOfRangePolicy {
    template <class Rng>
    __device__ static int select_path(const cn_chunk_view&, const cn_path_board&, Rng&, uint64_t*) {
        return 99;
    }
    template <class Rng>
    __device__ static int rtx_path(const cn_chunk_view&, const cn_path_board&, Rng&, uint64_t*) {
        return -1;
    }
    __device__ static int64_t pacing(const cn_chunk_view&) { return 0; }
};

}  // namespace cn_policy

#endif
