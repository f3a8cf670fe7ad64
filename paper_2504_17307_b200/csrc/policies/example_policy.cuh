// Example transport policy plug-in (include/chunknet_policy.cuh), built into
// ../libchunknet_b200_user.so by `make user` (any header defining
// CnUserPolicy works the same way: `make USER_POLICY=/abs/path.cuh`):
// P2 over ECN marks for fresh chunks (two draws from the connection's
// stream), retransmissions on the least-RTT path.  oracle/ref_harness.cpp
// installs the same policy in the reference (ExampleUserPolicy) for the
// parity goldens sender_user_*.npz.
struct CnUserPolicy {
    template <class Rng>
    __device__ static int select_path(const cn_chunk_view&, const cn_path_board& b, Rng& rng, uint64_t* st) {
        if (b.n_paths == 1) return 0;
        const int a = static_cast<int>(rng.next_below(b.n_paths));
        int c = static_cast<int>(rng.next_below(b.n_paths - 1));
        if (c >= a) ++c;
        st[0] += 1;  // fresh chunks placed
        return b.ecn_ewma[c] < b.ecn_ewma[a] ? c : a;
    }
    template <class Rng>
    __device__ static int rtx_path(const cn_chunk_view&, const cn_path_board& b, Rng&, uint64_t*) {
        int best = 0;
        for (int p = 1; p < b.n_paths; ++p)
            if (b.rtt_ewma[p] < b.rtt_ewma[best]) best = p;
        return best;
    }
    __device__ static int64_t pacing(const cn_chunk_view&) { return 0; }
};
