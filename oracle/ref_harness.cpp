// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (oracle side, never shipped).
//
// Drives the UNMODIFIED reference chunknet library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) to
//   * record packet traces from its discrete-event simulator (DES),
//   * replay delivered data packets into a fresh Transport's receive path
//     (Transport::handle_packet, src/transport.cpp:565) and capture the ack
//     stream in emission order,
//   * time that receive path on the host's cores (bench.py cpu baseline),
//   * emit RngStream / select_path draw sequences (rng.hpp:29-60, lb.cpp:7-27),
//   * replay timed acks into a sender (handle_ack, transport.cpp:849-942).
// Private members are reached by compiling THIS translation unit with
// `private` defined as `public`; the library objects are compiled normally,
// access specifiers do not change layout.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#define private public
#include "chunknet/config.hpp"
#include "chunknet/eqds.hpp"
#include "chunknet/event_queue.hpp"
#include "chunknet/experiment.hpp"
#include "chunknet/lb.hpp"
#include "chunknet/network.hpp"
#include "chunknet/packet.hpp"
#include "chunknet/rng.hpp"
#include "chunknet/topology.hpp"
#include "chunknet/transport.hpp"
#include "chunknet/wire.hpp"
#undef private

#include "chunknet_b200.h"

using namespace chunknet;

namespace {

thread_local std::string g_err;
thread_local bool g_ordered = false;  // records of an ordered-reliability run (go-back-N NACKs)
// introspection probes of the next sender replay (cnref_set_probes)
thread_local std::vector<int64_t> g_probe_t;
thread_local int64_t* g_probe_out = nullptr;
thread_local uint32_t g_probe_stride = 0;

// Payload generator of the reference tests (test_transport.cpp:63-71).
std::shared_ptr<std::vector<uint8_t>> pattern(uint64_t n, uint64_t seed) {
    auto v = std::make_shared<std::vector<uint8_t>>(n);
    uint64_t x = seed;
    for (uint64_t i = 0; i < n; ++i) {
        if (i % 8 == 0) x = splitmix64(x + i);
        (*v)[i] = static_cast<uint8_t>(x >> ((i % 8) * 8));
    }
    return v;
}

// The device engine's built-in policy plug-ins (include/chunknet_policy.cuh),
// restated as reference TransportPolicy subclasses (policy.hpp:39-67) and
// installed with Transport::set_policy_factory: one instance per connection.
struct RoundRobinPolicy : TransportPolicy {
    uint32_t cb;
    uint64_t next = 0;
    explicit RoundRobinPolicy(uint32_t c) : cb(c) {}
    uint32_t on_chunk_size(uint64_t rem) override { return rem < cb ? static_cast<uint32_t>(rem) : cb; }
    int on_select_path(const ChunkView&, const PathScoreboard& b, RngStream&) override {
        return static_cast<int>(next++ % static_cast<uint64_t>(b.n_paths()));
    }
    int on_tx_rtx_chunk(const ChunkView& c, const PathScoreboard& b, RngStream&) override {
        const int n = b.n_paths();
        int p = static_cast<int>(next++ % static_cast<uint64_t>(n));
        if (n > 1 && p == c.prev_path) p = (p + 1) % n;
        return p;
    }
};
struct SinglePathPolicy : TransportPolicy {
    uint32_t cb;
    explicit SinglePathPolicy(uint32_t c) : cb(c) {}
    uint32_t on_chunk_size(uint64_t rem) override { return rem < cb ? static_cast<uint32_t>(rem) : cb; }
    int on_select_path(const ChunkView& v, const PathScoreboard& b, RngStream&) override {
        const uint64_t h = static_cast<uint64_t>(static_cast<uint32_t>(v.src)) * 2654435761ull +
                           static_cast<uint64_t>(static_cast<uint32_t>(v.dst));
        return static_cast<int>(h % static_cast<uint64_t>(b.n_paths()));
    }
};
// paper_2504_17307_b200/csrc/policies/example_policy.cuh (the plug-in example)
struct ExampleUserPolicy : TransportPolicy {
    uint32_t cb;
    explicit ExampleUserPolicy(uint32_t c) : cb(c) {}
    uint32_t on_chunk_size(uint64_t rem) override { return rem < cb ? static_cast<uint32_t>(rem) : cb; }
    int on_select_path(const ChunkView&, const PathScoreboard& b, RngStream& rng) override {
        const int n = b.n_paths();
        if (n == 1) return 0;
        const int a = static_cast<int>(rng.next_below(static_cast<uint64_t>(n)));
        int c = static_cast<int>(rng.next_below(static_cast<uint64_t>(n - 1)));
        if (c >= a) ++c;
        return b.ecn_score(c) < b.ecn_score(a) ? c : a;
    }
    int on_tx_rtx_chunk(const ChunkView&, const PathScoreboard& b, RngStream&) override {
        int best = 0;
        for (int p = 1; p < b.n_paths(); ++p)
            if (b.rtt_score(p) < b.rtt_score(best)) best = p;
        return best;
    }
};
void install_policy(Transport& tr, int policy, uint32_t cb) {
    if (policy == 1)
        tr.set_policy_factory([cb](int, int) { return std::make_unique<RoundRobinPolicy>(cb); });
    else if (policy == 2)
        tr.set_policy_factory([cb](int, int) { return std::make_unique<SinglePathPolicy>(cb); });
    else if (policy == 3)
        tr.set_policy_factory([cb](int, int) { return std::make_unique<ExampleUserPolicy>(cb); });
}

cn_pkt_hdr to_rec(const Packet& p) {
    cn_pkt_hdr r;
    std::memset(&r, 0, sizeof r);
    r.src = p.src;
    r.dst = p.dst;
    r.path_id = p.path_id;
    r.hdr = encode_header(p.hdr);
    r.chunk_offset = p.chunk_offset;
    r.chunk_len = p.chunk_len;
    r.payload_len = static_cast<uint16_t>(p.payload_len);
    r.seq_in_chunk = static_cast<uint8_t>(p.seq_in_chunk);
    r.flags = (p.is_rtx ? CN_PKT_RTX : 0) | (p.ecn ? CN_PKT_ECN : 0) |
              (p.trimmed ? CN_PKT_TRIMMED : 0);
    r.tx_time = p.tx_time;
    r.msg_seq = p.msg_seq;
    r.msg_tag = p.msg_tag;
    r.msg_len = p.msg_len;
    return r;
}

Packet from_rec(const cn_pkt_hdr& r) {
    Packet p;
    p.kind = PacketKind::data;
    p.src = r.src;
    p.dst = r.dst;
    p.path_id = r.path_id;
    p.hdr = decode_header(r.hdr);
    p.chunk_offset = r.chunk_offset;
    p.chunk_len = r.chunk_len;
    p.payload_len = r.payload_len;
    p.seq_in_chunk = r.seq_in_chunk;
    p.is_rtx = r.flags & CN_PKT_RTX;
    p.ecn = r.flags & CN_PKT_ECN;
    p.trimmed = r.flags & CN_PKT_TRIMMED;
    p.tx_time = r.tx_time;
    p.msg_seq = r.msg_seq;
    p.msg_tag = r.msg_tag;
    p.msg_len = r.msg_len;
    return p;
}

cn_ack_rec ack_rec(const Packet& p, uint32_t idx, int64_t aux) {
    cn_ack_rec a;
    std::memset(&a, 0, sizeof a);
    a.src = p.src;
    a.dst = p.dst;
    a.hdr = encode_header(p.hdr);
    a.echo_path_id = p.echo_path_id;
    a.cum_csn = p.cum_csn;
    a.flags = (p.cum_valid ? CN_ACK_CUM_VALID : 0) |
              (p.ecn_echo ? CN_ACK_ECN_ECHO : 0) |
              (p.kind == PacketKind::nack ? CN_ACK_NACK : 0) |
              (p.kind == PacketKind::credit ? CN_ACK_CREDIT : 0) |
              (p.kind == PacketKind::rts_ack ? CN_ACK_RTS_ACK : 0);
    if (p.kind == PacketKind::nack) a.cum_csn = p.nack_csn;

    a.pkt_index = idx;
    a.msg_seq = p.msg_seq;
    a.sack[0] = p.sack[0];
    a.sack[1] = p.sack[1];
    if (p.kind == PacketKind::credit) a.sack[0] = p.credit_bytes;
    if (p.kind == PacketKind::nack && g_ordered) {  // sequence-gap NACK (transport.cpp:690-707)
        a.flags |= CN_ACK_GBN | (p.nack_trim ? CN_ACK_NACK_TRIM : 0);
        a.sack[0] = p.nack_psn;
    }
    a.echo_tx_time = p.echo_tx_time;
    a.aux = aux;
    return a;
}

Packet from_ack(const cn_ack_rec& a) {
    Packet p;
    p.kind = (a.flags & CN_ACK_NACK)      ? PacketKind::nack
             : (a.flags & CN_ACK_CREDIT)  ? PacketKind::credit
             : (a.flags & CN_ACK_RTS_ACK) ? PacketKind::rts_ack
                                          : PacketKind::ack;
    if (a.flags & CN_ACK_CREDIT) p.credit_bytes = static_cast<uint32_t>(a.sack[0]);
    if (a.flags & CN_ACK_NACK) {
        p.nack_csn = a.cum_csn;
        p.nack_trim = true;
        if (a.flags & CN_ACK_GBN) {
            p.nack_psn = a.sack[0];
            p.nack_trim = (a.flags & CN_ACK_NACK_TRIM) != 0;
        }
    }
    p.src = a.src;
    p.dst = a.dst;
    p.hdr = decode_header(a.hdr);
    p.echo_path_id = a.echo_path_id;
    p.cum_csn = a.cum_csn;
    p.cum_valid = a.flags & CN_ACK_CUM_VALID;
    p.ecn_echo = a.flags & CN_ACK_ECN_ECHO;
    p.msg_seq = a.msg_seq;
    p.sack[0] = a.sack[0];
    p.sack[1] = a.sack[1];
    p.echo_tx_time = a.echo_tx_time;
    return p;
}

template <class T>
bool write_vec(const std::string& path, const std::vector<T>& v) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) return false;
    if (!v.empty()) std::fwrite(v.data(), sizeof(T), v.size(), f);
    std::fclose(f);
    return true;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------ DES recorder
struct cnref_scenario {
    int32_t topo_kind;   // 0 star, 1 fat tree
    int32_t topo_arg;    // n hosts (star) or k (fat tree)
    double rate_bps;
    int64_t link_delay_ns;
    int64_t qcap_bytes;
    double loss;         // at every host egress
    uint64_t seed;
    uint32_t chunk_bytes;
    int32_t paths;
    int32_t lb;          // LbPolicy
    int32_t cc;          // CcConfig::Algo
    int32_t cc_scope;    // CcConfig::Scope
    int32_t engines;
    int32_t conn_split;
    int32_t dupack_threshold;
    int64_t rto_min;
    int32_t n_flows;
    int32_t window;      // messages outstanding per flow
    int64_t cutoff_ns;
    int32_t queue_mode;  // QueueMode: 0 drop_tail, 1 trim, 2 pause
    int32_t trim_depth;  // NetParams::trim_queue_depth (0 = default)
    int32_t receiver_driven;  // TransportConfig::receiver_driven (EQDS)
    int32_t ordered;          // TransportConfig::reliability == ordered (go-back-N)
    int32_t policy;           // 0 DefaultPolicy, 1 round robin, 2 single path, 3 example plug-in
    int32_t pad_policy;
};

struct cnref_flow {
    int32_t src, dst;
    uint64_t len;
    int32_t count;
    int32_t pad;
};

struct cnref_record_stats {
    uint64_t data_pkts;
    uint64_t acks_at_sender;
    uint64_t completions;
    uint64_t chunks_sent;
    uint64_t chunk_rtx;
    uint64_t fast_rtx;
    uint64_t rtos;
    uint64_t acks_sent;
    uint64_t loss_dropped;
    int64_t end_time;
    int32_t quiesced;
    int32_t n_hosts;
    uint64_t bytes_ok;  // completions whose data matched the source
};

const char* cnref_last_error() { return g_err.c_str(); }

int cnref_record(const cnref_scenario* sc, const cnref_flow* flows,
                 const char* outdir, cnref_record_stats* st) {
    try {
        Topology topo =
            sc->topo_kind == 0 ? build_star(sc->topo_arg) : build_fat_tree(sc->topo_arg);
        NetParams np;
        np.rate_bps = sc->rate_bps;
        np.link_delay_ns = sc->link_delay_ns;
        np.qcap_bytes = sc->qcap_bytes;
        np.mode = static_cast<QueueMode>(sc->queue_mode);
        if (sc->trim_depth > 0) np.trim_queue_depth = sc->trim_depth;
        EventQueue eq;
        Network net(topo, np, eq, sc->seed);
        if (sc->loss > 0) net.inject_loss_at_host_egress(sc->loss);

        TransportConfig tc;
        tc.chunk_bytes = sc->chunk_bytes;
        tc.paths = sc->paths;
        tc.lb = static_cast<LbPolicy>(sc->lb);
        tc.cc.algo = static_cast<CcConfig::Algo>(sc->cc);
        tc.cc.scope = static_cast<CcConfig::Scope>(sc->cc_scope);
        if (tc.cc.algo == CcConfig::Algo::swift)
            tc.cc.swift_target_ns = 3 * net.base_rtt_ns();
        tc.engines = sc->engines;
        tc.conn_split = sc->conn_split;
        tc.dupack_threshold = sc->dupack_threshold;
        tc.rto_min = sc->rto_min;
        tc.carry_payload = true;
        tc.receiver_driven = sc->receiver_driven != 0;
        if (sc->ordered) tc.reliability = TransportConfig::Reliability::ordered;
        g_ordered = sc->ordered != 0;
        Transport tr(net, eq, tc, sc->seed);

        std::vector<cn_pkt_hdr> data;
        std::vector<uint64_t> psns;
        std::vector<cn_ack_rec> acks;
        std::vector<cn_completion> cpls;
        struct SubRec { int64_t t; uint64_t len, tag; int32_t src, dst; };
        std::vector<SubRec> subs_log;
        net.set_trace([&](const TraceEvent& te) {
            if (std::strcmp(te.event, "deliver") != 0) return;
            const Packet& p = *te.pkt;
            if (p.kind == PacketKind::data) {
                data.push_back(to_rec(p));
                psns.push_back(p.conn_psn);
            }
            else if (p.kind == PacketKind::ack || p.kind == PacketKind::nack ||
                     p.kind == PacketKind::credit || p.kind == PacketKind::rts_ack)
                acks.push_back(ack_rec(p, 0, te.t));
        });

        // tags: flow * 1'000'000 + k ; payload = pattern(len, tag)
        std::vector<int> next(sc->n_flows, 0);
        std::map<uint64_t, std::shared_ptr<std::vector<uint8_t>>> srcs;
        uint64_t ok = 0;
        std::function<void(int)> submit = [&](int f) {
            const cnref_flow& fl = flows[f];
            if (next[f] >= fl.count) return;
            uint64_t tag = uint64_t(f) * 1000000ull + uint64_t(next[f]);
            auto buf = pattern(fl.len, tag);
            if (!tr.send_message_data(fl.src, fl.dst, buf, tag)) return;  // retried on completion
            subs_log.push_back({eq.now(), fl.len, tag, fl.src, fl.dst});
            srcs[tag] = buf;
            ++next[f];
        };
        tr.set_on_complete([&](uint64_t tag, int src, int dst, uint64_t len,
                               SimTime t, const std::vector<uint8_t>* d) {
            cn_completion c;
            std::memset(&c, 0, sizeof c);
            c.tag = tag;
            c.src = src;
            c.dst = dst;
            c.len = len;
            c.reserved = static_cast<uint64_t>(t);
            cpls.push_back(c);
            auto it = srcs.find(tag);
            if (d && it != srcs.end() && *d == *it->second) ++ok;
            int f = static_cast<int>(tag / 1000000ull);
            eq.schedule_in(0, [&submit, f] { submit(f); });
        });
        for (int f = 0; f < sc->n_flows; ++f)
            for (int w = 0; w < sc->window; ++w) submit(f);
        bool q = eq.run_until_idle(sc->cutoff_ns);

        std::string dir(outdir);
        if (!write_vec(dir + "/data.bin", data) || !write_vec(dir + "/psn.bin", psns) ||
            !write_vec(dir + "/acks_des.bin", acks) ||
            !write_vec(dir + "/completions_des.bin", cpls) || !write_vec(dir + "/submits.bin", subs_log))
            throw std::runtime_error("cannot write to " + dir);
        if (st) {
            st->data_pkts = data.size();
            st->acks_at_sender = acks.size();
            st->completions = cpls.size();
            st->chunks_sent = tr.stats().chunks_sent;
            st->chunk_rtx = tr.stats().chunk_rtx;
            st->fast_rtx = tr.stats().fast_rtx;
            st->rtos = tr.stats().rtos;
            st->acks_sent = tr.stats().acks_sent;
            st->loss_dropped = net.counters().loss_dropped_pkts;
            st->end_time = eq.now();
            st->quiesced = q ? 1 : 0;
            st->n_hosts = topo.n_hosts;
            st->bytes_ok = ok;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// -------------------------------------------------------- receive replay
// Feeds recorded data packets, in order, into Transport::handle_packet of a
// fresh instance and captures every ack it emits, in emission order, with
// the index of the packet that caused it.  Completions are captured with
// their reassembled bytes copied into `arena` (if non-null) at a running
// offset.
struct cnref_rx_out {
    uint64_t n_acks;
    uint64_t n_completions;
    uint64_t arena_used;
    uint64_t acks_sent_stat;
};

int cnref_rx_replay(const cn_pkt_hdr* recs, uint64_t n, int n_hosts,
                    uint32_t chunk_bytes, int carry_payload, cn_ack_rec* acks,
                    uint64_t max_acks, cn_completion* cpls, uint64_t max_cpls,
                    uint8_t* arena, uint64_t arena_bytes, cnref_rx_out* out,
                    const uint64_t* psn, int ordered) {
    try {
        g_ordered = ordered != 0;
        Topology topo = build_star(std::max(2, n_hosts));
        NetParams np;
        np.rate_bps = 1e12;
        np.link_delay_ns = 1;
        np.qcap_bytes = int64_t{1} << 40;
        EventQueue eq;
        Network net(topo, np, eq, 1);
        TransportConfig tc;
        tc.chunk_bytes = chunk_bytes;
        tc.carry_payload = carry_payload != 0;
        if (ordered) tc.reliability = TransportConfig::Reliability::ordered;
        Transport tr(net, eq, tc, 1);

        uint64_t na = 0, nc = 0, used = 0;
        uint64_t cur = 0;
        net.set_trace([&](const TraceEvent& te) {
            if (std::strcmp(te.event, "deliver") != 0) return;
            if (te.pkt->kind != PacketKind::ack && te.pkt->kind != PacketKind::nack) return;
            if (na < max_acks) acks[na] = ack_rec(*te.pkt, static_cast<uint32_t>(cur), 0);
            ++na;
        });
        std::unordered_map<uint64_t, std::shared_ptr<std::vector<uint8_t>>> srcs;
        tr.set_on_complete([&](uint64_t tag, int src, int dst, uint64_t len,
                               SimTime, const std::vector<uint8_t>* d) {
            if (nc < max_cpls) {
                cn_completion& c = cpls[nc];
                std::memset(&c, 0, sizeof c);
                c.tag = tag;
                c.src = src;
                c.dst = dst;
                c.len = len;
                c.pkt_index = static_cast<uint32_t>(cur);
                c.buf_offset = ~uint64_t{0};
                if (d && arena && used + d->size() <= arena_bytes) {
                    std::memcpy(arena + used, d->data(), d->size());
                    c.buf_offset = used;
                    used += (d->size() + 15) & ~uint64_t{15};
                }
            }
            ++nc;
        });
        for (uint64_t i = 0; i < n; ++i) {
            Packet p = from_rec(recs[i]);
            if (psn) p.conn_psn = psn[i];
            if (carry_payload) {
                auto& s = srcs[p.msg_tag ^ (p.msg_len << 40)];
                if (!s) s = pattern(p.msg_len, p.msg_tag);
                p.msg_data = s;
            }
            cur = i;
            // msg_seq recorded per completion through the MsgRecv before reset
            tr.handle_packet(p.dst, std::move(p));
            eq.run_until_idle(std::numeric_limits<SimTime>::max() / 2);
        }
        if (out) {
            out->n_acks = na;
            out->n_completions = nc;
            out->arena_used = used;
            out->acks_sent_stat = tr.stats().acks_sent;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Times the reference receive path: T threads, each owning one Transport
// (constructed outside the timer) and its own source buffers, replay the
// same recorded packet sequence `reps` times.  Acks go into the reference's
// own Network::inject (part of the measured path, as in the survey probe);
// the event queue is drained outside the timer.  Returns wall seconds of
// the slowest thread's timed region.
double cnref_rx_replay_bench(const cn_pkt_hdr* recs, uint64_t n, int n_hosts,
                             uint32_t chunk_bytes, int threads, int reps) {
    std::vector<double> secs(threads, 0.0);
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    auto work = [&](int t) {
        Topology topo = build_star(std::max(2, n_hosts));
        NetParams np;
        np.rate_bps = 1e12;
        np.link_delay_ns = 1;
        np.qcap_bytes = int64_t{1} << 40;
        std::unordered_map<uint64_t, std::shared_ptr<std::vector<uint8_t>>> srcs;
        for (uint64_t i = 0; i < n; ++i) {
            auto& s = srcs[recs[i].msg_tag ^ (recs[i].msg_len << 40)];
            if (!s) s = pattern(recs[i].msg_len, recs[i].msg_tag);
        }
        std::vector<Packet> pk;
        pk.reserve(n);
        for (uint64_t i = 0; i < n; ++i) {
            Packet p = from_rec(recs[i]);
            p.msg_data = srcs[recs[i].msg_tag ^ (recs[i].msg_len << 40)];
            pk.push_back(std::move(p));
        }
        ready.fetch_add(1);
        while (!go.load()) std::this_thread::yield();
        double total = 0;
        for (int r = 0; r < reps; ++r) {
            EventQueue eq;
            Network net(topo, np, eq, 1);
            TransportConfig tc;
            tc.chunk_bytes = chunk_bytes;
            tc.carry_payload = true;
            Transport tr(net, eq, tc, 1);
            uint64_t sink = 0;
            tr.set_on_complete([&](uint64_t, int, int, uint64_t len, SimTime,
                                   const std::vector<uint8_t>* d) {
                sink += len + (d ? (*d)[len / 2] : 0);
            });
            std::vector<Packet> batch = pk;  // copy outside the timer
            auto t0 = std::chrono::steady_clock::now();
            for (uint64_t i = 0; i < n; ++i) {
                int dst = batch[i].dst;
                tr.handle_packet(dst, std::move(batch[i]));
            }
            auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
            eq.run_until_idle(std::numeric_limits<SimTime>::max() / 2);
            if (sink == 0xdeadbeef) std::fprintf(stderr, "!");
        }
        secs[t] = total;
    };
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
    while (ready.load() < threads) std::this_thread::yield();
    go.store(true);
    for (auto& x : th) x.join();
    return *std::max_element(secs.begin(), secs.end());
}

// --------------------------------------------------------- sender replay
// A fresh reference Transport whose data packets all vanish at the host
// egress (inject_loss_at_host_egress(1.0), the reference tests' blackhole,
// test_transport.cpp:207-295): messages are submitted at given times and
// recorded acks are delivered to the sender at their recorded times
// (Transport::handle_packet -> handle_ack, transport.cpp:849-942).  Every
// transmission is captured from the "loss" trace event of its first packet:
// (time, msg_id, chunk index, path, is_rtx).  Timers (rto_fire) run inside
// the reference event queue.
struct cnref_tx_rec {
    int64_t t;
    uint32_t msg_id;
    uint32_t chunk;
    int32_t path;
    int32_t is_rtx;
    uint64_t msg_seq;
};

struct cnref_sender_stats {
    uint64_t chunks_sent, chunk_rtx, fast_rtx, rtos, msgs_completed, n_tx;
    int64_t base_rtt, rto_min, rto_max, end_time;
    int32_t n_paths, pad;
    int64_t bdp, commit_ahead;
    uint64_t rts_sent;
};

struct cnref_submit {
    int64_t t;
    uint64_t len;
    uint64_t tag;
};

// Probes for the next cnref_sender_replay on this thread: at each time t[i]
// (relative, like the inputs) the reference's introspection is written to
// out[i * stride ...]: outstanding_bytes, conn_credit, engine_inflight_msgs,
// engine_dispatched, engine_gauge, then (path_inflight, window_available)
// per path.  n = 0 clears.
void cnref_set_probes(const int64_t* t, uint32_t n, int64_t* out, uint32_t stride) {
    g_probe_t.assign(t, t + n);
    g_probe_out = out;
    g_probe_stride = stride;
}

int cnref_sender_replay(const cnref_scenario* sc, int src, int dst, const cnref_submit* subs,
                        uint64_t n_subs, const cn_ack_rec* acks, uint64_t n_acks,
                        cnref_tx_rec* out, uint64_t max_out, cnref_sender_stats* st) {
    try {
        Topology topo =
            sc->topo_kind == 0 ? build_star(sc->topo_arg) : build_fat_tree(sc->topo_arg);
        NetParams np;
        np.rate_bps = sc->rate_bps;
        np.link_delay_ns = sc->link_delay_ns;
        np.qcap_bytes = sc->qcap_bytes;
        np.mode = static_cast<QueueMode>(sc->queue_mode);
        if (sc->trim_depth > 0) np.trim_queue_depth = sc->trim_depth;
        EventQueue eq;
        Network net(topo, np, eq, sc->seed);
        net.inject_loss_at_host_egress(1.0);
        TransportConfig tc;
        tc.chunk_bytes = sc->chunk_bytes;
        tc.paths = sc->paths;
        tc.lb = static_cast<LbPolicy>(sc->lb);
        tc.cc.algo = static_cast<CcConfig::Algo>(sc->cc);
        tc.cc.scope = static_cast<CcConfig::Scope>(sc->cc_scope);
        if (tc.cc.algo == CcConfig::Algo::swift) tc.cc.swift_target_ns = 3 * net.base_rtt_ns();
        tc.engines = 1;
        tc.dupack_threshold = sc->dupack_threshold;
        tc.rto_min = sc->rto_min;
        tc.receiver_driven = sc->receiver_driven != 0;
        if (sc->ordered) tc.reliability = TransportConfig::Reliability::ordered;
        g_ordered = sc->ordered != 0;
        Transport tr(net, eq, tc, sc->seed);
        install_policy(tr, sc->policy, tc.chunk_bytes);
        if (tc.receiver_driven) tr.pacers_[dst].reset();  // the recorded credits drive the sender
        // Control packets skip the egress blackhole and reach the receiver: an
        // RTS is logged at delivery minus the (empty-fabric, constant) one-way
        // control latency of this pair, measured with a probe at t = 0.
        int64_t ctl_lat = -1;
        if (tc.receiver_driven) {
            Packet probe;
            probe.kind = PacketKind::rts;
            probe.src = src;
            probe.dst = dst;
            net.set_trace([&](const TraceEvent& te) {
                if (std::strcmp(te.event, "deliver") == 0 && te.pkt->kind == PacketKind::rts) ctl_lat = te.t;
            });
            net.inject(std::move(probe));
            eq.run_until_idle(int64_t{1} << 40);
            if (ctl_lat < 0) throw std::runtime_error("control latency probe lost");
        }
        const int64_t t0 = eq.now();  // inputs are scheduled relative to the probe's end (0 without)
        uint64_t n_out = 0;
        uint64_t last_key = ~uint64_t{0};
        uint32_t last_sq = 0;
        net.set_trace([&](const TraceEvent& te) {
            if (tc.receiver_driven && std::strcmp(te.event, "deliver") == 0 && te.pkt->kind == PacketKind::rts) {
                if (n_out < max_out) {
                    cnref_tx_rec& r = out[n_out];
                    r.t = te.t - ctl_lat - t0;
                    r.msg_id = 0;
                    r.chunk = 0xFFFFFFFFu;  // RTS record
                    r.path = -1;
                    r.is_rtx = te.pkt->is_rtx ? 1 : 0;
                    r.msg_seq = te.pkt->demand_bytes;
                }
                ++n_out;
                return;
            }
            if (std::strcmp(te.event, "loss") != 0) return;
            const Packet& p = *te.pkt;
            if (p.kind != PacketKind::data) return;
            // the first packet of each send_chunk call: a new (msg, chunk) or a
            // restart of the same one (a go-back-N resend may start mid-chunk)
            const uint64_t key = (static_cast<uint64_t>(p.msg_seq) << 32) ^ (p.chunk_offset / tc.chunk_bytes);
            const bool first = key != last_key || p.seq_in_chunk <= last_sq;
            last_key = key;
            last_sq = p.seq_in_chunk;
            if (!first) return;
            if (n_out < max_out) {
                cnref_tx_rec& r = out[n_out];
                r.t = te.t - t0;
                r.msg_id = p.hdr.msg_id;
                r.chunk = static_cast<uint32_t>(p.chunk_offset / tc.chunk_bytes);
                r.path = p.path_id | static_cast<int32_t>(p.seq_in_chunk << 16);  // + first packet sent
                r.is_rtx = p.is_rtx ? 1 : 0;
                r.msg_seq = p.msg_seq;
            }
            ++n_out;
        });
        for (uint64_t k = 0; k < n_subs; ++k) {
            cnref_submit sb = subs[k];
            eq.schedule(t0 + sb.t, [&tr, src, dst, sb] { tr.send_message(src, dst, sb.len, sb.tag); });
        }
        for (uint64_t k = 0; k < n_acks; ++k) {
            cn_ack_rec a = acks[k];
            eq.schedule(t0 + a.aux, [&tr, a, t0] {
                Packet p = from_ack(a);
                p.echo_tx_time += t0;  // the same shift as every send time
                int host = p.dst;
                tr.handle_packet(host, std::move(p));
            });
        }
        // Transport introspection (transport.cpp:1173-1209) at the probe times
        for (size_t i = 0; i < g_probe_t.size(); ++i) {
            int64_t* o = g_probe_out + i * g_probe_stride;
            const uint32_t w = g_probe_stride;
            eq.schedule(t0 + g_probe_t[i], [&tr, o, w, src, dst] {
                o[0] = tr.outstanding_bytes(src, dst);
                o[1] = tr.conn_credit(src, dst);
                o[2] = tr.engine_inflight_msgs(src, 0);
                o[3] = static_cast<int64_t>(tr.engine_dispatched(src, 0));
                o[4] = tr.engine_gauge(src, 0);
                for (uint32_t p = 0; 6 + 2 * p < w; ++p) {
                    o[5 + 2 * p] = tr.path_inflight(src, dst, static_cast<int>(p));
                    o[6 + 2 * p] = tr.window_available(src, dst, static_cast<int>(p));
                }
            });
        }
        eq.run_until_idle(sc->cutoff_ns);
        if (st) {
            st->chunks_sent = tr.stats().chunks_sent;
            st->chunk_rtx = tr.stats().chunk_rtx;
            st->fast_rtx = tr.stats().fast_rtx;
            st->rtos = tr.stats().rtos;
            st->msgs_completed = tr.stats().msgs_completed;
            st->n_tx = n_out;
            st->base_rtt = net.base_rtt_ns();
            st->rto_min = tr.rto_min_;
            st->rto_max = tr.rto_max_;
            st->end_time = eq.now() - t0;
            st->n_paths = tr.conns_.empty() ? 0 : static_cast<int>(tr.conns_[0].subs.size());
            st->bdp = net.bdp_bytes();
            st->commit_ahead = tr.commit_ahead_;
            st->rts_sent = tr.stats().rts_sent;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ------------------------------------------------------ host-level replay
// The reference sender of ONE source host with several connections (fan-out,
// engines, conn_split): every send_message of `src` (to its dst) and every
// ack / NACK / credit / rts_ack delivered at `src`, at their times, into a
// fresh Transport over a blackhole.  Connections open lazily in the
// replay's own conn_to order; conns_out[k] = dst of connection index k.
// Transmissions are logged in emission order with the connection index.
struct cnref_host_submit {
    int64_t t;
    uint64_t len;
    uint64_t tag;
    int32_t dst;
    int32_t pad;
};

struct cnref_host_tx {
    int64_t t;
    uint32_t msg_id;
    uint32_t chunk;
    int32_t path;
    int32_t is_rtx;
    uint64_t msg_seq;
    uint32_t conn;
    int32_t dst;
};

// probes: at each t[i], per engine e (inflight_msgs, dispatched, gauge), then
// per connection k < n_conn_probe: (outstanding, credit, then per path p <
// n_path_probe: path_inflight, window_available)
thread_local std::vector<int64_t> g_hprobe_t;
thread_local int64_t* g_hprobe_out = nullptr;
thread_local uint32_t g_hprobe_conns = 0, g_hprobe_paths = 0;

void cnref_set_host_probes(const int64_t* t, uint32_t n, int64_t* out, uint32_t n_conns, uint32_t n_paths) {
    g_hprobe_t.assign(t, t + n);
    g_hprobe_out = out;
    g_hprobe_conns = n_conns;
    g_hprobe_paths = n_paths;
}

int cnref_host_replay(const cnref_scenario* sc, int src, const cnref_host_submit* subs, uint64_t n_subs,
                      const cn_ack_rec* acks, uint64_t n_acks, cnref_host_tx* out, uint64_t max_out,
                      cnref_sender_stats* st, int32_t* conns_out, uint32_t max_conns, int32_t ecn_as_loss,
                      int32_t max_inflight_msgs) {
    try {
        Topology topo =
            sc->topo_kind == 0 ? build_star(sc->topo_arg) : build_fat_tree(sc->topo_arg);
        NetParams np;
        np.rate_bps = sc->rate_bps;
        np.link_delay_ns = sc->link_delay_ns;
        np.qcap_bytes = sc->qcap_bytes;
        np.mode = static_cast<QueueMode>(sc->queue_mode);
        if (sc->trim_depth > 0) np.trim_queue_depth = sc->trim_depth;
        EventQueue eq;
        Network net(topo, np, eq, sc->seed);
        net.inject_loss_at_host_egress(1.0);
        TransportConfig tc;
        tc.chunk_bytes = sc->chunk_bytes;
        tc.paths = sc->paths;
        tc.lb = static_cast<LbPolicy>(sc->lb);
        tc.cc.algo = static_cast<CcConfig::Algo>(sc->cc);
        tc.cc.scope = static_cast<CcConfig::Scope>(sc->cc_scope);
        tc.cc.ecn_as_loss = ecn_as_loss != 0;
        if (tc.cc.algo == CcConfig::Algo::swift) tc.cc.swift_target_ns = 3 * net.base_rtt_ns();
        tc.engines = sc->engines;
        tc.conn_split = sc->conn_split != 0;
        if (max_inflight_msgs > 0) tc.max_inflight_msgs = max_inflight_msgs;
        tc.dupack_threshold = sc->dupack_threshold;
        tc.rto_min = sc->rto_min;
        tc.receiver_driven = sc->receiver_driven != 0;
        if (sc->ordered) tc.reliability = TransportConfig::Reliability::ordered;
        g_ordered = sc->ordered != 0;
        Transport tr(net, eq, tc, sc->seed);
        install_policy(tr, sc->policy, tc.chunk_bytes);
        std::map<int, int64_t> ctl_lat;  // per destination: one-way control latency (RTS logging)
        if (tc.receiver_driven) {
            for (uint64_t k = 0; k < n_subs; ++k) {
                const int dst = subs[k].dst;
                if (ctl_lat.count(dst)) continue;
                tr.pacers_[dst].reset();  // the recorded credits drive the sender
                int64_t lat = -1;
                const int64_t t_start = eq.now();
                Packet probe;
                probe.kind = PacketKind::rts;
                probe.src = src;
                probe.dst = dst;
                net.set_trace([&](const TraceEvent& te) {
                    if (std::strcmp(te.event, "deliver") == 0 && te.pkt->kind == PacketKind::rts) lat = te.t - t_start;
                });
                net.inject(std::move(probe));
                eq.run_until_idle(int64_t{1} << 40);
                if (lat < 0) throw std::runtime_error("control latency probe lost");
                ctl_lat[dst] = lat;
            }
        }
        const int64_t t0 = eq.now();
        uint64_t n_out = 0;
        // the first packet of each send_chunk call (its packets are injected
        // back to back): a new (dst, msg, chunk) or a restart of the same one
        int last_dst = -1;
        uint64_t last_key = ~uint64_t{0};
        uint32_t last_sq = 0;
        auto conn_of = [&](int dst) -> int {
            auto it = tr.hosts_[src].conn_by_dst.find(dst);
            return it == tr.hosts_[src].conn_by_dst.end() ? -1 : it->second;
        };
        // RTS packets (control, exempt from the blackhole) are seen at
        // delivery; their send times come from stepping the event loop and
        // counting Stats::rts_sent per event (one control FIFO per host
        // egress: deliveries keep the send order on equal-latency paths)
        std::vector<cnref_host_tx> rts_rec;
        std::vector<int64_t> rts_sent_t;
        net.set_trace([&](const TraceEvent& te) {
            if (tc.receiver_driven && std::strcmp(te.event, "deliver") == 0 && te.pkt->kind == PacketKind::rts) {
                cnref_host_tx r;
                r.t = te.t;  // delivery time, replaced by the send time below
                r.msg_id = 0;
                r.chunk = 0xFFFFFFFFu;  // RTS record
                r.path = -1;
                r.is_rtx = te.pkt->is_rtx ? 1 : 0;
                r.msg_seq = te.pkt->demand_bytes;
                r.conn = static_cast<uint32_t>(conn_of(te.pkt->dst));
                r.dst = te.pkt->dst;
                rts_rec.push_back(r);
                return;
            }
            if (std::strcmp(te.event, "loss") != 0) return;
            const Packet& p = *te.pkt;
            if (p.kind != PacketKind::data) return;
            const uint64_t key = (static_cast<uint64_t>(p.msg_seq) << 32) ^ (p.chunk_offset / tc.chunk_bytes);
            const bool first = p.dst != last_dst || key != last_key || p.seq_in_chunk <= last_sq;
            last_dst = p.dst;
            last_key = key;
            last_sq = p.seq_in_chunk;
            if (!first) return;
            if (n_out < max_out) {
                cnref_host_tx& r = out[n_out];
                r.t = te.t - t0;
                r.msg_id = p.hdr.msg_id;
                r.chunk = static_cast<uint32_t>(p.chunk_offset / tc.chunk_bytes);
                r.path = p.path_id | static_cast<int32_t>(p.seq_in_chunk << 16);
                r.is_rtx = p.is_rtx ? 1 : 0;
                r.msg_seq = p.msg_seq;
                r.conn = static_cast<uint32_t>(conn_of(p.dst));
                r.dst = p.dst;
            }
            ++n_out;
        });
        for (uint64_t k = 0; k < n_subs; ++k) {
            cnref_host_submit sb = subs[k];
            eq.schedule(t0 + sb.t, [&tr, src, sb] { tr.send_message(src, sb.dst, sb.len, sb.tag); });
        }
        for (uint64_t k = 0; k < n_acks; ++k) {
            cn_ack_rec a = acks[k];
            eq.schedule(t0 + a.aux, [&tr, a, t0] {
                Packet p = from_ack(a);
                p.echo_tx_time += t0;
                int host = p.dst;
                tr.handle_packet(host, std::move(p));
            });
        }
        for (size_t i = 0; i < g_hprobe_t.size(); ++i) {
            const uint32_t ne = static_cast<uint32_t>(tc.engines), nk = g_hprobe_conns, npp = g_hprobe_paths;
            int64_t* o = g_hprobe_out + i * (3 * ne + nk * (2 + 2 * npp));
            eq.schedule(t0 + g_hprobe_t[i], [&tr, o, ne, nk, npp, src] {
                int64_t* q = o;
                for (uint32_t e = 0; e < ne; ++e) {
                    *q++ = tr.engine_inflight_msgs(src, static_cast<int>(e));
                    *q++ = static_cast<int64_t>(tr.engine_dispatched(src, static_cast<int>(e)));
                    *q++ = tr.engine_gauge(src, static_cast<int>(e));
                }
                for (uint32_t k = 0; k < nk; ++k) {
                    const int dst = k < tr.conns_.size() ? tr.conns_[k].dst : -1;
                    *q++ = dst >= 0 ? tr.outstanding_bytes(src, dst) : 0;
                    *q++ = dst >= 0 ? tr.conn_credit(src, dst) : 0;
                    for (uint32_t p = 0; p < npp; ++p) {
                        *q++ = dst >= 0 ? tr.path_inflight(src, dst, static_cast<int>(p)) : 0;
                        *q++ = dst >= 0 ? tr.window_available(src, dst, static_cast<int>(p)) : 0;
                    }
                }
            });
        }
        while (!eq.heap_.empty() && eq.heap_.top().t <= sc->cutoff_ns) {  // EventQueue::run_until_idle, stepped
            auto e = eq.heap_.top();
            eq.heap_.pop();
            eq.now_ = e.t;
            const uint64_t before = tr.stats_.rts_sent;
            e.fn();
            for (uint64_t i = before; i < tr.stats_.rts_sent; ++i) rts_sent_t.push_back(e.t);
        }
        if (tc.receiver_driven) {
            std::stable_sort(rts_rec.begin(), rts_rec.end(),
                             [](const cnref_host_tx& a, const cnref_host_tx& b) { return a.t < b.t; });
            for (size_t i = 0; i < rts_rec.size(); ++i) {
                cnref_host_tx r = rts_rec[i];
                if (i >= rts_sent_t.size() || rts_sent_t[i] + ctl_lat[r.dst] > r.t)
                    throw std::runtime_error("RTS send / delivery pairing failed");
                r.t = rts_sent_t[i] - t0;
                if (n_out < max_out) out[n_out] = r;
                ++n_out;
            }
        }
        for (size_t k = 0; k < tr.conns_.size() && k < max_conns; ++k) conns_out[k] = tr.conns_[k].dst;
        if (st) {
            st->chunks_sent = tr.stats().chunks_sent;
            st->chunk_rtx = tr.stats().chunk_rtx;
            st->fast_rtx = tr.stats().fast_rtx;
            st->rtos = tr.stats().rtos;
            st->msgs_completed = tr.stats().msgs_completed;
            st->n_tx = n_out;
            st->base_rtt = net.base_rtt_ns();
            st->rto_min = tr.rto_min_;
            st->rto_max = tr.rto_max_;
            st->end_time = eq.now() - t0;
            st->n_paths = static_cast<int>(tr.conns_.size());  // connections opened
            st->bdp = net.bdp_bytes();
            st->commit_ahead = tr.commit_ahead_;
            st->rts_sent = tr.stats().rts_sent;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ------------------------------------------------ randomized scenarios
// The reference's own scenario draws (tests/test_reliability_props.cpp:
// run_scenario :126-218 and the engine-invariance case :328-358), restated
// draw for draw over its RngStream so the generator's scenarios are
// exactly the reference suite's.  kind 0: "prop-scenario" (1,000-scenario
// suite), kind 1: "prop-engines" (engines 1 / 2 / 4 run the same specs).
struct cnref_prop_spec {
    int32_t star, topo_arg, ordered, receiver_driven, zero_loss, engines, conn_split, paths, lb, cc, cc_scope,
        n_msgs;
    uint32_t chunk_bytes, pad;
    double rate_bps, drop;
    int64_t link_delay_ns;
    int32_t src[8], dst[8];
    uint64_t len[8], tag[8];
};

int cnref_prop_spec_draw(uint64_t seed, int kind, cnref_prop_spec* o) {
    std::memset(o, 0, sizeof *o);
    if (kind == 0) {
        RngStream rng(seed, "prop-scenario");
        bool star = rng.next_below(4) == 0;
        o->star = star;
        o->topo_arg = star ? 8 : 4;
        const int n_hosts = star ? 8 : 16;  // build_star(8) / build_fat_tree(4)
        o->rate_bps = rng.next_below(2) ? 100e9 : 10e9;
        o->link_delay_ns = rng.next_below(2) ? 1000 : 200;
        o->zero_loss = seed % 4 == 0;
        o->drop = 0.0;
        if (!o->zero_loss) o->drop = (1.0 / 256) + rng.next_double() * (1.0 / 64 - 1.0 / 256);
        static const uint32_t kChunks[] = {4032, 8064, 16128, 32768};
        o->chunk_bytes = kChunks[rng.next_below(4)];
        static const int kPaths[] = {1, 2, 4, 8};
        o->paths = kPaths[rng.next_below(4)];
        o->engines = rng.next_below(2) ? 2 : 1;
        o->conn_split = o->engines > 1 && rng.next_below(2) == 0;
        o->lb = static_cast<int>(rng.next_below(3));
        switch (rng.next_below(3)) {
            case 0: o->cc = 0; break;
            case 1: o->cc = 1; break;
            default: o->cc = 2; break;
        }
        o->cc_scope = rng.next_below(2) ? 1 : 0;
        o->receiver_driven = seed % 10 == 3;
        o->ordered = seed % 10 == 7;
        if (o->receiver_driven) o->cc = 0;
        if (o->ordered) {
            o->paths = 1;
            o->engines = 1;
            o->conn_split = 0;
            o->receiver_driven = 0;
            if (o->cc == 2) o->cc = 1;
        }
        o->n_msgs = 3 + static_cast<int>(rng.next_below(3));
        for (int i = 0; i < o->n_msgs; ++i) {
            o->src[i] = static_cast<int>(rng.next_below(n_hosts));
            o->dst[i] = static_cast<int>(rng.next_below(n_hosts - 1));
            if (o->dst[i] >= o->src[i]) ++o->dst[i];
            uint64_t len = 4032 * (1 + rng.next_below(48)) + rng.next_below(4032);
            if (i == 1 && seed % 8 == 0) len = 1 + rng.next_below(4032);
            if (i == 0 && seed % 16 == 0) len = 1;
            o->len[i] = len;
            o->tag[i] = seed * 100 + static_cast<uint64_t>(i);
        }
        return 0;
    }
    RngStream rng(seed, "prop-engines");
    o->star = 0;
    o->topo_arg = 4;
    o->rate_bps = 100e9;
    o->link_delay_ns = 500;
    o->drop = 1.0 / 128;
    o->paths = 4;
    o->chunk_bytes = 16128;
    o->cc = 1;
    o->lb = 1;
    o->n_msgs = 6;
    for (int i = 0; i < 6; ++i) {
        o->src[i] = static_cast<int>(rng.next_below(16));
        o->dst[i] = static_cast<int>(rng.next_below(15));
        if (o->dst[i] >= o->src[i]) ++o->dst[i];
        o->len[i] = 1 + rng.next_below(65536);
        o->tag[i] = 1000 + static_cast<uint64_t>(i);
    }
    return 0;
}

// Times the reference sender on the same replay (construction and event
// scheduling outside the timer): T threads x reps replays.  Returns the
// slowest thread's seconds.
double cnref_sender_replay_bench(const cnref_scenario* sc, int src, int dst,
                                 const cnref_submit* subs, uint64_t n_subs,
                                 const cn_ack_rec* acks, uint64_t n_acks, int threads,
                                 int reps) {
    std::vector<double> secs(threads, 0.0);
    auto work = [&](int t) {
        Topology topo =
            sc->topo_kind == 0 ? build_star(sc->topo_arg) : build_fat_tree(sc->topo_arg);
        double total = 0;
        for (int r = 0; r < reps; ++r) {
            NetParams np;
            np.rate_bps = sc->rate_bps;
            np.link_delay_ns = sc->link_delay_ns;
            np.qcap_bytes = sc->qcap_bytes;
            EventQueue eq;
            Network net(topo, np, eq, sc->seed);
            net.inject_loss_at_host_egress(1.0);
            TransportConfig tc;
            tc.chunk_bytes = sc->chunk_bytes;
            tc.paths = sc->paths;
            tc.lb = static_cast<LbPolicy>(sc->lb);
            tc.engines = 1;
            tc.dupack_threshold = sc->dupack_threshold;
            Transport tr(net, eq, tc, sc->seed);
            for (uint64_t k = 0; k < n_subs; ++k) {
                cnref_submit sb = subs[k];
                eq.schedule(sb.t, [&tr, src, dst, sb] { tr.send_message(src, dst, sb.len, sb.tag); });
            }
            for (uint64_t k = 0; k < n_acks; ++k) {
                cn_ack_rec a = acks[k];
                eq.schedule(a.aux, [&tr, a] {
                    Packet p = from_ack(a);
                    int host = p.dst;
                    tr.handle_packet(host, std::move(p));
                });
            }
            auto t0 = std::chrono::steady_clock::now();
            eq.run_until_idle(sc->cutoff_ns);
            auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
        }
        secs[t] = total;
    };
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    return *std::max_element(secs.begin(), secs.end());
}

// ------------------------------------------------------------- RNG draws
void cnref_rng_u64(uint64_t seed, const char* name, int64_t index, uint64_t count,
                   uint64_t* out) {
    RngStream r = index < 0 ? RngStream(seed, name)
                            : RngStream(seed, name, static_cast<uint64_t>(index));
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

void cnref_next_below(uint64_t seed, const char* name, int64_t index,
                      const uint64_t* ns, uint64_t count, uint64_t* out) {
    RngStream r = index < 0 ? RngStream(seed, name)
                            : RngStream(seed, name, static_cast<uint64_t>(index));
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next_below(ns[i]);
}

void cnref_next_double(uint64_t seed, const char* name, int64_t index,
                       uint64_t count, double* out) {
    RngStream r = index < 0 ? RngStream(seed, name)
                            : RngStream(seed, name, static_cast<uint64_t>(index));
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next_double();
}

// select_path sequence on a fixed scoreboard (rtt/ecn scores given).
int cnref_select_paths(int policy, int n_paths, const double* rtt,
                       const double* ecn, uint64_t seed, const char* name,
                       int64_t index, uint64_t count, int32_t* out) {
    PathScoreboard b(n_paths, 0);
    for (int p = 0; p < n_paths; ++p) {
        b.rtt_[p] = rtt ? rtt[p] : 0.0;
        b.ecn_[p] = ecn ? ecn[p] : 0.0;
    }
    RngStream r = index < 0 ? RngStream(seed, name)
                            : RngStream(seed, name, static_cast<uint64_t>(index));
    for (uint64_t i = 0; i < count; ++i)
        out[i] = select_path(static_cast<LbPolicy>(policy), b, r);
    return 0;
}

// Times select_path: `conns` connections each with its own stream and
// board; `count` decisions per connection, round robin.  Returns seconds.
double cnref_select_paths_bench(int policy, int n_paths, int conns,
                                uint64_t count, int threads, uint64_t* checksum) {
    std::vector<double> secs(threads, 0.0);
    std::vector<uint64_t> sums(threads, 0);
    auto work = [&](int t) {
        int lo = conns * t / threads, hi = conns * (t + 1) / threads;
        std::vector<PathScoreboard> boards;
        std::vector<RngStream> rngs;
        for (int c = lo; c < hi; ++c) {
            boards.emplace_back(n_paths, 10000);
            RngStream init(77, "board", c);
            for (int p = 0; p < n_paths; ++p)
                boards.back().rtt_[p] = 10000.0 + double(init.next_below(5000));
            rngs.emplace_back(1, "transport.conn", c);
        }
        uint64_t s = 0;
        auto t0 = std::chrono::steady_clock::now();
        for (uint64_t k = 0; k < count; ++k)
            for (int c = 0; c < hi - lo; ++c)
                s += select_path(static_cast<LbPolicy>(policy), boards[c], rngs[c]);
        auto t1 = std::chrono::steady_clock::now();
        secs[t] = std::chrono::duration<double>(t1 - t0).count();
        sums[t] = s;
    };
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    uint64_t s = 0;
    for (auto v : sums) s += v;
    if (checksum) *checksum = s;
    return *std::max_element(secs.begin(), secs.end());
}

// ------------------------------------------------------------ wire codec
int cnref_encode_header(uint8_t conn, uint8_t msg, uint8_t csn, int last,
                        uint8_t rsvd, uint32_t* out) {
    try {
        *out = encode_header({conn, msg, csn, last != 0, rsvd});
        return 0;
    } catch (const FieldRangeError& e) {
        g_err = e.what();
        return CN_E_FIELD_RANGE;
    }
}

int cnref_csn_before(uint8_t a, uint8_t b, uint8_t base, int width, int* out) {
    try {
        SeqWindow w(base, width);
        *out = csn_before(a, b, w) ? 1 : 0;
        return 0;
    } catch (const OutOfWindowError& e) {
        g_err = e.what();
        return CN_E_OUT_OF_WINDOW;
    } catch (const FieldRangeError& e) {
        g_err = e.what();
        return CN_E_FIELD_RANGE;
    }
}

// EqdsReceiver (eqds.cpp) driven by a scripted event stream: every input
// scheduled at its time (in list order for ties), ticks as the pacer
// schedules them, run to cutoff.  Log records: grants and rts_acks in the
// order the callbacks fire.
struct cnref_eqds_event { int64_t t; int32_t type; int32_t sender; uint64_t arg; int32_t flag; int32_t pad; };
struct cnref_eqds_log { int64_t t; int32_t sender; uint32_t bytes; int32_t kind; int32_t pad; };
int cnref_eqds_replay(uint32_t quantum, int64_t tick_ns, int64_t bank_cap, int32_t grant_to_idle,
                      const cnref_eqds_event* ev, uint64_t n, int64_t cutoff, cnref_eqds_log* out,
                      uint64_t cap, uint64_t* n_out, uint64_t* grants_sent) {
    try {
        EventQueue eq;
        EqdsParams p;
        p.quantum = quantum;
        p.tick_ns = tick_ns;
        p.bank_cap = bank_cap;
        p.grant_to_idle = grant_to_idle != 0;
        uint64_t k = 0;
        auto put = [&](int32_t sender, uint32_t bytes, int32_t kind) {
            if (k < cap) out[k] = cnref_eqds_log{eq.now(), sender, bytes, kind, 0};
            ++k;
        };
        EqdsReceiver pacer(
            eq, p, [&](int s, uint32_t b) { put(s, b, 0); }, [&](int s) { put(s, 0, 1); });
        for (uint64_t i = 0; i < n; ++i) {
            cnref_eqds_event e = ev[i];
            eq.schedule(e.t, [&pacer, e] {
                if (e.type == 0)
                    pacer.on_rts(e.sender, e.arg, e.flag != 0);
                else if (e.type == 1)
                    pacer.on_chunk(e.sender, static_cast<uint32_t>(e.arg), e.flag != 0);
                else
                    pacer.on_trim(e.sender, static_cast<uint32_t>(e.arg));
            });
        }
        eq.run_until_idle(cutoff);
        *n_out = k;
        if (grants_sent) *grants_sent = pacer.grants_sent();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference's own experiment runner (ExperimentSpec INI text ->
// run_experiment) with run.trace = true: its trace.tsv text (experiment.cpp
// trace_line) -- golden input for the trace writer.  Returns the full length;
// copies at most cap bytes.
int64_t cnref_experiment_trace(const char* ini, char* out, uint64_t cap) {
    try {
        ExperimentSpec spec = ExperimentSpec::from_text(ini);
        spec.set("run.trace", "true");
        RunOutput ro = run_experiment(spec.plan());
        const std::string& t = ro.trace_tsv;
        if (out && cap) std::memcpy(out, t.data(), std::min<uint64_t>(cap, t.size()));
        return static_cast<int64_t>(t.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
