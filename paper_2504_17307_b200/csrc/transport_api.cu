// transport_api.cu -- the drop-in boundary in the shape of chunknet::Transport
// (/root/reference/proj/include/chunknet/transport.hpp:53-107).
//
// Host C++ around the device engines: the sender engine (tx.cu, every
// connection the object opens) and the receive path (rx.cu).  The
// reference's Transport is driven by its discrete-event loop -- every call
// acts at eq.now().  Here the caller's clock is explicit: send_message and
// the acks delivered at the senders are queued with their times,
// cn_transport_advance runs the device sender over the queue (timers up to
// a horizon), and the transmissions, ack/NACK records and completions are
// polled.  Connections open on first use in conn_to order (transport.cpp:
// 84-137), which fixes each one's RngStream index.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <numeric>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

using cnb::set_error;

namespace {

struct Ev {
    int64_t t;
    uint32_t type;  // 0 submit, 1 ack / NACK (events at one instant: submits first)
    uint32_t conn;
    uint64_t idx;
};

template <class T>
bool grow(T** p, uint64_t* cap, uint64_t need) {
    if (need <= *cap) return true;
    uint64_t c = std::max<uint64_t>(need, *cap * 2 + 64);
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (cudaMalloc(p, c * sizeof(T)) != cudaSuccess) {
        *cap = 0;
        return false;
    }
    *cap = c;
    return true;
}

}  // namespace

struct cn_transport {
    cn_transport_config c{};
    cn_rx* rx = nullptr;
    cn_tx* tx = nullptr;
    std::map<std::pair<int32_t, int32_t>, int32_t> conn_idx;
    std::vector<int32_t> conn_src;       // per connection
    std::vector<std::vector<Ev>> pend;   // per tx host
    std::vector<cn_tx_submit> subs;
    std::vector<cn_ack_rec> acks;
    cn_tx_rec* d_log = nullptr;
    cn_tx_stats* d_stats = nullptr;
    uint32_t* d_evoff = nullptr;
    uint64_t* d_ev = nullptr;
    cn_tx_submit* d_subs = nullptr;
    cn_ack_rec* d_ain = nullptr;
    uint64_t cap_ev = 0, cap_subs = 0, cap_ain = 0, cap_evoff = 0;
    cn_ack_rec* d_aout = nullptr;
    cn_completion* d_cpls = nullptr;
    cn_rx_result* d_res = nullptr;
    std::vector<cn_ack_rec> last_acks;
    std::vector<cn_completion> last_cpls;
    std::vector<cn_tx_stats> txs;
    uint64_t acks_sent = 0, nacks_sent = 0, delivered = 0;
};

extern "C" void cn_transport_config_default(cn_transport_config* c) {
    memset(c, 0, sizeof *c);
    c->engines = 1;      // TransportConfig defaults (transport.hpp:23-51)
    c->paths = 1;
    c->chunk_bytes = 32768;
    c->lb = CN_LB_OBLIVIOUS;
    c->max_inflight_msgs = 128;
    c->drr_quantum = 32768;
    c->rtx_avoid_prev_path = 1;
    c->dupack_threshold = 8;
    c->initial_credit = -1;
    c->credit_quantum = 32768;
    c->credit_bank_quanta = 4;
    c->cc_algo = CN_CC_NONE;  // CcConfig defaults (cc.hpp:37-51)
    c->mss = 4032;
    c->init_cwnd_pkts = 2.0;
    c->base_rtt_ns = 10000.0;
    c->max_conns = 64;
    c->max_batch = 1 << 16;
    c->log_cap = 1 << 16;
    c->chunk_pool = 1 << 20;
    c->arena_bytes = 64ull << 20;
}

extern "C" void cn_transport_destroy(cn_transport* h) {
    if (!h) return;
    cudaDeviceSynchronize();
    if (h->tx) cn_tx_destroy(h->tx);
    if (h->rx) cn_rx_destroy(h->rx);
    void* p[] = {h->d_log, h->d_stats, h->d_evoff, h->d_ev, h->d_subs, h->d_ain, h->d_aout, h->d_cpls, h->d_res};
    for (void* x : p)
        if (x) cudaFree(x);
    delete h;
}

extern "C" int cn_transport_create(const cn_transport_config* cfg, uint64_t seed, cn_transport** out) {
    if (!cfg || !out || !cfg->max_conns || !cfg->chunk_bytes || cfg->paths < 1 || cfg->rto_min <= 0) {
        set_error("cn_transport_create: bad config (paths >= 1, resolved rto_min > 0, max_conns > 0)");
        return CN_E_INVALID;
    }
    if (cfg->reliability == 1 && cfg->paths > 1) {
        set_error("cn_transport_create: ordered reliability with multipath (transport.cpp:21-26)");
        return CN_E_LOGIC;
    }
    if (cfg->engines < 1 || cfg->engines > 16 || cfg->reliability < 0 || cfg->reliability > 1 ||
        cfg->cc_algo < CN_CC_NONE || cfg->cc_algo > CN_CC_SWIFT || cfg->cc_scope < 0 || cfg->cc_scope > 1) {
        set_error("cn_transport_create: engines 1..16, reliability selective / ordered, cc none / cubic / swift, "
                  "scope global / per_path");
        return CN_E_INVALID;
    }
    if (cfg->reliability == 1 && (cfg->engines != 1 || cfg->conn_split)) {
        set_error("cn_transport_create: ordered delivery needs a single path and a single engine (transport.cpp:21-26)");
        return CN_E_LOGIC;
    }
    if (cfg->receiver_driven && cfg->initial_credit < 0) {
        // the reference resolves -1 to one BDP of its Network (transport.cpp:40-44)
        set_error("cn_transport_create: receiver_driven needs initial_credit resolved (one BDP, >= 0)");
        return CN_E_INVALID;
    }
    *out = nullptr;
    cn_transport* h = new (std::nothrow) cn_transport();
    if (!h) return CN_E_CAPACITY;
    h->c = *cfg;
    cn_tx_config tc;
    cn_tx_config_default(&tc);
    tc.chunk_bytes = cfg->chunk_bytes;
    tc.dupack_threshold = cfg->dupack_threshold;
    tc.rtx_avoid_prev_path = cfg->rtx_avoid_prev_path;
    tc.lb_policy = cfg->lb;
    tc.max_inflight_msgs = cfg->max_inflight_msgs;
    tc.max_paths = cfg->paths;
    tc.log_cap = cfg->log_cap;
    tc.rto_min = cfg->rto_min;
    tc.rto_max = cfg->rto_max;
    tc.commit_ahead = cfg->commit_ahead > 0 ? cfg->commit_ahead
                                            : std::max<int64_t>(2ll * cfg->chunk_bytes, 2ll * cfg->drr_quantum);
    tc.base_rtt_ns = cfg->base_rtt_ns;
    tc.seed = seed;
    tc.stream_index0 = 0;
    tc.chunk_pool = cfg->chunk_pool;
    tc.cc_algo = cfg->cc_algo;
    tc.drr_quantum = cfg->drr_quantum;
    tc.mss = cfg->mss;
    tc.cap_bytes = cfg->cap_bytes;
    tc.swift_target_ns = cfg->swift_target_ns;
    tc.init_cwnd_pkts = cfg->init_cwnd_pkts;
    tc.policy = cfg->policy;
    // receiver-driven mode (EQDS sender glue): credit and rts_ack records
    // arrive through cn_transport_handle_acks; RTS packets are logged as
    // transmissions with chunk 0xFFFFFFFF
    tc.receiver_driven = cfg->receiver_driven ? 1 : 0;
    tc.ordered = cfg->reliability == 1 ? 1 : 0;
    tc.credit_quantum = cfg->credit_quantum;
    tc.credit_bank_quanta = cfg->credit_bank_quanta;
    tc.initial_credit = cfg->receiver_driven ? cfg->initial_credit : 0;
    tc.engines = cfg->engines;
    tc.conn_split = cfg->conn_split;
    tc.cc_scope = cfg->cc_scope;
    tc.ecn_as_loss = cfg->ecn_as_loss;
    tc.cap_bytes = cfg->cap_bytes;
    int rc = cn_tx_create_empty(&tc, cfg->max_conns, cfg->max_conns_per_host, &h->tx);
    if (rc != CN_OK) {
        cn_transport_destroy(h);
        return rc;
    }
    cn_rx_config rcfg;
    cn_rx_config_default(&rcfg);
    rcfg.chunk_bytes = cfg->chunk_bytes;
    rcfg.carry_payload = cfg->carry_payload;
    rcfg.max_conns = std::max<uint32_t>(64, 2 * cfg->max_conns);
    rcfg.max_msgs = std::max<uint32_t>(256, 16 * cfg->max_conns);
    rcfg.chunk_pool = cfg->chunk_pool;
    rcfg.arena_bytes = cfg->carry_payload ? cfg->arena_bytes : 0;
    rcfg.max_batch = cfg->max_batch;
    rcfg.ordered = cfg->reliability == 1 ? 1 : 0;
    rc = cn_rx_create(&rcfg, &h->rx);
    if (rc != CN_OK) {
        cn_transport_destroy(h);
        return rc;
    }
    const uint64_t nc = cfg->max_conns, nb = cfg->max_batch + 16ull;
    bool ok = cudaMalloc(&h->d_log, nc * cfg->log_cap * sizeof(cn_tx_rec)) == cudaSuccess &&
              cudaMalloc(&h->d_stats, nc * sizeof(cn_tx_stats)) == cudaSuccess &&
              cudaMalloc(&h->d_aout, nb * sizeof(cn_ack_rec)) == cudaSuccess &&
              cudaMalloc(&h->d_cpls, nb * sizeof(cn_completion)) == cudaSuccess &&
              cudaMalloc(&h->d_res, sizeof(cn_rx_result)) == cudaSuccess;
    if (!ok) {
        set_error("cn_transport_create: out of device memory");
        cn_transport_destroy(h);
        return CN_E_CAPACITY;
    }
    cudaMemset(h->d_stats, 0, nc * sizeof(cn_tx_stats));
    h->txs.assign(nc, cn_tx_stats{});
    *out = h;
    return CN_OK;
}

// conn_to (transport.cpp:84-137): the connection opens on first use; its
// index (creation order) fixes its RngStream, its src its engine-sharing host
static int32_t open_conn(cn_transport* h, int32_t src, int32_t dst, bool create, int32_t n_paths = 0) {
    auto it = h->conn_idx.find({src, dst});
    if (it != h->conn_idx.end()) return it->second;
    if (!create) return -1;
    const int rc = cn_tx_open(h->tx, src, dst, n_paths > 0 ? n_paths : h->c.paths);
    if (rc < 0) return rc;
    h->conn_idx[{src, dst}] = rc;
    h->conn_src.push_back(src);
    const uint32_t nh = cn_tx_n_hosts(h->tx);
    if (h->pend.size() < nh) h->pend.resize(nh);
    return rc;
}

// conn_to with the topology's path count (min(paths, path_count(src, dst)),
// transport.cpp:97-99) supplied by the caller; send_message opens unknown
// pairs with `paths`
extern "C" int32_t cn_transport_open_conn(cn_transport* h, int32_t src, int32_t dst, int32_t n_paths) {
    if (!h || n_paths < 1 || n_paths > h->c.paths) {
        set_error("cn_transport_open_conn: n_paths outside [1, paths]");
        return CN_E_INVALID;
    }
    const int32_t k = open_conn(h, src, dst, false);
    if (k >= 0) return k;
    return open_conn(h, src, dst, true, n_paths);
}

extern "C" int32_t cn_transport_conn_index(cn_transport* h, int32_t src, int32_t dst) {
    return h ? open_conn(h, src, dst, false) : -1;
}

extern "C" int cn_transport_send_message(cn_transport* h, int32_t src, int32_t dst, uint64_t len, uint64_t tag,
                                         int64_t t) {
    if (!h) return CN_E_INVALID;
    if (len == 0) {
        set_error("send_message: empty message (transport.cpp:145)");
        return CN_E_INVALID;
    }
    const int32_t k = open_conn(h, src, dst, true);
    if (k < 0) return k;  // cn_tx_open set the message (capacity)
    h->subs.push_back(cn_tx_submit{t, len, tag});
    h->pend[cn_tx_conn_host(h->tx, k)].push_back(Ev{t, 0, static_cast<uint32_t>(k), h->subs.size() - 1});
    return 1;
}

extern "C" int cn_transport_handle_acks(cn_transport* h, const cn_ack_rec* acks, uint32_t n) {
    if (!h || (n && !acks)) return CN_E_INVALID;
    for (uint32_t i = 0; i < n; ++i) {
        // handle_ack / handle_nack look the connection up at the receiving host (:850-852)
        const int32_t k = open_conn(h, acks[i].dst, acks[i].src, false);
        if (k < 0) continue;
        h->acks.push_back(acks[i]);
        h->pend[cn_tx_conn_host(h->tx, k)].push_back(Ev{acks[i].aux, 1, static_cast<uint32_t>(k), h->acks.size() - 1});
    }
    return CN_OK;
}

extern "C" int cn_transport_advance(cn_transport* h, int64_t until, void* stream) {
    if (!h) return CN_E_INVALID;
    const uint32_t nh = cn_tx_n_hosts(h->tx);
    if (nh == 0) return CN_OK;
    // EventQueue::run_until(until): the queued inputs up to `until` run now,
    // later ones stay queued for the next advance
    std::vector<uint32_t> off(nh + 1, 0);
    std::vector<uint64_t> ev;
    std::vector<std::vector<Ev>> later(nh);
    for (uint32_t k = 0; k < nh; ++k) {
        auto& v = h->pend[k];
        std::stable_sort(v.begin(), v.end(), [](const Ev& a, const Ev& b) {
            return a.t != b.t ? a.t < b.t : a.type < b.type;
        });
        for (const Ev& e : v) {
            if (e.t > until) {
                later[k].push_back(e);
                continue;
            }
            ev.push_back((static_cast<uint64_t>(e.type) << 62) | (static_cast<uint64_t>(e.conn) << 40) | e.idx);
        }
        off[k + 1] = static_cast<uint32_t>(ev.size());
    }
    if (!grow(&h->d_ev, &h->cap_ev, ev.size() + 1) || !grow(&h->d_subs, &h->cap_subs, h->subs.size() + 1) ||
        !grow(&h->d_ain, &h->cap_ain, h->acks.size() + 1) || !grow(&h->d_evoff, &h->cap_evoff, nh + 1)) {
        set_error("cn_transport_advance: out of device memory");
        return CN_E_CAPACITY;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CNB_CUDA(cudaMemcpyAsync(h->d_evoff, off.data(), (nh + 1) * 4ull, cudaMemcpyHostToDevice, s));
    if (!ev.empty()) CNB_CUDA(cudaMemcpyAsync(h->d_ev, ev.data(), ev.size() * 8, cudaMemcpyHostToDevice, s));
    if (!h->subs.empty())
        CNB_CUDA(cudaMemcpyAsync(h->d_subs, h->subs.data(), h->subs.size() * sizeof(cn_tx_submit),
                                 cudaMemcpyHostToDevice, s));
    if (!h->acks.empty())
        CNB_CUDA(cudaMemcpyAsync(h->d_ain, h->acks.data(), h->acks.size() * sizeof(cn_ack_rec),
                                 cudaMemcpyHostToDevice, s));
    int rc = cn_tx_run(h->tx, h->d_evoff, h->d_ev, h->d_subs, h->d_ain, until, h->d_log, h->d_stats, stream);
    if (rc != CN_OK) return rc;
    const uint32_t nc = static_cast<uint32_t>(h->conn_src.size());
    CNB_CUDA(cudaMemcpyAsync(h->txs.data(), h->d_stats, nc * sizeof(cn_tx_stats), cudaMemcpyDeviceToHost, s));
    CNB_CUDA(cudaStreamSynchronize(s));
    unsigned int st = 0;
    cn_tx_status(h->tx, &st);
    // keep the later inputs (re-indexed into fresh submit / ack arrays)
    std::vector<cn_tx_submit> subs2;
    std::vector<cn_ack_rec> acks2;
    for (uint32_t k = 0; k < nh; ++k) {
        for (Ev& e : later[k]) {
            if (e.type == 0) {
                subs2.push_back(h->subs[e.idx]);
                e.idx = subs2.size() - 1;
            } else {
                acks2.push_back(h->acks[e.idx]);
                e.idx = acks2.size() - 1;
            }
        }
        h->pend[k].swap(later[k]);
    }
    h->subs.swap(subs2);
    h->acks.swap(acks2);
    if (st) {
        set_error("cn_transport_advance: sender status 0x" + std::to_string(st) +
                  ((st & CN_TX_STATUS_LOG) ? " (transmit log overflow: poll more often or raise log_cap)" : ""));
        return (st & CN_TX_STATUS_POLICY) ? CN_E_LOGIC : CN_E_CAPACITY;
    }
    return CN_OK;
}

// transmissions since the last poll: host by host, each host's in emission
// order.  Records that do not fit `cap` stay queued for the next poll.
extern "C" int64_t cn_transport_poll_transmissions(cn_transport* h, cn_tx_rec* out, uint64_t cap, int32_t* conn_out) {
    if (!h) return CN_E_INVALID;
    const uint32_t nh = cn_tx_n_hosts(h->tx);
    std::vector<uint32_t> cnt(nh), took(nh, 0);
    int rc = cn_tx_log_counts(h->tx, cnt.data());
    if (rc != CN_OK) return rc;
    uint64_t k = 0;
    for (uint32_t x = 0; x < nh; ++x) {
        const uint32_t m = std::min(cnt[x], h->c.log_cap);
        if (!m || !out || k >= cap) continue;
        const uint64_t take = std::min<uint64_t>(m, cap - k);
        CNB_CUDA(cudaMemcpy(out + k, h->d_log + static_cast<uint64_t>(x) * h->c.log_cap, take * sizeof(cn_tx_rec),
                            cudaMemcpyDeviceToHost));
        if (conn_out)
            for (uint64_t j = 0; j < take; ++j) conn_out[k + j] = static_cast<int32_t>(out[k + j].conn);
        took[x] = static_cast<uint32_t>(take);
        k += take;
    }
    if (!out) return static_cast<int64_t>(std::accumulate(cnt.begin(), cnt.end(), uint64_t{0}));
    rc = cn_tx_log_consume(h->tx, h->d_log, took.data());
    if (rc != CN_OK) return rc;
    return static_cast<int64_t>(k);
}

static int handle_data(cn_transport* h, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload,
                       uint64_t stride, const uint64_t* d_msg_data, uint32_t n, void* stream) {
    if (!h) return CN_E_INVALID;
    if (n > h->c.max_batch) {
        set_error("cn_transport_handle_data: batch larger than max_batch");
        return CN_E_CAPACITY;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = d_msg_data ? cn_rx_batch_msgdata(h->rx, d_hdrs, d_psn, d_msg_data, n, h->d_aout, n + 16, h->d_cpls,
                                              n + 16, h->d_res, stream)
             : d_psn    ? cn_rx_batch_psn(h->rx, d_hdrs, d_psn, d_payload, stride, n, h->d_aout, n + 16,
                                          h->d_cpls, n + 16, h->d_res, stream)
                        : cn_rx_batch(h->rx, d_hdrs, d_payload, stride, n, h->d_aout, n + 16, h->d_cpls, n + 16,
                                      h->d_res, stream);
    if (rc != CN_OK) return rc;
    cn_rx_result r;
    CNB_CUDA(cudaMemcpyAsync(&r, h->d_res, sizeof r, cudaMemcpyDeviceToHost, s));
    CNB_CUDA(cudaStreamSynchronize(s));
    if (r.status) {
        set_error("cn_transport_handle_data: receive status 0x" + std::to_string(r.status));
        return (r.status & (CN_RXF_UNSUPPORTED | CN_RXF_ALIAS)) ? CN_E_UNSUPPORTED : CN_E_CAPACITY;
    }
    h->last_acks.resize(r.n_acks);
    h->last_cpls.resize(r.n_completions);
    if (r.n_acks)
        CNB_CUDA(cudaMemcpy(h->last_acks.data(), h->d_aout, r.n_acks * sizeof(cn_ack_rec), cudaMemcpyDeviceToHost));
    if (r.n_completions)
        CNB_CUDA(cudaMemcpy(h->last_cpls.data(), h->d_cpls, r.n_completions * sizeof(cn_completion),
                            cudaMemcpyDeviceToHost));
    for (const cn_ack_rec& a : h->last_acks) {
        if (a.flags & CN_ACK_NACK) ++h->nacks_sent;
        else ++h->acks_sent;
    }
    h->delivered += r.n_completions;
    return CN_OK;
}

extern "C" int cn_transport_handle_data_psn(cn_transport* h, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                                            const void* d_payload, uint64_t stride, uint32_t n, void* stream) {
    return handle_data(h, d_hdrs, d_psn, d_payload, stride, nullptr, n, stream);
}
extern "C" int cn_transport_handle_data(cn_transport* h, const cn_pkt_hdr* d_hdrs, const void* d_payload,
                                        uint64_t stride, uint32_t n, void* stream) {
    return handle_data(h, d_hdrs, nullptr, d_payload, stride, nullptr, n, stream);
}
extern "C" int cn_transport_handle_data_msgdata(cn_transport* h, const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn,
                                                const uint64_t* d_msg_data, uint32_t n, void* stream) {
    if (h && n > 0 && !d_msg_data) {
        set_error("cn_transport_handle_data_msgdata: null msg_data");
        return CN_E_INVALID;
    }
    return handle_data(h, d_hdrs, d_psn, nullptr, 0, d_msg_data, n, stream);
}

extern "C" int64_t cn_transport_poll_acks(cn_transport* h, cn_ack_rec* out, uint64_t cap) {
    if (!h) return CN_E_INVALID;
    const uint64_t n = h->last_acks.size();
    if (out) memcpy(out, h->last_acks.data(), std::min(n, cap) * sizeof(cn_ack_rec));
    return static_cast<int64_t>(n);
}

extern "C" int64_t cn_transport_poll_completions(cn_transport* h, cn_completion* out, uint64_t cap) {
    if (!h) return CN_E_INVALID;
    const uint64_t n = h->last_cpls.size();
    if (out) memcpy(out, h->last_cpls.data(), std::min(n, cap) * sizeof(cn_completion));
    return static_cast<int64_t>(n);
}

extern "C" int cn_transport_stats(cn_transport* h, cn_stats* o) {
    if (!h || !o) return CN_E_INVALID;
    memset(o, 0, sizeof *o);
    for (const cn_tx_stats& t : h->txs) {
        o->msgs_sent += t.msgs_sent;
        o->msgs_completed += t.msgs_completed;
        o->backpressured += t.backpressured;
        o->chunks_sent += t.chunks_sent;
        o->chunk_rtx += t.chunk_rtx;
        o->fast_rtx += t.fast_rtx;
        o->rtos += t.rtos;
        o->rts_sent += t.rts_sent;
    }
    o->acks_sent = h->acks_sent;
    o->nacks_sent = h->nacks_sent;
    o->delivered_msgs = h->delivered;
    return CN_OK;
}

extern "C" int64_t cn_transport_outstanding_bytes(cn_transport* h, int32_t src, int32_t dst) {
    if (!h) return CN_E_INVALID;
    const int32_t k = open_conn(h, src, dst, false);
    return k < 0 ? 0 : h->txs[k].inflight;
}

// Transport::path_inflight / window_available / conn_credit / engine_*
// (transport.cpp:1173-1209), from the device state after the last advance
extern "C" int64_t cn_transport_path_inflight(cn_transport* h, int32_t src, int32_t dst, int32_t path) {
    if (!h) return 0;
    const int32_t k = open_conn(h, src, dst, false);
    if (k < 0 || path < 0 || path >= static_cast<int32_t>(h->c.paths)) return 0;
    cn_tx_conn_state cs;
    std::vector<int64_t> inf(h->c.paths, 0);
    if (cn_tx_get_conn_state(h->tx, static_cast<uint32_t>(k), &cs, inf.data(), h->c.paths) != CN_OK) return 0;
    return path < cs.n_paths ? inf[path] : 0;
}

extern "C" int64_t cn_transport_window_available(cn_transport* h, int32_t src, int32_t dst, int32_t path) {
    if (!h) return 0;
    const int32_t k = open_conn(h, src, dst, false);
    int64_t w = 0;
    if (k < 0 || cn_tx_window_available(h->tx, static_cast<uint32_t>(k), path, &w) != CN_OK) return 0;
    return w;
}

extern "C" int64_t cn_transport_conn_credit(cn_transport* h, int32_t src, int32_t dst) {
    if (!h) return 0;
    const int32_t k = open_conn(h, src, dst, false);
    cn_tx_conn_state cs;
    if (k < 0 || cn_tx_get_conn_state(h->tx, static_cast<uint32_t>(k), &cs, nullptr, 0) != CN_OK) return 0;
    return cs.credit;
}

// engine introspection: any connection of the host names its engines
static bool host_engine(cn_transport* h, int32_t host, int32_t engine, cn_tx_engine_state* es) {
    if (!h || engine < 0 || engine >= h->c.engines) return false;
    for (size_t c = 0; c < h->conn_src.size(); ++c)
        if (h->conn_src[c] == host)
            return cn_tx_get_engine_state(h->tx, static_cast<uint32_t>(c), engine, es) == CN_OK;
    return false;
}

extern "C" int32_t cn_transport_engine_inflight_msgs(cn_transport* h, int32_t host, int32_t engine) {
    cn_tx_engine_state es;
    return host_engine(h, host, engine, &es) ? es.inflight_msgs : 0;
}

extern "C" uint64_t cn_transport_engine_dispatched(cn_transport* h, int32_t host, int32_t engine) {
    cn_tx_engine_state es;
    return host_engine(h, host, engine, &es) ? es.dispatched : 0;
}

extern "C" int64_t cn_transport_engine_gauge(cn_transport* h, int32_t host, int32_t engine) {
    cn_tx_engine_state es;
    return host_engine(h, host, engine, &es) ? es.gauge : 0;
}
