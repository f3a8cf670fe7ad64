// chunknet_b200.hpp -- C++ host facade over the C ABI (include/chunknet_b200.h).
//
// Keeps the reference's C++ vocabulary (/root/reference/proj/include/chunknet):
// ControlHeader / encode_header / decode_header / SeqWindow / csn_before
// (wire.hpp), the exception types (FieldRangeError, OutOfWindowError,
// std::invalid_argument, std::logic_error), Transport's receive side with
// set_on_complete (transport.hpp:60-107), and PathScoreboard/select_path
// (lb.hpp) as a batched PathScheduler.  Status codes from the ABI are turned
// back into the reference's exceptions here, on the host, so a reference
// caller keeps its error handling.  Header-only; link libchunknet_b200.so
// and libcudart.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "chunknet_b200.h"

namespace chunknet {
namespace b200 {

class FieldRangeError : public std::invalid_argument {
  public:
    using std::invalid_argument::invalid_argument;
};
class OutOfWindowError : public std::invalid_argument {
  public:
    using std::invalid_argument::invalid_argument;
};
class CudaError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

inline void check(int status, const char* what) {
    if (status == CN_OK) return;
    std::string msg = std::string(what) + ": " + cn_last_error();
    switch (status) {
        case CN_E_FIELD_RANGE: throw FieldRangeError(msg);
        case CN_E_OUT_OF_WINDOW: throw OutOfWindowError(msg);
        case CN_E_INVALID: throw std::invalid_argument(msg);
        case CN_E_LOGIC:
        case CN_E_UNSUPPORTED: throw std::logic_error(msg);
        case CN_E_CUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

// ---------------------------------------------------------------- wire.hpp
struct ControlHeader {
    uint8_t conn_id = 0, msg_id = 0, csn = 0;
    bool last_chunk = false;
    uint8_t reserved = 0;
    bool operator==(const ControlHeader&) const = default;
};

inline uint32_t encode_header(const ControlHeader& h) {
    cn_control_header c{h.conn_id, h.msg_id, h.csn, static_cast<uint8_t>(h.last_chunk), h.reserved};
    uint32_t w = 0;
    check(cn_encode_header(&c, &w), "encode_header");
    return w;
}

inline ControlHeader decode_header(uint32_t w) {
    cn_control_header c;
    cn_decode_header(w, &c);
    return {c.conn_id, c.msg_id, c.csn, c.last_chunk != 0, c.reserved};
}

struct SeqWindow {
    uint8_t base_csn = 0;
    int width = 128;
};

inline bool csn_before(uint8_t a, uint8_t b, const SeqWindow& w) {
    int out = 0;
    check(cn_csn_before(a, b, w.base_csn, w.width, &out), "csn_before");
    return out != 0;
}

// ------------------------------------------------------------ device buffer
template <class T>
class DeviceArray {
  public:
    DeviceArray() = default;
    explicit DeviceArray(size_t n) { resize(n); }
    ~DeviceArray() { cudaFree(p_); }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    void resize(size_t n) {
        if (n <= n_) return;
        cudaFree(p_);
        p_ = nullptr;
        if (cudaMalloc(&p_, n * sizeof(T)) != cudaSuccess) throw CudaError("cudaMalloc");
        n_ = n;
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }

  private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// ------------------------------------------------- Transport (receive side)
// Batched Transport::handle_packet for data packets (transport.cpp:565-803):
// the device receive path, ack records in emission order, and the completion
// callback per delivered message (transport.hpp:77-79).
class RxTransport {
  public:
    struct Stats {  // receive-side subset of Transport::Stats (transport.hpp:62-75)
        uint64_t msgs_completed = 0, acks_sent = 0, pkts_accepted = 0, bytes_accepted = 0;
    };
    // (tag, src, dst, len, batch packet index, device pointer of the message)
    using CompleteFn = std::function<void(uint64_t, int, int, uint64_t, uint32_t, const void*)>;

    explicit RxTransport(const cn_rx_config& cfg) : cfg_(cfg) {
        check(cn_rx_create(&cfg_, &rx_), "cn_rx_create");
        if (cudaMalloc(&result_, sizeof(cn_rx_result)) != cudaSuccess) throw CudaError("cudaMalloc");
    }
    ~RxTransport() {
        cn_rx_destroy(rx_);
        cudaFree(result_);
    }
    RxTransport(const RxTransport&) = delete;
    RxTransport& operator=(const RxTransport&) = delete;

    void set_on_complete(CompleteFn fn) { on_complete_ = std::move(fn); }
    const Stats& stats() const { return stats_; }
    void reset(cudaStream_t s = nullptr) { check(cn_rx_reset(rx_, s), "cn_rx_reset"); }
    // pipelined receivers: the outstanding payload scatter joins `s`
    void flush(cudaStream_t s = nullptr) { check(cn_rx_flush(rx_, s), "cn_rx_flush"); }
    void post(uint64_t tag, void* d_buf, uint64_t len, cudaStream_t s = nullptr) {
        check(cn_rx_post(rx_, tag, d_buf, len, s), "cn_rx_post");
    }

    // Runs the batch and returns the acks it emitted (host copies).
    std::vector<cn_ack_rec> handle_packets(const cn_pkt_hdr* d_hdrs, const void* d_payload,
                                           uint64_t stride, uint32_t n, cudaStream_t s = nullptr) {
        acks_.resize(n + 16);
        cpls_.resize(n + 16);
        check(cn_rx_batch(rx_, d_hdrs, d_payload, stride, n, acks_.data(), n + 16, cpls_.data(),
                          n + 16, result_, s),
              "cn_rx_batch");
        cn_rx_result r;
        if (cudaMemcpyAsync(&r, result_, sizeof r, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            throw CudaError("result readback");
        if (r.status) throw std::logic_error("rx batch rejected, status flags " + std::to_string(r.status));
        std::vector<cn_ack_rec> out(r.n_acks);
        std::vector<cn_completion> cp(r.n_completions);
        if (r.n_acks) cudaMemcpy(out.data(), acks_.data(), r.n_acks * sizeof(cn_ack_rec), cudaMemcpyDeviceToHost);
        if (r.n_completions)
            cudaMemcpy(cp.data(), cpls_.data(), r.n_completions * sizeof(cn_completion),
                       cudaMemcpyDeviceToHost);
        stats_.acks_sent += r.n_acks;
        stats_.msgs_completed += r.n_completions;
        stats_.pkts_accepted += r.n_copied;
        stats_.bytes_accepted += r.bytes_copied;
        last_completions_ = cp;
        if (on_complete_)
            for (const auto& c : cp)
                on_complete_(c.tag, c.src, c.dst, c.len, c.pkt_index, reinterpret_cast<const void*>(c.reserved));
        return out;
    }
    const std::vector<cn_completion>& last_completions() const { return last_completions_; }

  private:
    cn_rx_config cfg_;
    cn_rx* rx_ = nullptr;
    cn_rx_result* result_ = nullptr;
    DeviceArray<cn_ack_rec> acks_;
    DeviceArray<cn_completion> cpls_;
    std::vector<cn_completion> last_completions_;
    CompleteFn on_complete_;
    Stats stats_;
};

// ------------------------------------------- PathScoreboard + select_path
enum class LbPolicy { oblivious = CN_LB_OBLIVIOUS, p2_rtt = CN_LB_P2_RTT, p2_ecn = CN_LB_P2_ECN };

class PathScheduler {
  public:
    PathScheduler(uint32_t n_conns, uint32_t max_paths, double base_rtt_ns, uint64_t seed,
                  const char* stream = "transport.conn", int64_t index0 = 0)
        : n_(n_conns) {
        check(cn_sched_create(n_conns, max_paths, nullptr, base_rtt_ns, seed, stream, index0, &s_),
              "cn_sched_create");
    }
    ~PathScheduler() { cn_sched_destroy(s_); }
    PathScheduler(const PathScheduler&) = delete;
    PathScheduler& operator=(const PathScheduler&) = delete;

    // next `count` decisions of every connection: d_out[conn * count + k]
    void select(LbPolicy p, uint32_t count, int32_t* d_out, cudaStream_t s = nullptr) {
        check(cn_sched_select(s_, static_cast<int>(p), 1, nullptr, nullptr, nullptr, n_, count, d_out, s),
              "cn_sched_select");
    }
    double* rtt_scores() {
        double* r = nullptr;
        cn_sched_boards(s_, &r, nullptr);
        return r;
    }

  private:
    cn_sched* s_ = nullptr;
    uint32_t n_;
};

// ------------------------------------------------- transport.hpp:53-107
// chunknet::Transport's shape over the device engines (cn_transport_*): the
// caller's clock replaces the event loop -- queue sends and the acks the
// fabric delivered, advance to a time, poll what the transport did.
class Endpoint {
  public:
    explicit Endpoint(const cn_transport_config& cfg, uint64_t seed) {
        check(cn_transport_create(&cfg, seed, &h_), "cn_transport_create");
    }
    ~Endpoint() { cn_transport_destroy(h_); }
    Endpoint(const Endpoint&) = delete;
    Endpoint& operator=(const Endpoint&) = delete;

    // Transport::send_message (transport.hpp:88) at time t; throws on an
    // empty message like the reference (std::invalid_argument)
    void send_message(int src, int dst, uint64_t len, uint64_t tag, int64_t t) {
        int rc = cn_transport_send_message(h_, src, dst, len, tag, t);
        if (rc < 0) check(rc, "send_message");
    }
    // acks and trimmed-header NACKs delivered at the senders (aux = time)
    void handle_acks(const std::vector<cn_ack_rec>& acks) {
        check(cn_transport_handle_acks(h_, acks.data(), static_cast<uint32_t>(acks.size())), "handle_acks");
    }
    void advance(int64_t until, cudaStream_t s = nullptr) { check(cn_transport_advance(h_, until, s), "advance"); }
    // every send_chunk since the last poll, with its connection index
    std::vector<std::pair<int32_t, cn_tx_rec>> poll_transmissions() {
        std::vector<cn_tx_rec> r(1 << 20);
        std::vector<int32_t> c(r.size());
        int64_t n = cn_transport_poll_transmissions(h_, r.data(), r.size(), c.data());
        if (n < 0) check(static_cast<int>(n), "poll_transmissions");
        std::vector<std::pair<int32_t, cn_tx_rec>> out;
        for (int64_t i = 0; i < n && i < static_cast<int64_t>(r.size()); ++i) out.push_back({c[i], r[i]});
        return out;
    }
    // Transport::handle_packet for a batch of delivered data packets (device records)
    void handle_data(const cn_pkt_hdr* d_hdrs, const void* d_payload, uint64_t stride, uint32_t n,
                     cudaStream_t s = nullptr) {
        check(cn_transport_handle_data(h_, d_hdrs, d_payload, stride, n, s), "handle_data");
    }
    std::vector<cn_ack_rec> poll_acks() {
        std::vector<cn_ack_rec> a(static_cast<size_t>(cn_transport_poll_acks(h_, nullptr, 0)));
        cn_transport_poll_acks(h_, a.data(), a.size());
        return a;
    }
    std::vector<cn_completion> poll_completions() {
        std::vector<cn_completion> c(static_cast<size_t>(cn_transport_poll_completions(h_, nullptr, 0)));
        cn_transport_poll_completions(h_, c.data(), c.size());
        return c;
    }
    cn_stats stats() const {
        cn_stats s;
        check(cn_transport_stats(h_, &s), "stats");
        return s;
    }
    int64_t outstanding_bytes(int src, int dst) const { return cn_transport_outstanding_bytes(h_, src, dst); }
    // the rest of Transport's introspection (transport.hpp:101-107)
    int64_t path_inflight(int src, int dst, int path) const { return cn_transport_path_inflight(h_, src, dst, path); }
    int64_t window_available(int src, int dst, int path) const {
        return cn_transport_window_available(h_, src, dst, path);
    }
    int64_t conn_credit(int src, int dst) const { return cn_transport_conn_credit(h_, src, dst); }
    int engine_inflight_msgs(int host, int engine) const { return cn_transport_engine_inflight_msgs(h_, host, engine); }
    uint64_t engine_dispatched(int host, int engine) const { return cn_transport_engine_dispatched(h_, host, engine); }
    int64_t engine_gauge(int host, int engine) const { return cn_transport_engine_gauge(h_, host, engine); }
    // ordered reliability: each packet's conn_psn beside its header
    void handle_data_psn(const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const void* d_payload, uint64_t stride,
                         uint32_t n, cudaStream_t s = nullptr) {
        check(cn_transport_handle_data_psn(h_, d_hdrs, d_psn, d_payload, stride, n, s), "handle_data_psn");
    }
    // send_message_data path: each packet names its message's device data (Packet::msg_data)
    void handle_data_msgdata(const cn_pkt_hdr* d_hdrs, const uint64_t* d_psn, const uint64_t* d_msg_data,
                             uint32_t n, cudaStream_t s = nullptr) {
        check(cn_transport_handle_data_msgdata(h_, d_hdrs, d_psn, d_msg_data, n, s), "handle_data_msgdata");
    }

  private:
    cn_transport* h_ = nullptr;
};

}  // namespace b200
}  // namespace chunknet
