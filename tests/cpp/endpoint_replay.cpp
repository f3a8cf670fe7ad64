// C++ boundary object on the device: chunknet::b200::Endpoint driven like
// chunknet::Transport -- send_message + the acks the reference DES delivered
// at the sender, advance, poll -- must reproduce the reference sender's
// transmit log (golden fixture exported by tests/test_cpp.py).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "chunknet_b200.hpp"

using namespace chunknet::b200;

template <class T>
static std::vector<T> load(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) { std::perror(path); std::exit(2); }
    std::fseek(f, 0, SEEK_END);
    long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::vector<T> v(n / sizeof(T));
    if (n && std::fread(v.data(), 1, n, f) != static_cast<size_t>(n)) std::exit(2);
    std::fclose(f);
    return v;
}

int main(int argc, char** argv) {
    if (argc < 14) return 2;
    auto subs = load<cn_tx_submit>(argv[1]);
    auto acks = load<cn_ack_rec>(argv[2]);
    struct Want {  // the reference harness's record (oracle/ref_harness.cpp cnref_tx_rec)
        int64_t t;
        uint32_t msg_id, chunk;
        int32_t path, is_rtx;
        uint64_t msg_seq;
    };
    auto want = load<Want>(argv[3]);
    cn_transport_config c;
    cn_transport_config_default(&c);
    c.chunk_bytes = std::atoi(argv[4]);
    c.paths = std::atoi(argv[5]);
    c.lb = std::atoi(argv[6]);
    c.rto_min = std::atoll(argv[7]);
    c.rto_max = std::atoll(argv[8]);
    c.commit_ahead = std::atoll(argv[9]);
    c.base_rtt_ns = std::atof(argv[10]);
    c.max_conns = 2;
    c.chunk_pool = 1 << 18;
    c.log_cap = 1 << 17;
    const int src = std::atoi(argv[12]), dst = std::atoi(argv[13]);
    Endpoint ep(c, std::strtoull(argv[11], nullptr, 10));
    for (const auto& s : subs) ep.send_message(src, dst, s.len, s.tag, s.t);
    ep.handle_acks(acks);
    ep.advance(60000000000ll);
    auto tx = ep.poll_transmissions();
    if (tx.size() != want.size()) { std::fprintf(stderr, "tx %zu != %zu\n", tx.size(), want.size()); return 1; }
    for (size_t i = 0; i < tx.size(); ++i)
        if (tx[i].second.t != want[i].t || tx[i].second.msg_id != want[i].msg_id ||
            tx[i].second.chunk != want[i].chunk || tx[i].second.path != want[i].path ||
            tx[i].second.is_rtx != want[i].is_rtx || tx[i].second.msg_seq != want[i].msg_seq || tx[i].first != 0 ||
            tx[i].second.dst != dst) {
            std::fprintf(stderr, "tx %zu differs\n", i);
            return 1;
        }
    cn_stats st = ep.stats();
    std::printf("CPP_ENDPOINT_OK tx=%zu rtx=%llu\n", tx.size(), static_cast<unsigned long long>(st.chunk_rtx));
    try {
        ep.send_message(src, dst, 0, 1, 0);
        return 1;
    } catch (const std::invalid_argument&) {  // send_message throws on an empty message (transport.cpp:145)
    }
    return 0;
}
