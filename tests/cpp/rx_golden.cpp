// C++ host facade on the device: replay a recorded reference trace through
// chunknet::b200::RxTransport and compare the ack stream with the
// reference's (golden fixture exported by tests/test_cpp.py).
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
    if (argc < 5) { std::fprintf(stderr, "usage: rx_golden data.bin staging.bin acks.bin chunk_bytes\n"); return 2; }
    auto hdrs = load<cn_pkt_hdr>(argv[1]);
    auto staging = load<uint8_t>(argv[2]);
    auto want = load<cn_ack_rec>(argv[3]);
    cn_rx_config cfg;
    cn_rx_config_default(&cfg);
    cfg.chunk_bytes = static_cast<uint32_t>(std::atoi(argv[4]));
    cfg.arena_bytes = 64 << 20;
    cfg.chunk_pool = 1 << 18;
    cfg.max_batch = static_cast<uint32_t>(hdrs.size());
    RxTransport tr(cfg);
    int done = 0;
    tr.set_on_complete([&](uint64_t, int, int, uint64_t, uint32_t, const void* d) { done += d != nullptr; });
    DeviceArray<cn_pkt_hdr> dh(hdrs.size());
    DeviceArray<uint8_t> ds(staging.size());
    cudaMemcpy(dh.data(), hdrs.data(), hdrs.size() * sizeof(cn_pkt_hdr), cudaMemcpyHostToDevice);
    cudaMemcpy(ds.data(), staging.data(), staging.size(), cudaMemcpyHostToDevice);
    auto acks = tr.handle_packets(dh.data(), ds.data(), CN_MAX_PAYLOAD, static_cast<uint32_t>(hdrs.size()));
    if (acks.size() != want.size()) { std::fprintf(stderr, "acks %zu != %zu\n", acks.size(), want.size()); return 1; }
    for (size_t i = 0; i < acks.size(); ++i) {
        acks[i].aux = want[i].aux = 0;
        acks[i].reserved = want[i].reserved = 0;
        if (std::memcmp(&acks[i], &want[i], sizeof(cn_ack_rec)) != 0) { std::fprintf(stderr, "ack %zu differs\n", i); return 1; }
    }
    std::printf("CPP_RX_OK acks=%zu completions=%d\n", acks.size(), done);
    return 0;
}
