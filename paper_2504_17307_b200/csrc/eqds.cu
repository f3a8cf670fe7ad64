// eqds.cu -- the EQDS receiver-driven pull pacer on the device (sm_100a).
//
// Restates EqdsReceiver (/root/reference/proj/src/eqds.cpp:7-104,
// include/chunknet/eqds.hpp) -- one per receiving host: per-sender demand /
// granted / rtx_owed, three epoch-stamped FIFO service lists (retransmit
// owed, demand, idle top-up), one credit quantum granted per tick, ticks
// spaced by the time one quantum takes at line rate.  Every receiving host
// is independent, so the device runs one thread per
// receiver over that receiver's time-ordered input stream (RTS, chunk
// arrivals, trimmed headers) and fires its own ticks in between, in the
// DES's (time, seq) order: inputs were queued first, so they precede a tick
// due at the same instant.  Outputs are the grants and RTS acknowledgements
// in callback order.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>

#include "common.cuh"

namespace cnb {

enum : uint8_t { EL_NONE = 0, EL_RTX = 1, EL_ACTIVE = 2, EL_IDLE = 3 };

struct EqSender {
    int64_t demand, granted, rtx_owed;
    uint32_t epoch;
    uint8_t list;
    uint8_t pad[3];
};

struct EqRecv {
    int64_t tick_at, next_grant_t;
    uint64_t grants_sent;
    uint32_t n_senders, ticking, head[3], tail[3], log_n, status;
};

struct EqDev {
    uint32_t n_recv, max_senders, key_mask, qcap, log_cap, quantum, grant_to_idle, pad;
    int64_t tick_ns, bank_cap;
    EqRecv* recv;
    int32_t* keys;        // [n_recv][key_mask+1] sender id or -1
    uint32_t* slot_of;    // [n_recv][key_mask+1]
    EqSender* senders;    // [n_recv][max_senders]
    int32_t* sender_id;   // [n_recv][max_senders]
    uint64_t* queues;     // [n_recv][3][qcap] (slot << 32) | epoch
};

struct Pacer {
    const EqDev& d;
    EqRecv& R;
    int32_t* keys;
    uint32_t* slot;
    EqSender* S;
    int32_t* ids;
    uint64_t* q;
    cn_eqds_log* log;

    __device__ uint32_t find(int32_t id) {  // std::map operator[] (default-constructs)
        uint32_t h = (static_cast<uint32_t>(id) * 2654435761u) & d.key_mask;
        for (;;) {
            const int32_t k = keys[h];
            if (k == id) return slot[h];
            if (k == -1) {
                if (R.n_senders >= d.max_senders) {
                    R.status |= 1u;
                    return 0;
                }
                const uint32_t s = R.n_senders++;
                keys[h] = id;
                slot[h] = s;
                ids[s] = id;
                memset(&S[s], 0, sizeof(EqSender));
                return s;
            }
            h = (h + 1) & d.key_mask;
        }
    }
    __device__ void push(int l, uint32_t s) {
        uint64_t* Q = q + static_cast<uint64_t>(l) * d.qcap;
        if (R.tail[l] - R.head[l] >= d.qcap) {
            R.status |= 2u;  // service list overflow
            return;
        }
        Q[R.tail[l] % d.qcap] = (static_cast<uint64_t>(s) << 32) | S[s].epoch;
        ++R.tail[l];
    }
    __device__ void reclassify(uint32_t s) {  // eqds.cpp:7-26
        EqSender& x = S[s];
        uint8_t want;
        if (x.rtx_owed > 0) want = EL_RTX;
        else if (x.demand > x.granted) want = EL_ACTIVE;
        else if (d.grant_to_idle && x.granted < d.bank_cap) want = EL_IDLE;
        else want = EL_NONE;
        if (want == x.list) return;
        x.list = want;
        ++x.epoch;
        if (want != EL_NONE) push(want - 1, s);
    }
    __device__ void ensure_ticking(int64_t now) {  // eqds.cpp:28-34
        if (R.ticking) return;
        if (R.head[0] == R.tail[0] && R.head[1] == R.tail[1] && R.head[2] == R.tail[2]) return;
        R.ticking = 1;
        R.tick_at = now > R.next_grant_t ? now : R.next_grant_t;
    }
    __device__ int64_t pop_valid(int l, uint8_t want) {  // eqds.cpp:36-46
        uint64_t* Q = q + static_cast<uint64_t>(l) * d.qcap;
        while (R.head[l] != R.tail[l]) {
            const uint64_t e = Q[R.head[l] % d.qcap];
            ++R.head[l];
            const uint32_t s = static_cast<uint32_t>(e >> 32);
            if (S[s].list == want && S[s].epoch == static_cast<uint32_t>(e)) return s;
        }
        return -1;
    }
    __device__ void emit(int64_t t, int32_t sender, uint32_t bytes, int32_t kind) {
        if (R.log_n < d.log_cap) {
            cn_eqds_log r;
            r.t = t;
            r.sender = sender;
            r.bytes = bytes;
            r.kind = kind;
            r.pad = 0;
            log[R.log_n] = r;
        } else {
            R.status |= 4u;
        }
        ++R.log_n;
    }
    __device__ void tick() {  // eqds.cpp:48-68
        const int64_t now = R.tick_at;
        R.ticking = 0;
        int64_t s = pop_valid(0, EL_RTX);
        if (s < 0) s = pop_valid(1, EL_ACTIVE);
        if (s < 0) s = pop_valid(2, EL_IDLE);
        if (s < 0) return;
        EqSender& x = S[s];
        x.granted += d.quantum;
        if (x.rtx_owed > 0) {
            const int64_t v = x.rtx_owed - static_cast<int64_t>(d.quantum);
            x.rtx_owed = v > 0 ? v : 0;
        }
        ++R.grants_sent;
        R.next_grant_t = now + d.tick_ns;
        emit(now, ids[s], d.quantum, 0);
        x.list = EL_NONE;
        reclassify(static_cast<uint32_t>(s));
        ensure_ticking(now);
    }
    __device__ void on_rts(int64_t now, int32_t id, uint64_t demand, bool rtx) {  // eqds.cpp:70-85
        const uint32_t s = find(id);
        EqSender& x = S[s];
        x.granted = 0;
        x.demand = static_cast<int64_t>(demand);
        if (rtx && x.rtx_owed < static_cast<int64_t>(d.quantum)) x.rtx_owed = d.quantum;
        emit(now, id, 0, 1);
        reclassify(s);
        ensure_ticking(now);
    }
    __device__ void on_chunk(int64_t now, int32_t id, uint32_t bytes, bool was_rtx) {  // eqds.cpp:87-94
        const uint32_t s = find(id);
        EqSender& x = S[s];
        int64_t v = x.demand - static_cast<int64_t>(bytes);
        x.demand = v > 0 ? v : 0;
        v = x.granted - static_cast<int64_t>(bytes);
        x.granted = v > 0 ? v : 0;
        if (was_rtx) {
            v = x.rtx_owed - static_cast<int64_t>(bytes);
            x.rtx_owed = v > 0 ? v : 0;
        }
        reclassify(s);
        ensure_ticking(now);
    }
    __device__ void on_trim(int64_t now, int32_t id, uint32_t len) {  // eqds.cpp:96-105
        const uint32_t s = find(id);
        EqSender& x = S[s];
        const int64_t v = x.granted - static_cast<int64_t>(len);
        x.granted = v > 0 ? v : 0;
        x.rtx_owed += len;
        reclassify(s);
        ensure_ticking(now);
    }
};

__global__ void k_eqds_run(EqDev d, const uint32_t* __restrict__ ev_off, const cn_eqds_event* __restrict__ ev,
                           int64_t end_time, cn_eqds_log* __restrict__ log, uint32_t* __restrict__ log_n) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= d.n_recv) return;
    const uint64_t kb = static_cast<uint64_t>(r) * (d.key_mask + 1);
    const uint64_t sb = static_cast<uint64_t>(r) * d.max_senders;
    Pacer P{d,
            d.recv[r],
            d.keys + kb,
            d.slot_of + kb,
            d.senders + sb,
            d.sender_id + sb,
            d.queues + static_cast<uint64_t>(r) * 3 * d.qcap,
            log + static_cast<uint64_t>(r) * d.log_cap};
    P.R.log_n = 0;
    for (uint32_t k = ev_off[r]; k < ev_off[r + 1]; ++k) {
        const cn_eqds_event e = ev[k];
        while (P.R.ticking && P.R.tick_at < e.t) P.tick();
        if (e.type == CN_EQ_RTS) P.on_rts(e.t, e.sender, e.arg, e.flag != 0);
        else if (e.type == CN_EQ_CHUNK) P.on_chunk(e.t, e.sender, static_cast<uint32_t>(e.arg), e.flag != 0);
        else P.on_trim(e.t, e.sender, static_cast<uint32_t>(e.arg));
    }
    while (P.R.ticking && P.R.tick_at <= end_time) P.tick();
    log_n[r] = P.R.log_n;
}

__global__ void k_eqds_init(EqDev d) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t nk = static_cast<uint64_t>(d.n_recv) * (d.key_mask + 1);
    for (uint64_t x = i; x < nk; x += static_cast<uint64_t>(gridDim.x) * blockDim.x) d.keys[x] = -1;
    for (uint64_t x = i; x < d.n_recv; x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        memset(&d.recv[x], 0, sizeof(EqRecv));
}

}  // namespace cnb

using namespace cnb;

struct cn_eqds {
    EqDev d;
    int tpb = 128;  // threads (receivers) per block
};

extern "C" void cn_eqds_config_default(cn_eqds_config* c) {
    memset(c, 0, sizeof *c);
    c->quantum = 32768;  // EqdsParams::quantum / TransportConfig::credit_quantum
    c->grant_to_idle = 1;
    c->max_senders = 1024;
    c->queue_cap = 1 << 14;
    c->log_cap = 1 << 16;
}

extern "C" int cn_eqds_create(const cn_eqds_config* cfg, uint32_t n_receivers, cn_eqds** out) {
    if (!cfg || !out || !n_receivers || !cfg->quantum || !cfg->max_senders || !cfg->queue_cap || cfg->tick_ns < 0) {
        set_error("cn_eqds_create: bad config");
        return CN_E_INVALID;
    }
    *out = nullptr;
    cn_eqds* h = new (std::nothrow) cn_eqds();
    if (!h) return CN_E_CAPACITY;
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        while (h->tpb > 32 && (n_receivers + h->tpb - 1) / h->tpb < static_cast<uint32_t>(sms)) h->tpb /= 2;
    }
    EqDev& d = h->d;
    d.n_recv = n_receivers;
    d.max_senders = cfg->max_senders;
    uint32_t km = 1;
    while (km < 2 * cfg->max_senders) km <<= 1;
    d.key_mask = km - 1;
    d.qcap = cfg->queue_cap;
    d.log_cap = cfg->log_cap;
    d.quantum = cfg->quantum;
    d.grant_to_idle = cfg->grant_to_idle ? 1 : 0;
    d.tick_ns = cfg->tick_ns;
    d.bank_cap = cfg->bank_cap;
    const uint64_t nr = n_receivers;
    bool ok = cudaMalloc(&d.recv, nr * sizeof(EqRecv)) == cudaSuccess &&
              cudaMalloc(&d.keys, nr * km * 4) == cudaSuccess &&
              cudaMalloc(&d.slot_of, nr * km * 4) == cudaSuccess &&
              cudaMalloc(&d.senders, nr * d.max_senders * sizeof(EqSender)) == cudaSuccess &&
              cudaMalloc(&d.sender_id, nr * d.max_senders * 4) == cudaSuccess &&
              cudaMalloc(&d.queues, nr * 3 * static_cast<uint64_t>(d.qcap) * 8) == cudaSuccess;
    if (!ok) {
        set_error("cn_eqds_create: out of device memory");
        cn_eqds_destroy(h);
        return CN_E_CAPACITY;
    }
    k_eqds_init<<<1024, 256>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cn_eqds_destroy(h);
        return cuda_status(e, "cn_eqds_create");
    }
    *out = h;
    return CN_OK;
}

extern "C" void cn_eqds_destroy(cn_eqds* h) {
    if (!h) return;
    cudaDeviceSynchronize();
    void* p[] = {h->d.recv, h->d.keys, h->d.slot_of, h->d.senders, h->d.sender_id, h->d.queues};
    for (void* x : p)
        if (x) cudaFree(x);
    delete h;
}

extern "C" int cn_eqds_run(cn_eqds* h, const uint32_t* d_ev_off, const cn_eqds_event* d_events, int64_t end_time,
                           cn_eqds_log* d_log, uint32_t* d_log_n, void* stream) {
    if (!h || !d_ev_off || !d_log || !d_log_n) {
        set_error("cn_eqds_run: bad arguments");
        return CN_E_INVALID;
    }
    // one thread per receiver, each a sequential event loop: spread the
    // receivers over every SM before stacking warps on one
    k_eqds_run<<<(h->d.n_recv + h->tpb - 1) / h->tpb, h->tpb, 0, static_cast<cudaStream_t>(stream)>>>(
        h->d, d_ev_off, d_events, end_time, d_log, d_log_n);
    CNB_CUDA(cudaGetLastError());
    return CN_OK;
}

extern "C" int cn_eqds_status(cn_eqds* h, uint32_t receiver, uint32_t* status, uint64_t* grants_sent) {
    if (!h || receiver >= h->d.n_recv) return CN_E_INVALID;
    EqRecv r;
    CNB_CUDA(cudaMemcpy(&r, h->d.recv + receiver, sizeof r, cudaMemcpyDeviceToHost));
    if (status) *status = r.status;
    if (grants_sent) *grants_sent = r.grants_sent;
    return CN_OK;
}
