// abi.cu -- error plumbing, version, and the wire codec of the C ABI.
#include <cuda_runtime.h>
#include <stdio.h>

#include <string>

#include "common.cuh"

namespace cnb {
static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_status(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return CN_E_CUDA;
}
}  // namespace cnb

extern "C" const char* cn_last_error(void) { return cnb::g_last_error.c_str(); }

extern "C" const char* cn_version(void) {
    return "chunknet_b200 0.1 (sm_100a, CUDA " CNB_STR(__CUDACC_VER_MAJOR__) "." CNB_STR(__CUDACC_VER_MINOR__) ")";
}

// encode_header (src/wire.cpp:5-14)
extern "C" int cn_encode_header(const cn_control_header* h, uint32_t* out) {
    if (!h || !out) {
        cnb::set_error("cn_encode_header: null argument");
        return CN_E_INVALID;
    }
    if (h->msg_id > 127) {
        cnb::set_error("msg_id must fit 7 bits, got " + std::to_string(h->msg_id));
        return CN_E_FIELD_RANGE;
    }
    *out = cnb::enc_hdr(h->conn_id, h->msg_id, h->csn, h->last_chunk ? 1u : 0u, h->reserved);
    return CN_OK;
}

// decode_header (src/wire.cpp:16-24)
extern "C" void cn_decode_header(uint32_t w, cn_control_header* out) {
    if (!out) return;
    out->conn_id = static_cast<uint8_t>(w >> 24);
    out->msg_id = static_cast<uint8_t>((w >> 17) & 0x7f);
    out->csn = static_cast<uint8_t>((w >> 9) & 0xff);
    out->last_chunk = static_cast<uint8_t>((w >> 8) & 1u);
    out->reserved = static_cast<uint8_t>(w & 0xff);
}

// csn_before (src/wire.cpp:26-40) over SeqWindow (wire.hpp:47-66)
extern "C" int cn_csn_before(uint8_t a, uint8_t b, uint8_t base, int width, int* out) {
    if (width < 1 || width > 128) {
        cnb::set_error("SeqWindow width must be in [1,128], got " + std::to_string(width));
        return CN_E_FIELD_RANGE;
    }
    auto in_win = [&](uint8_t x) { return static_cast<uint8_t>(x - base) < width; };
    if (!in_win(a) || !in_win(b)) {
        uint8_t bad = in_win(a) ? b : a;
        cnb::set_error("csn " + std::to_string(bad) + " outside window base=" +
                       std::to_string(base) + " width=" + std::to_string(width));
        return CN_E_OUT_OF_WINDOW;
    }
    if (out) *out = static_cast<int8_t>(a - b) < 0 ? 1 : 0;
    return CN_OK;
}
