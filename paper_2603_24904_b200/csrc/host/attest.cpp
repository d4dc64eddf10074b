// The attestation wire format (proj/src/attest.cpp:31-64): model id, input
// hash and output hash (32 bytes each) then bond and challenge period as
// little-endian u64 -- 112 bytes. Re-execution (make / verify / dispute)
// lives with the GPU engine in engine.cu.
#include <cstring>
#include <string>

#include "common.hpp"
#include "dimg.h"

namespace {

void put_u64(uint8_t* out, uint64_t v) {
    for (int i = 0; i < 8; ++i) out[i] = uint8_t(v >> (8 * i));
}

uint64_t get_u64(const uint8_t* in) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(in[i]) << (8 * i);
    return v;
}

std::string hex(const uint8_t* d) {
    static const char* k = "0123456789abcdef";
    std::string s(64, '0');
    for (int i = 0; i < 32; ++i) {
        s[2 * i] = k[d[i] >> 4];
        s[2 * i + 1] = k[d[i] & 15];
    }
    return s;
}

}  // namespace

using namespace dimg;

extern "C" {

dimg_status dimg_attestation_encode(const dimg_attestation* a, uint8_t out[112]) {
    DIMG_API_GUARD({
        std::memcpy(out, a->model_id, 32);
        std::memcpy(out + 32, a->input_hash, 32);
        std::memcpy(out + 64, a->output_hash, 32);
        put_u64(out + 96, a->bond);
        put_u64(out + 104, a->challenge_period);
    })
}

dimg_status dimg_attestation_decode(const uint8_t* bytes, size_t n, dimg_attestation* out) {
    DIMG_API_GUARD({
        if (n != 112) fail_parse(DIMG_PARSE_TRUNCATED, "attestation: expected 112 bytes");
        std::memcpy(out->model_id, bytes, 32);
        std::memcpy(out->input_hash, bytes + 32, 32);
        std::memcpy(out->output_hash, bytes + 64, 32);
        out->bond = get_u64(bytes + 96);
        out->challenge_period = get_u64(bytes + 104);
    })
}

dimg_status dimg_attestation_text(const dimg_attestation* a, char* buf, size_t cap, size_t* len) {
    // Attestation::to_text (proj/src/attest.cpp:54-62)
    DIMG_API_GUARD({
        const std::string s = "model_id=" + hex(a->model_id) + "\ninput_hash=" + hex(a->input_hash) +
                              "\noutput_hash=" + hex(a->output_hash) + "\nbond=" + std::to_string(a->bond) +
                              "\nchallenge_period=" + std::to_string(a->challenge_period) + "\n";
        if (len) *len = s.size();
        if (buf && cap) {
            const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    })
}

}  // extern "C"
