// Host model container: the canonical DIM1 bytes plus views into them
// (proj/include/dim/model.hpp:50-60 keeps the same pair: tensors + `bytes`).
// Layout of DIM1 (proj/README.md "File formats", proj/src/model.cpp:217-249):
//   "DIM1" u32 version=1, u32 n_layers d_model n_heads d_ffn vocab max_ctx,
//   f64 rope_theta, u32 tensor count, directory (u16 name len, name, u32 rows,
//   u32 cols, u8 kind), then payloads in directory order: kind 0 = rows x i64
//   scale then rows*cols i8; kind 1 = cols x i64.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace dimg {

void validate_config(const dimg_config& c);  // proj/src/model.cpp:95-109

struct HostModel {
    dimg_config cfg{};
    std::vector<uint8_t> bytes;          // canonical DIM1 container
    // quantised tensors in directory order: tok_embd, 7 per layer, output
    std::vector<size_t> q_rows, q_cols, q_scale_off, q_data_off;  // offsets into bytes
    std::vector<size_t> norm_off;        // dense tensors (2L+1), offsets into bytes
    std::vector<int64_t> scales;         // aligned copy of every scale, directory order
    std::vector<int64_t> norms;          // aligned copy of every norm gain
    std::vector<dimg_qtensor> layer_desc;

    dimg_model_desc desc() const;
};

// device >= 0: the weight stream synthesised on that GPU (same bytes)
HostModel gen_toy_model(uint64_t seed, const dimg_config& cfg, int threads, int device = -1);
HostModel deserialize(const uint8_t* bytes, size_t n);
HostModel serialize_desc(const dimg_model_desc& d);

// Tables built on the host with the reference's FP64 expressions, then
// uploaded; the device never evaluates a transcendental.
void build_rope(double theta, uint32_t d_head, uint32_t max_ctx, int64_t* cos_out, int64_t* sin_out);
int64_t exp_lut_entry(int i);
int64_t invsqrt_seed(int b);
int64_t q16_from_ratio(int64_t num, int64_t den);

}  // namespace dimg
