// Tensor-parallel glue. A decode step on rank r of g:
//
//   QKV GEMV (this rank's heads) -> attention (its heads, its KV cache)
//   -> WO GEMV over its head columns, EPI_RAW: the PRE-SCALE int64
//      accumulators acc_r[i] = sum_{j in r's columns} w[i,j] x[j]
//   -> sum over ranks -> x = clamp(x + (sum acc_r * s) >> 16)       (tp_resid_kernel)
//   -> GATE/UP GEMV (its FFN rows, silu*up) -> DOWN GEMV over its FFN columns,
//      EPI_RAW -> sum over ranks -> residual                          (tp_resid_kernel)
//   ... lm_head over its vocab rows -> local argmax (tp_argmax_kernel)
//   -> every rank's (max, lowest index) pair -> the same pick on every rank
//      (tp_pick_kernel): tokens[pos + 1], pos + 1.
//
// Exactness: dense_forward (proj/src/kernels.cpp:18-30) sums w*x in int64
// (wrapping) BEFORE the (acc * s) >> 16 rescale; integer addition mod 2^64 is
// associative, so summing the ranks' partial accumulators (in any order: a
// uint64 all-reduce or the kernel below) gives the reference's acc bit for
// bit -- the same argument as the reference's chunk invariance
// (proj/src/kernels.cpp:32-50, proj/tests/test_kernels.cpp:79-97). The
// rescale, residual and clamp then run redundantly on every rank. The
// argmax order (max, lowest index) is total, so the pick is rank-independent
// (select_greedy, proj/src/engine.cpp:113-120).
#pragma once

#include <cstdint>

#include "gemv.cuh"
#include "q16.cuh"

namespace dimg::dev {

// x[i] = clamp(x[i] + ((sum_p parts[p][i]) * s[i]) >> 16): the residual after
// a row-parallel projection. n_parts = 1 after an NCCL all-reduce (the sum is
// already in parts[0]); = g on one device (the local backend), where each
// rank's raw GEMV wrote its own slot of a [g][n] buffer.
__global__ void tp_resid_kernel(int64_t* __restrict__ x, const int64_t* __restrict__ parts, uint32_t n_parts,
                                uint32_t part_stride, const int64_t* __restrict__ s, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t acc = 0;
        for (uint32_t p = 0; p < n_parts; ++p) acc += uint64_t(parts[size_t(p) * part_stride + i]);
        x[i] = add_clamp(x[i], scale_row(int64_t(acc), s[i]));
    }
}

// One rank's lm_head slice: (max logit, lowest global index) -> best[0..1];
// the row is also copied to the kept-logits slot (pos - logit_base) when it
// is < keep_cap (EngineOptions::keep_logits). One CTA of TP_ARG_THREADS.
constexpr int TP_ARG_THREADS = 1024;
__global__ void __launch_bounds__(TP_ARG_THREADS)
    tp_argmax_kernel(const int64_t* __restrict__ row, uint32_t n, uint32_t v0, const Ctl* ctl,
                     int64_t* __restrict__ keep, uint32_t keep_stride, unsigned long long* best) {
    const uint32_t slot = ctl->pos - ctl->logit_base;
    const bool kept = keep && slot < ctl->keep_cap;
    int64_t bv = INT64_MIN;
    uint32_t bi = 0xFFFFFFFFu;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t v = row[i];
        if (kept) keep[size_t(slot) * keep_stride + i] = v;
        if (better(v, v0 + i, bv, bi)) {
            bv = v;
            bi = v0 + i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ov, oi, bv, bi)) {
            bv = ov;
            bi = oi;
        }
    }
    __shared__ int64_t sv[32];
    __shared__ uint32_t si[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < TP_ARG_THREADS / 32; ++w)
            if (better(sv[w], si[w], bv, bi)) {
                bv = sv[w];
                bi = si[w];
            }
        best[0] = (unsigned long long)bv;
        best[1] = bi;
    }
}

// The greedy pick over the g ranks' pairs (gathered [g][2]); identical on
// every rank. Appends the token and advances the position.
__global__ void tp_pick_kernel(const unsigned long long* __restrict__ pairs, uint32_t g, uint32_t* tokens, Ctl* ctl) {
    int64_t bv = INT64_MIN;
    uint32_t bi = 0xFFFFFFFFu;
    for (uint32_t r = 0; r < g; ++r) {
        const int64_t v = int64_t(pairs[2 * r]);
        const uint32_t i = uint32_t(pairs[2 * r + 1]);
        if (better(v, i, bv, bi)) {
            bv = v;
            bi = i;
        }
    }
    const uint32_t pos = ctl->pos;
    tokens[pos + 1] = bi;
    ctl->pos = pos + 1;
}

}  // namespace dimg::dev
