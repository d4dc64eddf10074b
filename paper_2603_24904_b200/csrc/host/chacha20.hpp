// ChaCha20 keystream (RFC 8439 block function) as used by the reference's
// seeded RNG (proj/src/chacha20.cpp:48-96): key = BLAKE3(seed as u64 LE),
// nonce 0, block counter from 0, bytes consumed in order.
//
// The toy-model weights (proj/src/model.cpp:189-215) are the first W bytes of
// that stream that are not 0xFF, each mapped to b - 127. The reference draws
// them one byte at a time (83 s at 7B). Here the keystream is produced in
// independent 1 MiB segments on all cores, 0xFF bytes are counted per segment,
// an exclusive prefix sum gives every segment's output offset, and a second
// pass compacts -- the same bytes in the same order.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>

namespace dimg::chacha {

using Key = std::array<uint32_t, 8>;

void block(const Key& key, uint32_t counter, uint8_t out[64]);
Key key_from_seed(uint64_t seed);

// Sequential stream reader (prompts, small draws).
class Stream {
  public:
    explicit Stream(const Key& k) : key_(k) {}
    uint8_t u8();
    uint32_t u32();

  private:
    Key key_;
    uint32_t ctr_ = 0;
    uint8_t buf_[64];
    unsigned pos_ = 64;
};

struct Span {
    int8_t* dst;
    size_t len;
};

// Writes the accepted weight bytes (b != 0xFF -> b - 127) of the seed's
// stream, in order, into the concatenation of `spans` (the container's
// tensor payloads); threads <= 0 = all hardware threads.
void weight_stream(uint64_t seed, const Span* spans, size_t n_spans, int threads);
// The same stream generated on GPU `device` (engine.cu, kernels/chacha.cuh)
// and copied into the host spans.
void gpu_weight_stream(int device, uint64_t seed, const Span* spans, size_t n_spans);

}  // namespace dimg::chacha
