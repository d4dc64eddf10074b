// BLAKE3 (plain hash mode, 32-byte output) for the host side of the engine:
// output hash of token ids (proj/src/engine.cpp:104-111), weight hash of the
// DIM1 container (proj/src/model.cpp:310) and the ChaCha20 seed key
// (proj/src/chacha20.cpp:57-62).
//
// The reference hashes with one thread, block by block. Here the input is cut
// into aligned 1 MiB subtrees whose chaining values are computed in parallel
// and folded into the same binary tree the spec defines, so a 6.75 GB
// container hashes in seconds instead of minutes. Bit-identical output.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace dimg::b3 {

using Digest = std::array<uint8_t, 32>;

// One-shot hash; threads <= 0 uses all hardware threads.
Digest hash(const void* data, size_t len, int threads = 0);

// Incremental hasher for small streams (token ids).
class Hasher {
  public:
    Hasher();
    void update(const void* data, size_t len);
    Digest finalize() const;

  private:
    std::vector<uint8_t> buf_;
};

}  // namespace dimg::b3
