// Exercises the C++ mirror of the reference API (csrc/include/dimg/dim.hpp).
//   api_test host   -- container, hashes, errors (no GPU)
//   api_test gpu    -- generate_greedy / InferenceSession on cuda:0 against
//                      goldens passed on the command line
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dimg/dim.hpp"

#define REQUIRE(c)                                                   \
    do {                                                             \
        if (!(c)) {                                                  \
            std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                \
        }                                                            \
    } while (0)

int host() {
    dimg::ModelConfig cfg{2, 16, 2, 32, 32, 64};
    auto m = dimg::gen_toy_model(7, cfg);
    auto b = m.bytes();
    auto m2 = dimg::deserialize(b);
    REQUIRE(m2.weight_hash() == m.weight_hash());
    std::vector<uint8_t> bad(b.begin(), b.end());
    bad[0] = 'X';
    try {
        dimg::deserialize(bad);
        REQUIRE(false);
    } catch (const dimg::ParseError& e) {
        REQUIRE(e.kind == dimg::ParseError::Kind::bad_magic);
    }
    uint32_t ids[] = {5, 9};
    REQUIRE(dimg::hash_token_ids(ids).hex().size() == 64);
    int64_t logits[] = {3, 7, 7, 1};
    REQUIRE(dimg::select_greedy(logits) == 1);
    dimg::ModelConfig bad_cfg{1, 6, 4, 8, 8, 16};
    try {
        bad_cfg.validate();
        REQUIRE(false);
    } catch (const std::invalid_argument&) {
    }
    // RTAB round trip and the reference's error kinds (proj/src/rope.cpp:41-93)
    auto t = dimg::build_rope_tables(10000.0, 8, 16);
    auto rb = dimg::serialize_rope_tables(t);
    REQUIRE(rb.size() == 24 + 2 * 16 * 4 * 8);
    REQUIRE(dimg::deserialize_rope_tables(rb) == t);
    rb.push_back(0);
    try {
        dimg::deserialize_rope_tables(rb);
        REQUIRE(false);
    } catch (const dimg::ParseError& e) {
        REQUIRE(e.kind == dimg::ParseError::Kind::invariant);
    }
    rb.resize(20);
    try {
        dimg::deserialize_rope_tables(rb);
        REQUIRE(false);
    } catch (const dimg::ParseError& e) {
        REQUIRE(e.kind == dimg::ParseError::Kind::truncated);
    }
    try {
        dimg::load_rope_tables("/nonexistent/dir/t.rtab");
        REQUIRE(false);
    } catch (const std::runtime_error&) {
    }
    std::printf("host ok %s\n", m.weight_hash().hex().c_str());
    return 0;
}

int gpu(const char* want_hash) {
    dimg::ModelConfig cfg{2, 16, 2, 32, 32, 64};
    auto m = dimg::gen_toy_model(7, cfg);
    uint32_t prompt[] = {3, 1, 4};
    auto r = dimg::generate_greedy(m, prompt, 12);
    REQUIRE(r.output_hash.hex() == want_hash);
    dimg::InferenceSession s(m);
    try {
        s.forward(99, 0);
        REQUIRE(false);
    } catch (const std::out_of_range&) {
    }
    try {
        s.forward(1, 5);
        REQUIRE(false);
    } catch (const std::logic_error&) {
    }
    try {
        dimg::generate_greedy(m, prompt, 1000);
        REQUIRE(false);
    } catch (const dimg::ContextOverflow&) {
    }
    std::printf("gpu ok %s\n", r.output_hash.hex().c_str());
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) return gpu(argc > 2 ? argv[2] : "");
    return host();
}
