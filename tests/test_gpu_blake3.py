"""GPU BLAKE3 of model bytes (weight_hash / deserialize,
proj/src/model.cpp:310-316) against the reference's known answers and the
host implementation (itself pinned to the reference KATs in test_oracle.py /
test_host.py).

Lengths cover every boundary of the device tree: partial blocks and chunks,
the 256-chunk CTA fold (256 KiB), the second fold level (64 MiB), odd node
counts carried up at several levels, and unaligned device pointers (the
byte-wise load path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2603_24904_b200 as P
    return P


def _pattern(n):
    return (np.arange(n, dtype=np.int64) % 251).astype(np.uint8).tobytes()


def test_official_vectors(P, kat):
    assert P.blake3_gpu(b"").hex() == "af1349b9f5f9a1a6a0404dea36dcc9499bcb25c9adc112b7cc9a93cae41f3262"
    assert P.blake3_gpu(_pattern(1)).hex() == "2d3adedff11b61f14c886e35afa036736dcd87a74d27b5c1510225d0f592e213"
    assert P.blake3_gpu(_pattern(1024)).hex() == "42214739f095a406f3fc83deb889744ac00df831c10daa55189b5d121c855af7"
    assert P.blake3_gpu(_pattern(1025)).hex() == "d00278ae47eb27b34faecf67b4fe263f82d5412916c1ffd97c8cb7fb814b8444"
    for n, h in kat["blake3_pattern"].items():
        assert P.blake3_gpu(_pattern(int(n))).hex() == h, n


KIB = 1024
LENGTHS = [1, 63, 64, 65, 1023, 1024, 1025, 2047, 2048, 2049, 3071, 3072, 3073, 5000, 31744, 100000,
           256 * KIB - 1, 256 * KIB, 256 * KIB + 1, 3 * 256 * KIB + 5, 257 * 256 * KIB + 999,
           64 * KIB * KIB - KIB, 64 * KIB * KIB, 64 * KIB * KIB + 1, 129 * 256 * KIB * 3 + 17]


@pytest.mark.parametrize("n", LENGTHS)
def test_matches_host(P, n):
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert P.blake3_gpu(data).hex() == P.weight_hash(data), n


def test_device_pointer_and_unaligned(P):
    import torch
    rng = np.random.default_rng(7)
    host = rng.integers(0, 256, 3 * 256 * KIB + 777, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    torch.cuda.synchronize()
    for off in (0, 1, 3, 16):
        n = host.size - off - 5
        got, ms = P.blake3_device(dev.data_ptr() + off, n, timed=True)
        assert got.hex() == P.weight_hash(host[off:off + n].tobytes()), off
        assert ms > 0


def test_model_container_hash(P):
    """The weight hash of a model container (the bytes deserialize hashes)."""
    m = P.gen_toy_model(3, P.ModelConfig(2, 64, 2, 160, 100, 64))
    assert P.blake3_gpu(m.bytes).hex() == m.weight_hash
