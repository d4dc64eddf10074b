import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (7B-shaped models)")


def has_gpu() -> bool:
    """Asks the CUDA driver directly, so a GPU box whose libdimg.so failed to
    build runs (and fails) the gpu tests instead of skipping them."""
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return False
    if cu.cuInit(0) != 0:
        return False
    n = ctypes.c_int(0)
    return cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_models():
    with open(os.path.join(GOLDEN, "models.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_7b():
    p = os.path.join(GOLDEN, "models_7b.json")
    if not os.path.exists(p):
        pytest.skip("models_7b.json not generated")
    with open(p) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ops_fixture():
    return dict(np.load(os.path.join(GOLDEN, "ops.npz")))


def ops_cases(fx, kind):
    n = int(fx[f"{kind}_n"])
    out = []
    for i in range(n):
        j = 0
        case = []
        while f"{kind}_{i}_{j}" in fx:
            case.append(fx[f"{kind}_{i}_{j}"])
            j += 1
        out.append(case)
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


def wild_arrays(cfg_tuple, seed, toy_scales, toy_norms):
    """Recreates tests/golden/make_golden.py's wild-model scales/gains."""
    rng = np.random.default_rng(seed)
    s = rng.integers(1, 1 << 22, size=toy_scales.shape, dtype=np.int64)
    n = rng.integers(-(1 << 21), 1 << 21, size=toy_norms.shape, dtype=np.int64)
    return s, n
