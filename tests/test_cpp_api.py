"""The C++ mirror of the reference API (csrc/include/dimg/dim.hpp), compiled
and run against libdimg.so."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PKG = os.path.join(ROOT, "paper_2603_24904_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "api_test")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(PKG, "csrc", "include"), os.path.join(ROOT, "tests", "cpp", "api_test.cpp"),
                    "-L", PKG, "-ldimg", f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_cpp_api_host(binary):
    r = subprocess.run([binary, "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("host ok")


@pytest.mark.gpu
def test_cpp_api_gpu(binary, golden_models):
    want = golden_models["small_s7"]["output_hash"]
    r = subprocess.run([binary, "gpu", want], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
