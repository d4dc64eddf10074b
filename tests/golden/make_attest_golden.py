"""Writes tests/golden/attest.json by running the REFERENCE's attestation code
(proj/src/attest.cpp, compiled into oracle/_ref/libdimref.so with the shim's
ref_attestation / ref_verify) on the fixture of proj/tests/test_attest.cpp:
gen_toy_model(1001, {2 layers, d 16, 2 heads, ffn 32, vocab 32, ctx 64}),
prompt {4, 8, 15}, 10 new tokens, bond 1000, challenge period 100.

    python tests/golden/make_attest_golden.py      (needs /root/reference)
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Config, Reference  # noqa: E402

CFG = (2, 16, 2, 32, 32, 64)
PROMPT = [4, 8, 15]
MAX_NEW = 10


def main():
    ref = Reference()
    lib = ref.lib
    u8p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)
    lib.ref_attestation.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, u8p,
                                    C.c_char_p, C.c_size_t]
    lib.ref_verify.argtypes = [u8p, C.c_void_p, u32p, C.c_uint32, C.c_uint32, C.c_char_p, C.c_size_t]
    m = ref.gen_toy(1001, Config(*CFG))
    prompt = np.array(PROMPT, np.uint32)
    wire = (C.c_uint8 * 112)()
    text = C.create_string_buffer(1024)
    assert lib.ref_attestation(m.h, prompt.ctypes.data_as(u32p), 3, MAX_NEW, 1000, 100, wire, text, 1024) == 0
    honest = bytes(wire)

    def verify(w, p):
        out = C.create_string_buffer(1024)
        buf = (C.c_uint8 * 112)(*w)
        pp = np.array(p, np.uint32)
        assert lib.ref_verify(buf, m.h, pp.ctypes.data_as(u32p), len(p), MAX_NEW, out, 1024) == 0
        return out.value.decode()

    tampered = bytearray(honest)
    tampered[64 + 7] ^= 0x20                    # output hash byte 7 (test_attest.cpp:69-78)
    wrong_model = bytearray(honest)
    wrong_model[0] ^= 1                         # model id byte 0 (:122-135)
    gold = {"config": list(CFG), "seed": 1001, "prompt": PROMPT, "max_new": MAX_NEW, "bond": 1000,
            "challenge_period": 100, "wire": honest.hex(), "text": text.value.decode(),
            "verify": {"honest": verify(honest, PROMPT), "tampered_output": verify(bytes(tampered), PROMPT),
                       "wrong_model": verify(bytes(wrong_model), PROMPT),
                       "tampered_prompt": verify(honest, [4, 9, 15])}}
    with open(os.path.join(HERE, "attest.json"), "w") as f:
        json.dump(gold, f, indent=1)
    print(json.dumps(gold, indent=1))


if __name__ == "__main__":
    main()
