"""Writes tests/golden/rtab.json from the REFERENCE's RTAB codec
(serialize_rope_tables / deserialize_rope_tables, proj/src/rope.cpp:41-93,
compiled into oracle/_ref/libdimref.so, shims ref_rtab_serialize /
ref_rtab_parse):

  tables   reference-serialized artifacts of build_rope_tables(theta, dh, ctx)
           (hex; small shapes) plus the BLAKE3 of a 7B-shaped one
  parse    mutated byte strings (bad magic, bad version, truncations at
           every header field and inside the payload, empty dimensions,
           trailing bytes) with the reference's outcome: 0 or the
           ParseError kind (0 bad_magic, 1 bad_version, 2 truncated,
           3 invariant)

    python tests/golden/make_rtab_golden.py      (needs /root/reference)
"""
import ctypes as C
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Reference  # noqa: E402


def main():
    ref = Reference()
    lib = ref.lib
    lib.ref_rtab_serialize.argtypes = [C.c_double, C.c_uint32, C.c_uint32, C.c_void_p, C.c_size_t,
                                       C.POINTER(C.c_size_t)]
    lib.ref_rtab_parse.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_int)]

    def ser(theta, dh, ctx):
        n = C.c_size_t()
        assert lib.ref_rtab_serialize(theta, dh, ctx, None, 0, C.byref(n)) == 0
        buf = (C.c_uint8 * n.value)()
        assert lib.ref_rtab_serialize(theta, dh, ctx, buf, n.value, C.byref(n)) == 0
        return bytes(buf)

    def parse(b):
        k = C.c_int()
        rc = lib.ref_rtab_parse(b, len(b), C.byref(k))
        return 0 if rc == 0 else (100 + k.value if rc == 7 else rc)

    tables = []
    for theta, dh, ctx in ((10000.0, 8, 16), (10000.0, 2, 8), (500000.0, 64, 24), (10000.0, 128, 5)):
        tables.append({"theta": theta, "d_head": dh, "max_ctx": ctx, "hex": ser(theta, dh, ctx).hex()})
    big = ser(10000.0, 128, 4096)
    base = ser(10000.0, 8, 16)
    cases = [base, b"XTAB" + base[4:], base[:4] + struct.pack("<I", 2) + base[8:], base + b"\0",
             base[:-1], base[:3], base[:6], base[:10], base[:14], base[:20], base[:24], base[:100],
             base[:8] + struct.pack("<I", 0) + base[12:], base[:12] + struct.pack("<I", 0) + base[16:],
             base[:8] + struct.pack("<I", 17) + base[12:], b"", b"RTAB"]
    parse_cases = [{"hex": c.hex(), "outcome": parse(c)} for c in cases]
    out = {"tables": tables, "big": {"theta": 10000.0, "d_head": 128, "max_ctx": 4096, "size": len(big),
                                     "blake3": ref.blake3(big)}, "parse": parse_cases}
    with open(os.path.join(HERE, "rtab.json"), "w") as f:
        json.dump(out, f, indent=1)
    print([p["outcome"] for p in parse_cases])


if __name__ == "__main__":
    main()
