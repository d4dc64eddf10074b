"""Per-source-line stall samples of the persistent decode kernel.

    python tools/ncu_lines.py REPORT.ncu-rep [LIB.so] [--from L0 --to L1] [--top N]

Maps each SASS address in ncu's source page to the (file, line) the
-lineinfo debug info of the same libdimg.so assigns it (nvdisasm -g), then
sums the warp-stall samples per line -- ncu's own CUDA-source view does not
resolve lines for this multi-header build. `--from/--to` restricts to a line
range of persistent.cuh (e.g. one function) and prints that range's total.
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

KERNEL = "_ZN4dimg3dev24decode_persistent_kernelENS0_6PkArgsE"  # --kernel overrides (mangled name)


def sass_lines(lib, kernel=KERNEL):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "engine.sm_100a.cubin", os.path.abspath(lib)], cwd=d,
                       check=True, capture_output=True)
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, "engine.sm_100a.cubin")], check=True,
                             capture_output=True, text=True).stdout
    m = {}
    inside = False
    cur = ("?", 0)
    for ln in out.splitlines():
        if ln.startswith(".text."):
            inside = ln.startswith(".text." + kernel + ":")
            continue
        if not inside:
            continue
        g = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (os.path.basename(g.group(1)), int(g.group(2)))
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("lib", nargs="?", default="paper_2603_24904_b200/libdimg.so")
    ap.add_argument("--from", dest="lo", type=int, default=0)
    ap.add_argument("--to", dest="hi", type=int, default=10 ** 9)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel", default=KERNEL, help="mangled kernel name (nvdisasm section)")
    ap.add_argument("--file", default="persistent.cuh", help="source file the line range refers to")
    ap.add_argument("--select", default=None, help="ncu -k filter (regex) when the report holds several kernels")
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"]
    if a.select:
        cmd += ["-k", "regex:" + a.select, "-c", "1"]
    txt = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if rows and rows[0] and rows[0][0] == "Kernel Name":  # a multi-kernel report: its first section
        end = next((i for i in range(1, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
        rows = rows[:end]
    hdr = rows[1]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][ia], 16)
    m = sass_lines(a.lib, a.kernel)
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    per = collections.Counter()
    why = collections.Counter()
    total = 0
    for r in data:
        s = int(r[iss] or 0)
        total += s
        f, line = m.get(int(r[ia], 16) - base, ("?", 0))
        if f == a.file and not (a.lo <= line <= a.hi):
            continue
        if f != a.file and (a.lo > 0 or a.hi < 10 ** 9):
            continue
        per[(f, line)] += s
        for i in reasons:
            why[hdr[i]] += int(r[i] or 0)
    sel = sum(per.values())
    print(f"samples: kernel {total}, selected {sel} ({100.0 * sel / max(1, total):.1f}%)")
    tw = sum(why.values())
    print("stall reasons:", ", ".join(f"{k[6:]} {100.0 * v / max(1, tw):.1f}%" for k, v in why.most_common(8)))
    for (f, line), s in per.most_common(a.top):
        print(f"{s:8d} {100.0 * s / max(1, total):5.1f}%  {f}:{line}")


if __name__ == "__main__":
    main()
