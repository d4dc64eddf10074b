"""C5 B=8 / B=64 timing of library builds (DIMG_LIB=...), each in its own
process, alternated over two rounds.

    python tools/batch_libs.py LIB_A LIB_B ...
"""
import os
import subprocess
import sys

from batch_ab import CHILD  # noqa: E402

for rnd in range(2):
    for lib in sys.argv[1:]:
        o = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, DIMG_LIB=os.path.abspath(lib)),
                           capture_output=True, text=True)
        print(f"{lib}: " + (" | ".join(o.stdout.strip().splitlines()) or o.stderr[-800:]), flush=True)
