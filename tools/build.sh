#!/bin/bash
# Builds libdimg.so and reports errors / the persistent kernel's resources.
cd "$(dirname "$0")/.." || exit 1
if ! make -s -C paper_2603_24904_b200/csrc -j8 > /tmp/build.log 2>&1; then
  grep -E "error" /tmp/build.log | head -20; echo BUILD FAILED; exit 1
fi
grep -A3 "decode_persistent" paper_2603_24904_b200/csrc/build/ptxas.log | grep -E "registers|spill" | head -2
ls -la --time-style=+%T paper_2603_24904_b200/libdimg.so
