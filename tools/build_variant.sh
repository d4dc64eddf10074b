#!/bin/bash
# Experiment builds of libdimg: tools/build_variant.sh NAME -DFLAG ...
#   -> tools/_libs/libdimg_NAME.so (load with DIMG_LIB=...; never the product)
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2603_24904_b200/csrc -j8 > /dev/null
name=$1; shift
mkdir -p tools/_libs
C=paper_2603_24904_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -Iinclude -I$C "$@" \
  -c $C/engine.cu -o tools/_libs/engine_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_libs/libdimg_$name.so \
  $(ls $C/build/*.o | grep -v engine.cu.o) tools/_libs/engine_$name.o -Xcompiler -pthread
echo tools/_libs/libdimg_$name.so
