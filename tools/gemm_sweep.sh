#!/bin/bash
# GEMM shape sweep of the 7B decode-batch / prefill products (tools/gemm_bench.cu).
B=${GEMM_BENCH:-tools/_libs/gemm_bench}
for ks in 1 2 3; do $B 12288 4096 8 16 $ks 0; done
for ks in 1 2 4 8; do $B 4096 4096 8 16 $ks 1; done
for ks in 1 2 4 8; do $B 4096 4096 8 16 $ks 1 1; done
$B 22016 4096 8 16 1 0
$B 22016 4096 8 16 1 0 1
for ks in 1 2 4 8; do $B 4096 11008 8 16 $ks 1; done
$B 32000 4096 8 16 1 0
for ks in 1 2 4; do $B 4096 4096 64 64 $ks 1; done
$B 12288 4096 64 64 1 0
$B 22016 4096 64 64 1 0
$B 22016 4096 64 16 1 0
$B 12288 4096 64 16 1 0
$B 4096 4096 64 16 2 1
$B 22016 4096 2048 64 1 0
$B 4096 11008 2048 64 1 1
