#!/bin/bash
# Like abl_build.sh, for macros of exact.cu (compiled with -fmad=false, as in build.py).
# Usage: tools/abl_build_exact.sh NAME -DMACRO ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=varlib/$name; mkdir -p $out
B=paper_2202_12567_b200/build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -fmad=false \
  -I include -I paper_2202_12567_b200/csrc "$@" -Xptxas -v -c paper_2202_12567_b200/csrc/exact.cu -o $out/exact.o 2> $out/ptxas.txt
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/liblmc.so $out/exact.o $B/complete.o $B/mals.o $B/lmc_api.o
echo $out/liblmc.so
