#!/bin/bash
# Build diagnostic variants of liblmc.so with ablation macros in complete.cu (timing insight only:
# the numerics of these builds are wrong by construction).  Usage: tools/abl_build.sh NAME -DMACRO ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=varlib/$name; mkdir -p $out
B=paper_2202_12567_b200/build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off \
  -I include -I paper_2202_12567_b200/csrc "$@" -c paper_2202_12567_b200/csrc/complete.cu -o $out/complete.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/liblmc.so $B/exact.o $out/complete.o $B/mals.o $B/lmc_api.o
echo $out/liblmc.so
