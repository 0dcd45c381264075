#!/bin/bash
# Build a variant of liblmc.so with build macros in complete2.cu (A/B timing of the q <= 16 ADM).
# Usage: tools/abl2_build.sh NAME -DMACRO=... ; then LMC_LIB=varlib/NAME/liblmc.so python ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=varlib/$name; mkdir -p $out
B=paper_2202_12567_b200/build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off \
  -I include -I paper_2202_12567_b200/csrc -Xptxas -v "$@" -c paper_2202_12567_b200/csrc/complete2.cu -o $out/complete2.o 2> $out/ptxas.txt
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/liblmc.so $B/exact.o $B/complete.o $out/complete2.o $B/mals.o $B/lighttree.o $B/lmc_api.o -L/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib
grep -A2 "k_adm2ILi8ELb0" $out/ptxas.txt | grep -E "spill|Used" | tr '\n' ' '; echo
echo $out/liblmc.so
