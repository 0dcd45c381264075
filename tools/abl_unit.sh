#!/bin/bash
# Build a variant of liblmc.so with one translation unit recompiled under extra macros (A/B timing).
# Usage: tools/abl_unit.sh NAME UNIT.cu -DMACRO=... ; then LMC_LIB=varlib/NAME/liblmc.so python ...
set -e
cd "$(dirname "$0")/.."
name=$1; unit=$2; shift 2
out=varlib/$name; mkdir -p $out
B=paper_2202_12567_b200/build
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib
extra=""; case $unit in exact.cu|lighttree.cu) extra="-fmad=false";; esac
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off $extra \
  -I include -I paper_2202_12567_b200/csrc -Xptxas -v "$@" -c paper_2202_12567_b200/csrc/$unit -o $out/${unit%.cu}.o 2> $out/ptxas.txt
objs=""
for u in exact complete complete2 mals lighttree lmc_api; do
  if [ "$u.cu" = "$unit" ]; then objs="$objs $out/$u.o"; else objs="$objs $B/$u.o"; fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/liblmc.so $objs -L$NCCL -l:libnccl.so.2 -Xlinker -rpath -Xlinker $NCCL
echo $out/liblmc.so
