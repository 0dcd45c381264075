#!/bin/bash
# Build a variant of liblmc.so with one compilation unit rebuilt under extra flags and linked with
# the in-tree objects (A/B timing and diagnostic builds; run paper_2202_12567_b200/build.py first).
# Usage: tools/variant_build.sh NAME UNIT.cu -DMACRO=... ;  then LMC_LIB=varlib/NAME/liblmc.so ...
set -e
cd "$(dirname "$0")/.."
name=$1; unit=$2; shift 2
B=paper_2202_12567_b200/build
out=varlib/$name; mkdir -p $out
fmad=""
case $unit in exact.cu|lighttree.cu|slice.cu) fmad="-fmad=false";; esac
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off $fmad \
  -I include -I paper_2202_12567_b200/csrc "$@" -c paper_2202_12567_b200/csrc/$unit -o $out/${unit%.cu}.o
objs=""
for u in exact complete complete2 mals lighttree slice lmc_api; do
  if [ "$u.cu" = "$unit" ]; then objs="$objs $out/$u.o"; else objs="$objs $B/$u.o"; fi
done
NL=$(python -c "import sys; sys.path.insert(0,'paper_2202_12567_b200'); import build; print(' '.join(build._nccl_link()))")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/liblmc.so $objs $NL
echo $out/liblmc.so
