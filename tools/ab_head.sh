#!/bin/bash
# Build varlib/head/liblmc.so: the library with FILE (a csrc/*.cu unit) taken from git HEAD and the
# other units from the current build -- the A side of an A/B timing run (LMC_LIB=varlib/head/...).
# Usage: tools/ab_head.sh complete.cu [extra nvcc flags]
set -e
cd "$(dirname "$0")/.."
f=$1; shift
B=paper_2202_12567_b200/build
mkdir -p varlib/head
extra=""
[ "$f" = exact.cu ] && extra="-fmad=false"
git show HEAD:paper_2202_12567_b200/csrc/$f > paper_2202_12567_b200/csrc/_head_$f
trap 'rm -f paper_2202_12567_b200/csrc/_head_'$f EXIT
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off $extra \
  -I include -I paper_2202_12567_b200/csrc "$@" -c paper_2202_12567_b200/csrc/_head_$f -o varlib/head/${f%.cu}.o
objs=""
for u in exact complete mals lmc_api; do
  if [ "$u.cu" = "$f" ]; then objs="$objs varlib/head/$u.o"; else objs="$objs $B/$u.o"; fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o varlib/head/liblmc.so $objs
echo varlib/head/liblmc.so
