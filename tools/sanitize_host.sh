#!/bin/bash
# AddressSanitizer + UBSan on the host code: the oracle (all oracle pins) and liblmc's
# host runtime (lmc_api.cu: validation, BVH build, partition planning, and -- with a GPU -- whole
# small frames).  compute-sanitizer is not available on this pool; these cover the host side.
set -u
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/sanitize_host.log}
ASAN=$(gcc -print-file-name=libasan.so); UBSAN=$(gcc -print-file-name=libubsan.so)
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib
B=paper_2202_12567_b200/build
T=$(mktemp -d)
python paper_2202_12567_b200/build.py > /dev/null
gcc -O1 -g -fsanitize=address,undefined -fno-omit-frame-pointer -ffp-contract=off -fopenmp -fPIC -shared -I oracle \
  -o $T/liboracle.so oracle/oracle.c -lm
nvcc -O1 -g -std=c++17 -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC,-ffp-contract=off,-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer \
  -I include -I paper_2202_12567_b200/csrc -c paper_2202_12567_b200/csrc/lmc_api.cu -o $T/lmc_api.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fsanitize=address,-fsanitize=undefined -o $T/liblmc.so \
  $B/exact.o $B/complete.o $B/complete2.o $B/mals.o $B/lighttree.o $T/lmc_api.o -L$NCCL -l:libnccl.so.2 \
  -Xlinker -rpath -Xlinker $NCCL
export LD_PRELOAD="$ASAN $UBSAN" ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0 UBSAN_OPTIONS=print_stacktrace=1
{
  echo "== oracle pins under ASan/UBSan"
  ORACLE_LIB=$T/liboracle.so python -m pytest -q -p no:cacheprovider tests/test_oracle_*.py 2>&1 | tail -2
  echo "== liblmc host code under ASan/UBSan (CPU tests)"
  LMC_LIB=$T/liblmc.so python -m pytest -q -p no:cacheprovider tests/test_bvh_host.py tests/test_abi.py \
    tests/test_dist_cpu.py -k "plan or bvh or abi or exports or struct or status" 2>&1 | tail -2
  if python -c "import torch, sys; sys.exit(0 if torch.cuda.is_available() else 1)" 2>/dev/null; then
    echo "== liblmc host code under ASan/UBSan (GPU frames)"
    for c in c1 t_interior t_mesh "c1 1 solver=1" "t_interior 2 warm_start=1 row_importance=1 resolve_mode=1"; do
      LMC_LIB=$T/liblmc.so python tools/one_frame.py $c 2>&1 | tail -1
    done
  fi
} > $out 2>&1
echo "sanitizer reports: $(grep -c 'runtime error\|ERROR: AddressSanitizer' $out)" >> $out
cat $out
