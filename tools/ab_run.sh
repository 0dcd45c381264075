#!/bin/bash
# A/B timing on the GPU box: varlib/base/liblmc.so (A) against the in-tree build (B), alternating.
# Usage: tools/ab_run.sh CONFIG SOLVER REPS   (writes gpurun_out/ab_<config>_<solver>_{A,B}_<i>.json)
cfg=$1; solver=$2; reps=${3:-2}
for i in $(seq 1 $reps); do
  LMC_LIB=varlib/base/liblmc.so python bench.py --config $cfg --solver $solver --no-cpu-baseline --no-e2e --steps 3 \
    > gpurun_out/ab_${cfg}_${solver}_A_$i.json 2>/dev/null
  python bench.py --config $cfg --solver $solver --no-cpu-baseline --no-e2e --steps 3 \
    > gpurun_out/ab_${cfg}_${solver}_B_$i.json 2>/dev/null
done
for f in gpurun_out/ab_${cfg}_${solver}_*.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],2), d['roofline']['kernel_ms'] if 'kernel_ms' in d['roofline'] else '', round(d['roofline']['frac'],4))"
done
