#!/bin/bash
# Time several library builds on one box, interleaved: tools/ab_multi.sh CONFIG SOLVER REPS lib1 lib2 ...
# ("tree" = the in-tree build).  Prints ms/frame, kernel ms and roofline fraction per run.
cfg=$1; solver=$2; reps=$3; shift 3
for i in $(seq 1 $reps); do
  for v in "$@"; do
    if [ "$v" = tree ]; then lib=""; else lib=varlib/$v/liblmc.so; fi
    LMC_LIB=$lib python bench.py --config $cfg --solver $solver --no-cpu-baseline --no-e2e --steps 3 \
      > gpurun_out/abm_${cfg}_${v}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/abm_${cfg}_${v}_$i.json').read().strip().splitlines()[-1]); print('$v', $i, round(d['ms_per_step'],2), round(d['roofline'].get('kernel_ms',0),2), {k: round(x,2) for k,x in d['ms_per_stage'].items()})"
  done
done
