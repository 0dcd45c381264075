set -x
for i in 1 2; do for v in base co2 co4; do LMC_LIB=varlib/$v/liblmc.so python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/s16_${v}_$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/s16_${v}_$i.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_stage']['coarsen'],3), round(d['ms_per_step'],2))"; done; done
