set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/h_gputests.log 2>&1; tail -3 gpurun_out/h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h_smoke.log 2>&1; tail -1 gpurun_out/h_smoke.log
timeout 600 python bench.py > gpurun_out/h_bench_c4.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/h_bench_c4.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
