# round-2 final measurement set (one B200): GPU tests, smoke, bench lines, reference arm, C5 sweep,
# C4 launch list; outputs under gpurun_out/
set -x
python paper_2202_12567_b200/build.py > /dev/null
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.log 2>&1; tail -3 gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1; tail -2 gpurun_out/r02_smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; tail -c 400 gpurun_out/r02_bench_c4.json
for c in c2 c3 c_mesh; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --solver mals --no-cpu-baseline > gpurun_out/r02_bench_c4_mals.json 2>/dev/null
timeout 600 python bench.py --config c2 --solver mals --no-cpu-baseline > gpurun_out/r02_bench_c2_mals.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/r02_reference_c4.json 2>/dev/null; tail -c 300 gpurun_out/r02_reference_c4.json
timeout 1200 python tools/sweep_c5.py 3 8 > gpurun_out/r02_c5_sweep.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_c4_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -20
