set -x
python paper_2202_12567_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1; tail -3 gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1; tail -2 gpurun_out/r02_smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; tail -c 600 gpurun_out/r02_bench_c4.json
for c in c2 c3 c_mesh; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --solver mals --no-cpu-baseline > gpurun_out/r02_bench_c4_mals.json 2>/dev/null
timeout 600 python bench.py --config c2 --solver mals --no-cpu-baseline > gpurun_out/r02_bench_c2_mals.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/r02_reference_c4.json 2>/dev/null; cat gpurun_out/r02_reference_c4.json | tail -c 300
timeout 1200 python tools/sweep_c5.py 3 8 > gpurun_out/r02_c5_sweep.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_c4_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_adm" -c 1 -o gpurun_out/r02_k_adm_c4 python tools/one_frame.py c4 1 > gpurun_out/r02_ncu_adm.log 2>&1
ls -la gpurun_out | tail -20
