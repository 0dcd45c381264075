# round-2 final measurement set (session 2; one B200): outputs under gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
# k_adm C4 capture first, so the bench lines carry its DRAM bytes (profiles/r02_traffic.json)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adm -c 1 -o gpurun_out/f_k_adm_c4 python tools/one_frame.py c4 1 > gpurun_out/f_ncu_adm.log 2>&1
python tools/ncu_summary.py gpurun_out/f_k_adm_c4.ncu-rep > gpurun_out/f_k_adm_c4_ncu.txt 2>&1
python tools/traffic_update.py gpurun_out/f_k_adm_c4.ncu-rep c4/adm/q16 "k_adm<16>" profiles/r02_k_adm_c4_ncu.txt
cp profiles/r02_traffic.json gpurun_out/f_r02_traffic.json
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; tail -3 gpurun_out/f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -2 gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err; tail -c 300 gpurun_out/f_bench_c4.json
for c in c2 c3 c_mesh; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/f_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --solver mals --no-cpu-baseline > gpurun_out/f_bench_c4_mals.json 2>/dev/null
timeout 600 python bench.py --config c2 --solver mals --no-cpu-baseline > gpurun_out/f_bench_c2_mals.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/f_reference_c4.json 2>/dev/null; tail -c 300 gpurun_out/f_reference_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/f_c4_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sl_tile|k_sl_scatter|k_layout" -c 3 -o gpurun_out/f_slicing_c4 python tools/one_frame.py c4 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/f_slicing_c4.ncu-rep > gpurun_out/f_slicing_c4_ncu.txt 2>&1
timeout 1200 python tools/sweep_c5.py 3 8 > gpurun_out/f_c5_sweep.json 2>/dev/null
ls -la gpurun_out | tail -30
