set -x
timeout 600 python bench.py > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err; tail -c 300 gpurun_out/g_bench_c4.json
for c in c2 c3 c_mesh; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/g_bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --solver mals --no-cpu-baseline > gpurun_out/g_bench_c4_mals.json 2>/dev/null
timeout 600 python bench.py --config c2 --solver mals --no-cpu-baseline > gpurun_out/g_bench_c2_mals.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/g_reference_c4.json 2>/dev/null
timeout 1200 python tools/sweep_c5.py 3 8 > gpurun_out/g_c5_sweep.json 2>/dev/null
