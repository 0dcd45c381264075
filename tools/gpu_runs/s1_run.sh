set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s1_gputests.log 2>&1; tail -3 gpurun_out/s1_gputests.log
timeout 600 python bench.py > gpurun_out/s1_bench_c4.json 2> gpurun_out/s1_bench_c4.err; tail -c 600 gpurun_out/s1_bench_c4.json
