set -x
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/s23_tests.log 2>&1; tail -3 gpurun_out/s23_tests.log
ALL_RANKS=1 PARTITION=1 timeout 1200 python tools/rank_times.py c4 3 2 4 8 > gpurun_out/rank_times_inter.json 2> gpurun_out/rank_times_inter.err; tail -3 gpurun_out/rank_times_inter.err
