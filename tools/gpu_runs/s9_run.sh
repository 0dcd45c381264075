set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/s9_tests.log 2>&1; tail -2 gpurun_out/s9_tests.log
timeout 900 python -m pytest tests/test_gpu_parity_paths.py -m gpu -q -x -k "count_target or variants" > gpurun_out/s9_tests2.log 2>&1; tail -2 gpurun_out/s9_tests2.log
bash tools/ab_multi.sh c4 adm 1 base tree
