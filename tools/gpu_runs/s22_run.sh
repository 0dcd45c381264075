set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_paths.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/s22_tests.log 2>&1; tail -2 gpurun_out/s22_tests.log
bash tools/ab_multi.sh c4 adm 2 colold tree
