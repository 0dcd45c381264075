set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_paths.py tests/test_gpu_fuzz.py -m gpu -q -x -k "mals or MALS or fuzz" > gpurun_out/s13_tests.log 2>&1; tail -2 gpurun_out/s13_tests.log
bash tools/ab_multi.sh c2 mals 2 base tree quadr1
bash tools/ab_multi.sh c4 mals 1 base tree
