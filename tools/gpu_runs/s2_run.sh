set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/s2_parity.log 2>&1; tail -2 gpurun_out/s2_parity.log
bash tools/ab_multi.sh c4 adm 2 base tree
bash tools/ab_multi.sh c3 adm 1 base tree
