set -x
LMC_LIB=varlib/chol/liblmc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_paths.py -m gpu -q -x -k "mals" > gpurun_out/s10_chol_tests.log 2>&1; tail -2 gpurun_out/s10_chol_tests.log
bash tools/ab_multi.sh c2 mals 2 base chol
bash tools/ab_multi.sh c4 mals 1 base chol
