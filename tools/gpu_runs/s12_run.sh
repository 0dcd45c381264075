set -x
for v in rcp1 rcp0; do LMC_LIB=varlib/$v/liblmc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_paths.py -m gpu -q -x -k "mals" > gpurun_out/s12_${v}_tests.log 2>&1; tail -2 gpurun_out/s12_${v}_tests.log; done
bash tools/ab_multi.sh c2 mals 2 base rcp1 rcp0
