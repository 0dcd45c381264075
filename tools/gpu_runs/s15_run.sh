set -x
LMC_LIB=varlib/tma/liblmc.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_frames or c4_full or edge or c2_full" > gpurun_out/s15_tests.log 2>&1; tail -2 gpurun_out/s15_tests.log
bash tools/ab_multi.sh c4 adm 2 base tma
LMC_LIB=varlib/tma/liblmc.so timeout 600 ncu --set full --clock-control none -k regex:k_adm -c 1 -o gpurun_out/s15_tma python tools/one_frame.py c4 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/s15_tma.ncu-rep | head -40 > gpurun_out/s15_tma.txt
