set -x
LMC_LIB=varlib/lay2/liblmc.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_frames or c2_full or edge" > gpurun_out/s14_tests.log 2>&1; tail -2 gpurun_out/s14_tests.log
for i in 1 2; do for v in base lay2; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_layout --csv --log-file gpurun_out/s14_${v}_${i}.csv env LMC_LIB=varlib/$v/liblmc.so python tools/one_frame.py c4 2 > /dev/null 2>&1; echo $v; grep k_layout gpurun_out/s14_${v}_${i}.csv | awk -F'","' '{print $NF}'; done; done
