set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_frames or c4_full or c2_full or edge" > gpurun_out/s7_tests.log 2>&1; tail -2 gpurun_out/s7_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_layout --csv --log-file gpurun_out/s7_layout.csv python tools/one_frame.py c4 2 > /dev/null 2>&1
grep k_layout gpurun_out/s7_layout.csv | awk -F'","' '{print $NF}'
