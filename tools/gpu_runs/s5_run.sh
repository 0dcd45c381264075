set -x
timeout 900 python -m pytest tests/test_gpu_slicing.py -m gpu -q -x > gpurun_out/s5_slicing.log 2>&1; tail -3 gpurun_out/s5_slicing.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches.csv python tools/one_frame.py c4 2 > /dev/null 2>&1
tail -1 gpurun_out/s5_launches.csv
