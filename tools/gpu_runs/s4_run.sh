set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/s4_tests.log 2>&1; tail -3 gpurun_out/s4_tests.log
bash tools/ab_multi.sh c4 adm 1 base tree
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sl_ --csv --log-file gpurun_out/s4_sl_launches.csv python tools/one_frame.py c4 1 > /dev/null 2>&1
tail -3 gpurun_out/s4_sl_launches.csv
