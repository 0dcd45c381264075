set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layout -c 1 -o gpurun_out/s6_layout python tools/one_frame.py c4 1 > gpurun_out/s6_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/s6_layout.ncu-rep > gpurun_out/s6_layout.txt 2>&1
head -60 gpurun_out/s6_layout.txt
