bash tools/ab_multi.sh c2 mals 1 base nosolve
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mals -c 1 -o gpurun_out/s11_mals_c2 python tools/one_frame.py c2 1 solver=1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/s11_mals_c2.ncu-rep > gpurun_out/s11_mals_c2.txt 2>&1
NCU_K=k_mals python tools/ncu_lines.py gpurun_out/s11_mals_c2.ncu-rep > gpurun_out/s11_mals_lines.txt 2>&1
