set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_coarsen|k_pass1|k_eval_new|k_pass2" -c 4 -o gpurun_out/s8_stages python tools/one_frame.py c4 1 > gpurun_out/s8_ncu.log 2>&1
for k in k_coarsen k_pass1 k_eval_new k_pass2; do echo "== $k"; NCU_K=$k python tools/ncu_lines.py gpurun_out/s8_stages.ncu-rep 2>&1 | head -25; done > gpurun_out/s8_lines.txt
python tools/ncu_summary.py gpurun_out/s8_stages.ncu-rep > gpurun_out/s8_summary.txt 2>&1
