set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s3_gputests.log 2>&1; tail -5 gpurun_out/s3_gputests.log
bash tools/ab_multi.sh c4 adm 2 base tree
bash tools/ab_multi.sh c2 adm 1 base tree
