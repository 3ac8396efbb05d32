set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t5_kernels.log 2>&1
timeout 600 python tools/digest.py 4 > gpurun_out/digest5_new.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mqrcp_kernel --launch-skip 25 -c 1 -o gpurun_out/ncu5_mqrcp_glob python tools/ncu_cfg4.py numeric > gpurun_out/ncu5_q1.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mqrcp_kernel --launch-skip 9 -c 1 -o gpurun_out/ncu5_mqrcp_smem python tools/ncu_cfg4.py numeric > gpurun_out/ncu5_q2.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce" --csv --log-file gpurun_out/ncu_numeric4_m5.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m5.log 2>&1
