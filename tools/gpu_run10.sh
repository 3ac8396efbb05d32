set -x
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mqrcp_kernel --launch-skip 9 -c 1 -o gpurun_out/ncu10_mqrcp_smem python tools/ncu_cfg4.py numeric > gpurun_out/ncu10_q2.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:qrcp_cluster --launch-skip 20 -c 2 -o gpurun_out/ncu10_cluster python tools/ncu_cfg4.py numeric > gpurun_out/ncu10_q3.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"qrcp_kernel" --launch-skip 40 -c 2 -o gpurun_out/ncu10_qrcp1 python tools/ncu_cfg4.py numeric > gpurun_out/ncu10_q4.log 2>&1
