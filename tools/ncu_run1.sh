set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_apply4_metrics.csv python tools/ncu_cfg4.py apply > gpurun_out/ncu_a1.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"gemv_dev_kernel|spmv_csr_kernel" -c 8 -o gpurun_out/ncu_full_apply4 python tools/ncu_cfg4.py apply > gpurun_out/ncu_a2.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_numeric4_metrics.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_n1.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"mqrcp_kernel|ordered_reduce|qrcp_cluster" -c 6 -o gpurun_out/ncu_full_qr4 python tools/ncu_cfg4.py numeric > gpurun_out/ncu_n2.log 2>&1
ls -la gpurun_out
