set -x
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"gemv_dev_kernel|gemv_kernel" --launch-skip 20 -c 10 -o gpurun_out/s5_ncu_full_apply_prefetch python tools/ncu_cfg4.py apply > gpurun_out/ncu_a5.log 2>&1
tail -2 gpurun_out/ncu_a5.log
python tools/ncu_summary.py gpurun_out/s5_ncu_full_apply_prefetch.ncu-rep > gpurun_out/s5_ncu_full_apply_prefetch.txt 2>&1
cat gpurun_out/s5_ncu_full_apply_prefetch.txt | cut -c1-330
