set -x
# the dominant kernel (grouped GEMM) of one eager config[4] numeric pass, --set full: two windows of 30 launches
# (mid-sweep and the top separators at the end of the sweep)
for w in 2500 7600; do
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"gemm_grouped_kernel" --launch-skip $w -c 30 -o gpurun_out/s5_ncu_full_gemm_cfg4_w$w python tools/ncu_cfg4.py numeric > gpurun_out/ncu_g5_$w.log 2>&1
tail -1 gpurun_out/ncu_g5_$w.log
python tools/ncu_summary.py gpurun_out/s5_ncu_full_gemm_cfg4_w$w.ncu-rep > gpurun_out/s5_ncu_full_gemm_cfg4_w$w.txt 2>&1
cut -c1-300 gpurun_out/s5_ncu_full_gemm_cfg4_w$w.txt | head -32
done
