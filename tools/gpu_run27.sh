set -x
for v in new pfa new pfa; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/$v /"
done
export RSC_B200_LIB=$PWD/variants/librsc_pfa.so
timeout 600 python tools/apply_breakdown.py 4 > gpurun_out/s5_apply_breakdown_cfg4_pfa.txt 2>&1
tail -8 gpurun_out/s5_apply_breakdown_cfg4_pfa.txt
timeout 600 python tools/apply_time.py 2 1 2>&1 | grep "^task_mb" | sed "s/^/pfa cfg2 /"
unset RSC_B200_LIB
timeout 600 python tools/apply_time.py 2 1 2>&1 | grep "^task_mb" | sed "s/^/new cfg2 /"
