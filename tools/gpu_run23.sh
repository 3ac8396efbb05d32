set -x
for v in new mq2 new mq2; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 600 python tools/digest.py 4 2>&1 | grep "^cfg" | sed "s/^/$v /"
  timeout 300 python tools/qr_micro.py 6048 987 2 2>&1 | grep "^qrcp" | sed "s/^/$v /"
done
unset RSC_B200_LIB
RSC_BENCH_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_bench_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s4_ncu_bench.log 2>&1
tail -2 gpurun_out/s4_ncu_bench.log | cut -c1-300
ls -la gpurun_out/s4_launches_bench_cfg4.csv
