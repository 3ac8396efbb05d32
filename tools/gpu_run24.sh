# final round-2 evidence run: GPU tests, smoke, default bench line, reference-free; then the ncu launch
# list of one timed step of the same bench command
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_t_all.log 2>&1
tail -3 gpurun_out/s5_t_all.log
timeout 600 python __graft_entry__.py > gpurun_out/s5_smoke.log 2>&1; tail -1 gpurun_out/s5_smoke.log
for v in base new; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 300 python tools/qr_micro.py 6048 987 1 2>&1 | grep "^qrcp" | sed "s/^/$v /"
  timeout 300 python tools/qr_micro.py 6048 987 2 2>&1 | grep "^qrcp" | sed "s/^/$v /"
  timeout 300 python tools/qr_micro.py 9000 700 3 2>&1 | grep "^qrcp" | sed "s/^/$v /"
done
unset RSC_B200_LIB
timeout 1200 python bench.py > gpurun_out/s5_bench_final.json 2> gpurun_out/s5_bench_final.err
tail -c 1500 gpurun_out/s5_bench_final.json
RSC_BENCH_PROFILE_RANGE=1 timeout 3300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches_bench_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ncu_bench.log 2>&1
tail -2 gpurun_out/s5_ncu_bench.log | cut -c1-300
ls -la gpurun_out/s5_launches_bench_cfg4.csv
