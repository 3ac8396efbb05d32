set -x
RSC_GEMV_NOSHIFT=1 timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/noshift /"
timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/shift /"
RSC_GEMV_NOSHIFT=1 timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/noshift /"
timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/shift /"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_t_all4.log 2>&1
tail -3 gpurun_out/s5_t_all4.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s5_bench_final4.json 2> gpurun_out/s5_bench_final4.err
tail -c 900 gpurun_out/s5_bench_final4.json
