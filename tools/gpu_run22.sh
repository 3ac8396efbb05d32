set -x
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_alg_gpu.py -x -q > gpurun_out/s4_t1.log 2>&1
tail -3 gpurun_out/s4_t1.log
timeout 600 python tools/apply_treeinv.py 4 > gpurun_out/s4_treeinv_cfg4.txt 2>&1
grep tree_inv gpurun_out/s4_treeinv_cfg4.txt || tail -20 gpurun_out/s4_treeinv_cfg4.txt
timeout 600 python tools/apply_breakdown.py 4 > gpurun_out/s4_apply_breakdown_cfg4.txt 2>&1
tail -14 gpurun_out/s4_apply_breakdown_cfg4.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4_bench_treeinv.json 2> gpurun_out/s4_bench_treeinv.err
tail -c 1500 gpurun_out/s4_bench_treeinv.json
