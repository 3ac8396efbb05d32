set -x
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_kernels_gpu.py tests/test_plan_abi_gpu.py -x -q > gpurun_out/s4_t1.log 2>&1
tail -3 gpurun_out/s4_t1.log
timeout 600 python tools/apply_treeinv.py 4 2>&1 | grep "tree_inv"
timeout 600 python tools/apply_breakdown.py 4 > gpurun_out/s4_apply_breakdown_cfg4_b5.txt 2>&1
tail -12 gpurun_out/s4_apply_breakdown_cfg4_b5.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4_bench_b5.json 2> gpurun_out/s4_bench_b5.err
tail -c 900 gpurun_out/s4_bench_b5.json
