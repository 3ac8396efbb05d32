set -x
timeout 900 python -m pytest tests/test_plan_abi_gpu.py -x -q > gpurun_out/t8_plan.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t8_gpu.log 2>&1
timeout 600 python tools/apply_time.py 4 0 1 > gpurun_out/apply_time8.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err
