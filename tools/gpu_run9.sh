set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_plan_abi_gpu.py -x -q > gpurun_out/t11_kernels.log 2>&1
for c in 2 3 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest11.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench11.json 2> gpurun_out/bench11.err
timeout 600 python tools/prof_e2e.py 4 > gpurun_out/prof_e2e11.txt 2>&1
