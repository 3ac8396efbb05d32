set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_plan_abi_gpu.py -x -q > gpurun_out/t18_kernels.log 2>&1
for c in 2 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest18.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench18.json 2> gpurun_out/bench18.err
timeout 600 python tools/prof_numeric.py 4 > gpurun_out/prof_numeric18.txt 2>&1
