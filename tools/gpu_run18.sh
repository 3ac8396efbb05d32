set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t21_kernels.log 2>&1
for c in 2 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest21.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench21.json 2> gpurun_out/bench21.err
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q > gpurun_out/t21_full.log 2>&1
