set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t14_kernels.log 2>&1
for c in 2 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest14.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_lpt.json 2> gpurun_out/bench14_lpt.err
RSC_GEMM_NO_LPT=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_nolpt.json 2> gpurun_out/bench14_nolpt.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_lpt2.json 2> gpurun_out/bench14_lpt2.err
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_c1.json 2> gpurun_out/bench14_c1.err
