set -x
for c in 740 444 1480 2960; do RSC_GEMM_CTAS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench16_$c.json 2> gpurun_out/bench16_$c.err; done
