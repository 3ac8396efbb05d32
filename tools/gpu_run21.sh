set -x
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_plan_abi_gpu.py -x -q > gpurun_out/t25.log 2>&1
for mb in 0.0 0.25 0.5 1 2; do RSC_APPLY_TREE_CLUSTER_MB=$mb timeout 600 python tools/apply_time.py 4 1 > gpurun_out/apply_time25_$mb.txt 2>&1; done
