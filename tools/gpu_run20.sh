set -x
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_plan_abi_gpu.py tests/test_alg_gpu.py -x -q > gpurun_out/t24.log 2>&1
timeout 600 python tools/apply_time.py 4 0 1 > gpurun_out/apply_time24_cl.txt 2>&1
RSC_APPLY_TREE_CLUSTER=0 timeout 600 python tools/apply_time.py 4 0 1 > gpurun_out/apply_time24_nocl.txt 2>&1
