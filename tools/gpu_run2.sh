set -x
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 600 python tools/prof_numeric.py 4 > gpurun_out/prof_numeric4.txt 2>&1
timeout 600 python tools/apply_time.py 4 0 1 4 16 64 > gpurun_out/apply_time4.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mqrcp_kernel --launch-skip 25 -c 1 -o gpurun_out/ncu_mqrcp_glob python tools/ncu_cfg4.py numeric > gpurun_out/ncu_q1.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:mqrcp_kernel --launch-skip 9 -c 1 -o gpurun_out/ncu_mqrcp_smem python tools/ncu_cfg4.py numeric > gpurun_out/ncu_q2.log 2>&1
RSC_GEMM_STATS=1 timeout 600 python tools/ncu_cfg4.py numeric > gpurun_out/gemm_stats.txt 2>&1
