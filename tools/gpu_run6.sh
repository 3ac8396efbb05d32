set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t6_kernels.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_factor_gpu.py tests/test_alg_gpu.py -x -q > gpurun_out/t6_fullsize.log 2>&1
for c in 2 3 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest6_new.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce" --csv --log-file gpurun_out/ncu_numeric4_m6.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m6.log 2>&1
timeout 600 python tools/prof_e2e.py 4 > gpurun_out/prof_e2e6.txt 2>&1
