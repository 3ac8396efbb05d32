set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t12_kernels.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q > gpurun_out/t12_full.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench12.json 2> gpurun_out/bench12.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce" --csv --log-file gpurun_out/ncu_numeric4_m12.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m12.log 2>&1
