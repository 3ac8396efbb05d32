set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t7_gpu.log 2>&1
for c in 2 3 4; do timeout 600 python tools/digest.py $c >> gpurun_out/digest7.txt 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce" --csv --log-file gpurun_out/ncu_numeric4_m7.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m7.log 2>&1
