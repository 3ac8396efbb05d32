set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t4_kernels.log 2>&1
for c in 2 3 4; do
RSC_B200_LIB=$PWD/oldlib/librsc_head.so timeout 600 python tools/digest.py $c >> gpurun_out/digest4_old.txt 2>&1
timeout 600 python tools/digest.py $c >> gpurun_out/digest4_new.txt 2>&1
done
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_factor_gpu.py -x -q > gpurun_out/t4_fullsize.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce" --csv --log-file gpurun_out/ncu_numeric4_m4.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m4.log 2>&1
