set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/t3_kernels.log 2>&1
RSC_B200_LIB=$PWD/oldlib/librsc_head.so timeout 600 python tools/digest.py 2 3 4 > gpurun_out/digest_old.txt 2>&1
timeout 600 python tools/digest.py 2 3 4 > gpurun_out/digest_new.txt 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q > gpurun_out/t3_fullsize.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"qrcp|larft|ordered_reduce|gemm_grouped" --csv --log-file gpurun_out/ncu_numeric4_m3.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu_m3.log 2>&1
