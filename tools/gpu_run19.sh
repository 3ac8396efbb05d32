set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t23_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench23_default.json 2> gpurun_out/bench23_default.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none -k regex:gemm_grouped --csv --log-file gpurun_out/ncu_gemm23.csv python tools/ncu_cfg4.py numeric > gpurun_out/ncu23.log 2>&1
