set -x
RSC_GEMM_LOG=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_grouped --csv --log-file gpurun_out/ncu_gemm13.csv python tools/ncu_cfg4.py numeric > gpurun_out/gemm13.out 2> gpurun_out/gemmlog13.txt
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab1_cur.json 2> gpurun_out/ab1_cur.err
RSC_B200_LIB=$PWD/oldlib/librsc_mb4.so timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab1_mb4.json 2> gpurun_out/ab1_mb4.err
