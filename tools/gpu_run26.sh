# final state: GPU tests, smoke, digests (must equal the values in gpu_run25.sh), default bench line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_t_all2.log 2>&1
tail -3 gpurun_out/s5_t_all2.log
timeout 600 python __graft_entry__.py > gpurun_out/s5_smoke2.log 2>&1; tail -1 gpurun_out/s5_smoke2.log
timeout 900 python tools/digest.py 2 3 4 2>&1 | grep "^cfg"
timeout 300 python tools/qr_micro.py 6048 987 1 2>&1 | grep "^qrcp"
timeout 300 python tools/qr_micro.py 6048 987 2 2>&1 | grep "^qrcp"
timeout 1200 python bench.py > gpurun_out/s5_bench_final2.json 2> gpurun_out/s5_bench_final2.err
tail -c 1600 gpurun_out/s5_bench_final2.json
timeout 600 python tools/apply_breakdown.py 4 > gpurun_out/s5_apply_breakdown_cfg4_final.txt 2>&1
tail -12 gpurun_out/s5_apply_breakdown_cfg4_final.txt
