set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_t_all.log 2>&1
tail -3 gpurun_out/s4_t_all.log
timeout 600 python tools/apply_treeinv.py 4 2>&1 | grep "tree_inv 1"
timeout 600 python tools/prof_apply_build.py 4 > gpurun_out/s4_prof_apply_build.txt 2>&1
head -40 gpurun_out/s4_prof_apply_build.txt | cut -c1-150
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"mqrcp_kernel" --launch-skip 24 -c 9 -o gpurun_out/s4_ncu_full_mqrcp python tools/ncu_cfg4.py numeric > gpurun_out/ncu_q.log 2>&1
tail -3 gpurun_out/ncu_q.log
