set -x
# correctness first: digests must equal cfg2 163a8afe9b847c31/5241226882256968519, cfg3 e930259a99a9d722/3748356275046269567,
# cfg4 b113ceb5911cdaae/7949053538307843873
timeout 900 python tools/digest.py 2 3 4 2>&1 | grep "^cfg"
for v in pf0 new pfp pf0 new; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/$v /"
done
unset RSC_B200_LIB
timeout 600 python tools/apply_breakdown.py 4 > gpurun_out/s5_apply_breakdown_cfg4_pf.txt 2>&1
tail -12 gpurun_out/s5_apply_breakdown_cfg4_pf.txt
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_plan_abi_gpu.py tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
for k in "1 1" "0 1" "0 0" "0 1" "0 0"; do
set -- $k
RSC_GC=$1 RSC_GEMM_PDL=$2 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('gc', $1, 'pdl', $2, 'value', d['value'], 'numeric', d['config']['numeric_factor_s'], 'e2e', d['e2e']['value'], 'gemm_s', d['roofline']['kernel_seconds'], 'apply', d['hbm_roofline']['apply']['seconds'])"
done
