set -x
timeout 900 python tools/digest.py 2 3 4 2>&1 | grep "^cfg"
for v in final new final new; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'value', d['value'], 'numeric', d['config']['numeric_factor_s'], 'e2e', d['e2e']['value'], 'reduce_s', d['config']['kernel_time_top'].get('ordered_reduce_kernel'), 'gemm_s', d['roofline']['kernel_seconds'])"
done
