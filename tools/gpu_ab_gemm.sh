set -x
for v in head mb4 s3 s3mb3 cur; do
  if [ $v = cur ]; then L=""; else L="RSC_B200_LIB=$PWD/oldlib/librsc_$v.so"; fi
  env $L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
done
