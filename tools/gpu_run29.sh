set -x
for v in new fw mb4 mb6 rpb8 rpb2 new; do
  if [ $v = new ]; then unset RSC_B200_LIB; else export RSC_B200_LIB=$PWD/variants/librsc_$v.so; fi
  timeout 600 python tools/apply_time.py 4 1 2>&1 | grep "^task_mb" | sed "s/^/$v /"
done
