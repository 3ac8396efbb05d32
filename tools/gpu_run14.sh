set -x
for i in 1 2; do timeout 600 python tools/digest.py 2 >> gpurun_out/digest15_lpt.txt 2>&1; done
for i in 1 2; do RSC_GEMM_NO_LPT=1 timeout 600 python tools/digest.py 2 >> gpurun_out/digest15_nolpt.txt 2>&1; done
