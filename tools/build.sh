#!/bin/bash
# rebuild the in-tree library (from any cwd) and summarise ptxas usage of the hot kernels;
# a failed build prints the nvcc error and exits non-zero
cd /root/repo || exit 1
out=$(python -c "from paper_2510_10467_b200 import build; build.build()" 2>&1)
rc=$?
if [ $rc -ne 0 ]; then
    echo "$out" | grep -v "^ptxas" | grep -B2 -A6 -iE "error" | head -40
    echo "BUILD FAILED"
    exit $rc
fi
grep -A2 "gemv_batch_kernel\|batch_reduce\|gemm_mixedp" /root/repo/paper_2510_10467_b200/build/ptxas.log | grep -E "Used|spill" | sort | uniq -c
