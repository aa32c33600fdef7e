#!/bin/bash
# rebuild the in-tree library (from any cwd) and summarise ptxas usage of the hot kernels
cd /root/repo && python -c "from paper_2510_10467_b200 import build; build.build()" 2>&1 | grep -iE "error|warning" | head -20
grep -A2 "gemv_batch_kernel\|batch_reduce\|gemm_mixedp" /root/repo/paper_2510_10467_b200/build/ptxas.log | grep -E "Used|spill" | sort | uniq -c
