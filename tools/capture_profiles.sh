#!/bin/bash
# Run ON THE GPU BOX (gpurun): the bench command plain, then its launch list and
# one full capture of the hot kernel, all into gpurun_out/. Summarise here with
#   python tools/ncu_summary.py gpurun_out/prof_<tag>.ncu-rep
#   python tools/profiles_commit.py <tag>
set -e
TAG=${1:-r1}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemv_batch|batch_reduce" -c 40 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_batch_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > /dev/null 2>&1
ls -la gpurun_out/
