#!/bin/bash
# Run ON THE GPU BOX (gpurun): the bench command plain, then its launch list and
# one full capture of the hot kernel, plus one full capture of the cluster
# single-GEMV kernel (4096x4096 p=2), all into gpurun_out/. Summarise here with
#   python tools/profiles_commit.py <tag>
set -e
TAG=${1:-r2}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --sections none"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemv_batch|batch_reduce|gemv_cluster" -c 40 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_batch_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > /dev/null 2>&1
CL="python tools/gemv_probe.py --rows 4096 --cols 4096 --p 2 --iters 5 --copies 2"
$CL > gpurun_out/plain_cl_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_cluster -s 2 -c 1 \
    -o gpurun_out/prof_cl_$TAG $CL > /dev/null 2>&1
ls -la gpurun_out/
