#!/bin/bash
# ncu --set full of one kernel (regex $2) of a short bench run; tag $1; extra bench args after.
TAG=$1; KREGEX=$2; shift 2
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $*"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 5 -c 2 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$TAG.log
