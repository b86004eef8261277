#!/bin/bash
# ncu --set full of the binning kernels matching $2 in the probe (tag $1)
TAG=$1; K=${2:-k_onesweep}; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c ${CNT:-8} -o gpurun_out/prof_$TAG python tools/bin_probe.py --views 1 --reps 1 "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
