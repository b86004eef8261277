#!/bin/bash
# One GPU round trip: parity tests, a bench line, the ncu launch list of the bench command,
# and one `ncu --set full` capture of the kernels matching $KREGEX.
#   usage (under gpurun): bash tools/gpu_profile.sh <tag> [kernel-regex] [extra bench args]
TAG=${1:-r1}
KREGEX=${2:-"k_render_bwd|k_render_fwd|k_preprocess_bwd"}
if [ $# -ge 2 ]; then shift 2; else shift $#; fi
mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 "$@" > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $*"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_list_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 10 -c 10 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$TAG.log
