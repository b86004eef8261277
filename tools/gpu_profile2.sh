#!/bin/bash
# Round-2 profile: GPU tests, the default bench line (with the CPU baseline), the ncu launch
# list of a short bench run and one `ncu --set full` capture of every kernel of a few views.
#   usage (under gpurun): bash tools/gpu_profile2.sh <tag>
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
grep '^{' gpurun_out/bench_$TAG.log | head -c 400; echo
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_list_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess|k_render|k_ranges|k_tile_order" -s 60 -c 14 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" | tee -a gpurun_out/ncu_full_$TAG.log
