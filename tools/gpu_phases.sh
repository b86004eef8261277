#!/bin/bash
# Anatomy of a bench step: per-view phase events (RADE_PHASES: start, binned, fwd start, fwd
# end, K5 start, K5 end; ms from the first view of the last 5 steps) and per-kernel times under
# the concurrent schedule (RADE_PROF_CONC). usage: bash tools/gpu_phases.sh <tag> [bench args]
TAG=${1:-ph}; shift
mkdir -p gpurun_out
RADE_PHASES=gpurun_out/phases_$TAG.json RADE_PROF_CONC=1 timeout 600 python bench.py --steps 20 --warmup 5 \
  --no-cpu-baseline --no-e2e "$@" > gpurun_out/phases_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/phases_$TAG.log
grep -v "^{" gpurun_out/phases_$TAG.log | tail -3
