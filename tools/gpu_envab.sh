#!/bin/bash
# A/B of environment-variable variants of the bench (one bench line each, same build).
# usage: bash tools/gpu_envab.sh <tag> "<env A>" "<env B>" ...   (e.g. "RADE_PRIO=bin")
TAG=$1; shift
mkdir -p gpurun_out
i=0
for E in "$@"; do
  env $E timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/envab_${TAG}_$i.log 2>&1
  python - "$E" gpurun_out/envab_${TAG}_$i.log <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print(f"[{sys.argv[1]}] value {d['value']:.1f} step median {d['config']['step_ms']['median']:.3f} ms")
PY
  i=$((i+1))
done
