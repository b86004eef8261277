#!/bin/bash
# Quick GPU round trip: parity tests then one bench line. usage: bash tools/gpu_quick.sh <tag> [bench args]
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
for l in open(f"gpurun_out/bench_{tag}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", round(d["value"], 1), "e2e", round(d.get("e2e", {}).get("value", 0), 1))
        print({k: round(v, 4) for k, v in d["config"]["ms_per_view_by_kernel"].items()})
PY
