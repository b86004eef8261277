#!/bin/bash
# One bench line per BASELINE.json config shape (C1 NeRF-Synthetic, C2 DTU, C3 Mip-NeRF 360, C4 3M
# Gaussians at N = 1) -> gpurun_out/configs_<tag>.jsonl. usage: bash tools/gpu_configs.sh <tag>
TAG=${1:-c}
mkdir -p gpurun_out
: > gpurun_out/configs_$TAG.jsonl
for C in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg_${TAG}_$C.log 2>&1
  grep '^{' gpurun_out/cfg_${TAG}_$C.log >> gpurun_out/configs_$TAG.jsonl || tail -5 gpurun_out/cfg_${TAG}_$C.log
done
python - "$TAG" <<'PY'
import json, sys
for l in open(f"gpurun_out/configs_{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    c = d["config"]
    print(c["workload"][:40], "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1),
          "M", int(c["M_per_view"]), "vis", int(c["visible_per_view"]))
PY
