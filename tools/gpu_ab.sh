#!/bin/bash
# A/B timing of compile-time variants on one box: for each quoted flag set, rebuild librade.so
# with RADE_EXTRA_NVCC_FLAGS and run one bench line. usage: bash tools/gpu_ab.sh <tag> "<flags A>" "<flags B>" ...
TAG=$1; shift
mkdir -p gpurun_out
i=0
for F in "$@"; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > gpurun_out/ab_build_${TAG}_$i.log 2>&1 || { echo "build failed: $F"; tail gpurun_out/ab_build_${TAG}_$i.log; continue; }
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_$i.log 2>&1
  python - "$F" gpurun_out/ab_${TAG}_$i.log <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        k = d["config"]["ms_per_view_by_kernel"]
        print(f"[{sys.argv[1]}] value {d['value']:.1f}  fwd {k['render_fwd']:.4f} bwd {k['render_bwd']:.4f} pre {k['preprocess_fwd']:.4f} prebwd {k['preprocess_bwd']:.4f}")
PY
  i=$((i+1))
done
