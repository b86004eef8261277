#!/bin/bash
# A/B of compile-time variants on the NEXT rows (tools/bench_next.py): usage bash tools/gpu_abnext.sh "<flags A>" ...
for F in "$@"; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > /dev/null 2>&1
  echo "[$F]"; timeout 600 python tools/bench_next.py 2>&1 | grep -o '"ms_per_32_views": [0-9.]*\|"fused_voxels": [0-9]*\|"row": "NEXT-4 marching_cubes", "workload": "[^"]*", "ms": [0-9.]*'
done
