#!/bin/bash
# A/B of compile-time variants on the binning probe: bash tools/gpu_binab.sh "<flags A>" "<flags B>" ...
mkdir -p gpurun_out
for F in "$@"; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > /dev/null 2>&1 || { echo "build failed: $F"; continue; }
  echo "[$F]"
  timeout 300 python tools/bin_probe.py --reps 10 2>&1 | grep -v "^ *$" | head -16
done
