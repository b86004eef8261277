#!/bin/bash
# Per-variant probe times + ncu instruction counts of the binning kernels:
#   bash tools/gpu_binab_ncu.sh "<flags A>" "<flags B>" ...
mkdir -p gpurun_out
for F in "$@"; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > /dev/null 2>&1 || { echo "build failed: $F"; continue; }
  echo "[$F]"
  timeout 300 python tools/bin_probe.py --reps 10 2>&1 | grep -E "views|depth|scan|dupl|tile_sort"
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_onesweep|k_scan|k_bin_hist" --csv --log-file gpurun_out/binabn.csv python tools/bin_probe.py --views 1 --reps 1 > /dev/null 2>&1
  python - <<'PY'
import csv
from collections import defaultdict
rows = [r for r in csv.reader(open("gpurun_out/binabn.csv")) if len(r) > 5]
hdr = [r for r in rows if "Metric Name" in r][0]
ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(dict); names = {}
for r in rows:
    if r is hdr or "Metric Name" in r: continue
    per[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")); names[int(r[ii])] = r[ki].split("(")[0][-22:]
ids = sorted(per)[-9:]
print("   ", "  ".join(f"{names[i]}: {per[i]['gpu__time_duration.sum']/1e3:.1f}us/{per[i]['smsp__inst_executed.sum']/1e6:.1f}M" for i in ids))
PY
done
