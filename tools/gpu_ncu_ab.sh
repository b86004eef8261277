#!/bin/bash
# Per-variant ncu metrics of one kernel: usage bash tools/gpu_ncu_ab.sh <kernel-regex> "<flags A>" "<flags B>" ...
K=$1; shift
mkdir -p gpurun_out
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"
for F in "$@"; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > /dev/null 2>&1
  B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  $B > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"$K" -s 4 -c 2 --csv --log-file gpurun_out/ncuab.csv $B > /dev/null 2>&1
  echo "[$F]"
  python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/ncuab.csv")) if len(r) > 5]
hdr = [r for r in rows if "Metric Name" in r][0]
rows = [r for r in rows if r is not hdr and "Metric Name" not in r]
mi, vi = hdr.index("Metric Name"), hdr.index("Metric Value")
from collections import defaultdict
agg = defaultdict(list)
for r in rows:
    if len(r) > vi:
        agg[r[mi]].append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"  {k}: {sum(v)/len(v):.4g}")
PY
done
