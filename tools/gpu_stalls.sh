#!/bin/bash
# Warp-state (stall reason) breakdown of K3 and K4 in a C3 bench step.
# usage: bash tools/gpu_stalls.sh [tag]   -> gpurun_out/stalls_<tag>.csv
TAG=${1:-cur}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > /dev/null 2>&1 || { echo "bench failed"; exit 1; }
timeout 900 ncu --section WarpStateStats --section SchedulerStats --section Occupancy --section LaunchStats \
  --clock-control none -k regex:"${KREGEX:-k_render_(fwd|bwd)}" -s ${KSKIP:-8} -c ${KCOUNT:-2} --csv --page raw \
  --log-file gpurun_out/stalls_${TAG}.csv $B > /dev/null 2>&1
python - gpurun_out/stalls_${TAG}.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "")[:60])
    for k, v in d.items():
        if ("issue_stalled" in k and k.endswith("per_issue_active.ratio")) or k in (
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
                "smsp__warps_eligible.avg.per_cycle_active", "gpu__time_duration.sum",
                "smsp__average_warp_latency_per_inst_issued.ratio"):
            try:
                if float(v.replace(",", "")) > 0.5 or "stalled" not in k:
                    print(f"   {k}: {v}")
            except ValueError:
                pass
PY
