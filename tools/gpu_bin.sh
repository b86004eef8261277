#!/bin/bash
# Binning probe on the GPU: event times, the ncu launch list, and a full capture of the sort
# passes. usage: bash tools/gpu_bin.sh <tag> [probe args]
TAG=${1:-b}; shift
mkdir -p gpurun_out
timeout 300 python tools/bin_probe.py "$@" > gpurun_out/binprobe_$TAG.log 2>&1
cat gpurun_out/binprobe_$TAG.log
P="python tools/bin_probe.py --views 2 --reps 1 $*"
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/binlaunch_$TAG.csv $P > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(f"gpurun_out/binlaunch_{sys.argv[1]}.csv")) if len(r) > 5]
hdr = [r for r in rows if "Metric Name" in r][0]
ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(dict); names = {}
for r in rows:
    if r is hdr or "Metric Name" in r: continue
    per[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")); names[int(r[ii])] = r[ki].split("(")[0][:60]
for i in sorted(per)[-40:]:
    m = per[i]
    print(f"{i:4d} {names[i]:60s} {m.get('gpu__time_duration.sum',0)/1e3:8.1f} us  warps {m.get('sm__warps_active.avg.pct_of_peak_sustained_active',0):5.1f}%  dram {(m.get('dram__bytes_read.sum',0)+m.get('dram__bytes_write.sum',0))/1e6:7.1f} MB  inst {m.get('smsp__inst_executed.sum',0)/1e6:6.2f} M")
PY
