"""Summarise gpurun_out ncu artefacts into profiles/ (launch shares, per-kernel key metrics,
DRAM traffic per launch). Usage: python tools/ncu_summary.py <tag>"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
lines = []

# ---- launch list: shares of device time (cold-cache, serialised)
lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lp):
    rows = list(csv.reader(open(lp)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        name = r[ki]
        short = name.split("(")[0].replace("void ", "").replace("rade::<unnamed>::", "")
        if "cub::" in name:
            short = name.split("<")[0].replace("void ", "") + ("(u32 keys)" if "unsigned int, unsigned int, unsigned int" in name else "")
        agg[short].append(float(r[vi]))
    tot = sum(sum(v) for v in agg.values())
    lines.append(f"# ncu launch list ({tag}): share of summed device time, cold-cache serialised\n")
    lines.append("| kernel | launches | avg us | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
    lines.append("")

# ---- full-set report: key metrics per profiled launch
rp = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
traffic = {}
if os.path.exists(rp):
    raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "lts__t_bytes.sum", "smsp__inst_executed.sum"]
    col = {w: hdr.index(w) for w in want if w in hdr}
    ki = hdr.index("Kernel Name")
    lines.append(f"# ncu --set full ({tag}): per profiled launch\n")
    lines.append("| kernel | " + " | ".join(f"{w} [{units[col[w]]}]" for w in col) + " |")
    lines.append("|---" * (len(col) + 1) + "|")
    per = defaultdict(list)
    issue = defaultdict(list)
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("rade::<unnamed>::", "")[:60]
        lines.append(f"| {name} | " + " | ".join(r[col[w]] for w in col) + " |")

        def val(w):
            x = float(r[col[w]].replace(",", ""))
            u = units[col[w]]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if "dram__bytes_read.sum" in col:
            per[name].append(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
        if "smsp__issue_active.avg.pct_of_peak_sustained_active" in col:
            issue[name].append(val("smsp__issue_active.avg.pct_of_peak_sustained_active"))

    def bench_name(name):
        """ncu kernel name -> (the bench's kernel name, launches per bench launch): K2's depth sort is
        K2h + 4 onesweep passes (pass 0 and 3 x pass 1-3), K5 = its kernels summed"""
        n = name.split("::")[-1].replace("(int)", "")
        for pre, b, k in (("k_render_bwd", "render_bwd", 1), ("k_render_fwd", "render_fwd", 1),
                          ("k_preprocess_fwd", "preprocess_fwd", 1),
                          # bench's K5 launch = one rd_preprocess_bwd_views per round of 4 views:
                          # the batched SH kernel once, the batched K5b64 + K5b once (blockIdx.y =
                          # view; per-view K5b64 + K5b four times in older captures)
                          ("k_preprocess_bwd_sh", "preprocess_bwd", 1),
                          ("k_preprocess_bwd_geo_views", "preprocess_bwd", 1),
                          ("k_preprocess_bwd64_views", "preprocess_bwd", 1), ("k_preprocess_bwd", "preprocess_bwd", 4),
                          ("k_bin_hist", "depth_sort", 1), ("k_onesweep<0>", "depth_sort", 1),
                          ("k_onesweep<1>", "depth_sort", 3), ("k_scan", "scan", 1),
                          ("k_onesweep<2>", "duplicate", 1), ("k_onesweep<3>", "tile_sort", 1),
                          ("k_ranges", "ranges", 1)):
            if n.startswith(pre):
                return b, k
        return None, 0
    agg_t, agg_i = defaultdict(float), defaultdict(list)
    for name, v in per.items():
        b, k = bench_name(name)
        if b:  # a bench launch = its kernels summed
            agg_t[b] += k * sum(v) / len(v)
            agg_i[b] += issue.get(name, [])
    traffic = dict(agg_t)
    issue_pct = {b: sum(v) / len(v) for b, v in agg_i.items() if v}
    lines.append("")
open(os.path.join(out_dir, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
if traffic:
    tp = os.path.join(out_dir, "traffic.json")
    old = json.load(open(tp)) if os.path.exists(tp) else {}
    old = {k: v for k, v in old.items() if isinstance(v, dict)}  # drop the pre-r1w flat layout
    for b, t in traffic.items():
        old[b] = {"dram_bytes_per_launch": t, "issue_active_pct": issue_pct.get(b), "capture": tag}
    old["_about"] = {"what": "per bench kernel (one C-ABI launch; K5 = its 3 kernels summed): dram__bytes_read.sum + "
                             "dram__bytes_write.sum per launch and smsp__issue_active (% of peak, active cycles) "
                             "from the latest `ncu --set full` capture that contains it (profiles/ncu_<capture>.md)"}
    json.dump(old, open(tp, "w"), indent=1)
print("\n".join(lines))
