"""Top SASS lines of a kernel by warp-stall samples and by instructions, from an ncu report's
source page. usage: python tools/ncu_hot.py <rep> <kernel-substring> [occurrence] [top]"""
import csv, subprocess, sys
rep, ksub = sys.argv[1], sys.argv[2]
occ = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sel = [b for b in blocks if ksub in b["name"]][occ]
hdr = sel["rows"][0]
data = sel["rows"][1:]
si, ii, ai = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
tot_s = sum(float(r[si] or 0) for r in data)
tot_i = sum(float(r[ii] or 0) for r in data)
print(sel["name"][:100], f"samples {tot_s:.0f} instructions {tot_i:.0f}")
# stall reason columns
rc = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:top]:
    print(f"{idx:5d} {float(r[si] or 0)/tot_s*100:5.1f}% inst {float(r[ii] or 0)/tot_i*100:5.1f}%  {r[ai].strip()[:70]}")
print("--- by instructions")
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][ii] or 0))[:top]:
    print(f"{idx:5d} {float(r[si] or 0)/tot_s*100:5.1f}% inst {float(r[ii] or 0)/tot_i*100:5.1f}%  {r[ai].strip()[:70]}")
