"""Binning probe: K1 + K2 of a few C3 views on one stream, per-kernel CUDA-event times (the
ABI's profiling hooks) and the wall time of preprocess+bin per view. Development tool.

    python tools/bin_probe.py [--config c3] [--views 8] [--reps 5] [--tile 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--views", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tile", type=int, default=8)
args = ap.parse_args()

scene, cams, opt = sg.config_scene_and_cameras(args.config)
opt.tile = args.tile
g = P.Gaussians.from_numpy(scene, "cuda")

view = P.View()
s = torch.cuda.current_stream()
for c in cams[: args.views]:  # warm-up (allocations)
    P.rd_preprocess(view, g, c, opt)
    P.rd_bin(view)
torch.cuda.synchronize()
P.rd_set_profiling(view, True)
P.rd_get_timings(view, reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
nv = 0
for _ in range(args.reps):
    for c in cams[: args.views]:
        P.rd_preprocess(view, g, c, opt)
        P.rd_bin(view)
        nv += 1
e1.record()
torch.cuda.synchronize()
t = P.rd_get_timings(view)
print(f"views {nv}: {e0.elapsed_time(e1) / nv:.4f} ms per view (preprocess + bin, one stream, host syncs incl.)")
for k, v in t["ms"].items():
    if v:
        print(f"  {k:16s} {v / nv:.4f} ms")
print("  M per view", t.get("n_duplicates", 0) / max(nv, 1), "visible", P.rd_view_stats(view)["n_visible"])

lib = P._native.load()
if hasattr(lib, "rd_debug_bin_trace"):  # built with -DRD_BIN_TRACE: phases of the last tile pass
    import ctypes
    import numpy as np
    M = P.rd_view_stats(view)["n_duplicates"]
    nb = min(8192, (M + 4095) // 4096)
    buf = np.zeros((nb, 6), np.uint64)
    lib.rd_debug_bin_trace(buf.ctypes.data_as(ctypes.c_void_p), nb)
    t = buf[:, :5].astype(np.float64)
    t0 = t[:, 0].min()
    ph = np.diff(t, axis=1)
    print(f"tile pass blocks {nb}: span {(t[:, 4].max() - t0) / 1e3:.1f} us; per block (median / p90 us):")
    for k, name in enumerate(("load+setup", "rank", "lookback", "scatter")):
        print(f"  {name:10s} {np.median(ph[:, k]) / 1e3:.2f} / {np.percentile(ph[:, k], 90) / 1e3:.2f}")
    print("  start offsets (us) of blocks 0, 600, 1200, 2400:", [(t[i, 0] - t0) / 1e3 for i in (0, 600, 1200, 2400) if i < nb])
