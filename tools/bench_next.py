"""Measurement of the NEXT rows on the C3 workload (B200), one JSON line each:

  normal_consistency  L_n forward + backward per view (image-space, HBM-bound)
  tsdf_integrate      fusion of 32 C3 median depth maps into a 256³ volume (HBM-bound)
  marching_cubes      mesh extraction from that volume (count, scan, emit)
  filter3d            the bench step with the Mip-Splatting 3D filter on (frames/s)

    python tools/bench_next.py [--steps K]

Kernel times are CUDA-event timed on the launching stream after warm-up; achieved
bandwidth counts algorithmic bytes only (stated per line) against MEASURED_PEAKS.json.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6540.8


def timed(fn, reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 20
    peak = hbm_peak()
    scene, cams, opt = sg.config_scene_and_cameras("C3")
    g = P.Gaussians.from_numpy(scene)
    opts = dict(tile=8, alpha_min=opt.alpha_min, alpha_max=opt.alpha_max, T_min=opt.T_min, median_T=opt.median_T,
                dilation=opt.dilation, bg=opt.bg, sh_degree=opt.sh_degree, guard_band=opt.guard_band)
    view = P.View()
    maps = []
    for cam in cams[:32]:
        out, view = P.render(g, cam, opts, view)
        maps.append({k: v.clone() for k, v in out.items()})
    torch.cuda.synchronize()
    H, W = cams[0].height, cams[0].width

    # ---- L_n forward + backward
    m = maps[0]
    Ln = torch.empty((H, W), device="cuda")
    gL = torch.randn((H, W), device="cuda")
    gD, gA, gN = torch.zeros((H, W), device="cuda"), torch.zeros((H, W), device="cuda"), \
        torch.zeros((3, H, W), device="cuda")

    def ln():
        P.rd_normal_consistency(cams[0], m["depth"], m["alpha"], m["normal"], consistency=Ln)
        P.rd_normal_consistency_bwd(cams[0], m["depth"], m["normal"], gL, gD, gA, gN)

    for _ in range(3):
        ln()
    ms = timed(ln, steps)
    byts = H * W * (4 * 3 + 4 + 12 + 4) + H * W * (4 * 2 + 12 + 4 + 4 * 2 + 12 * 2)  # fwd in/out + bwd in/RMW
    print(json.dumps({"row": "NEXT-2 normal_consistency fwd+bwd", "workload": "C3 1237x822, one view",
                      "ms": ms, "achieved_GBps": byts / (ms * 1e-3) / 1e9, "peak_GBps": peak,
                      "frac": byts / (ms * 1e-3) / 1e9 / peak,
                      "bytes": "fwd: depth (3 taps, cached), alpha, normal in, L_n out; bwd: depth, normal, g in, "
                               "dL/dD (atomic RMW), dL/dA, dL/dN RMW"}), flush=True)

    # ---- TSDF fusion of 32 C3 median depth maps into 256^3
    D = torch.stack([mm["depth"] for mm in maps]).contiguous()
    vol = P.TsdfVolume((-3.0, -3.0, -2.0), 6.0 / 256, (256, 256, 256), max_depth=30.0)
    P.rd_tsdf_integrate(vol, D, cams[:32])

    def fuse():
        P.rd_tsdf_integrate(vol, D, cams[:32])

    ms = timed(fuse, max(3, steps // 4))
    nvox = 256 ** 3
    byts = nvox * 16  # tsdf + weight read and written once per 32-view launch
    print(json.dumps({"row": "NEXT-4 tsdf_integrate", "workload": "32 C3 median depth maps -> 256^3 voxels",
                      "ms_per_32_views": ms, "voxel_updates_per_s": nvox * 32 / (ms * 1e-3),
                      "achieved_GBps": byts / (ms * 1e-3) / 1e9, "peak_GBps": peak,
                      "frac": byts / (ms * 1e-3) / 1e9 / peak,
                      "bytes": "16 B per voxel per launch (tsdf + weight in and out); the depth gathers hit L2",
                      "fused_voxels": int((vol.weight > 0).sum().item())}), flush=True)

    # ---- marching cubes on the fused 256^3 volume (count + scan + emit, one sync)
    ntri = P.rd_marching_cubes(vol).shape[0]

    def mc():
        P.rd_marching_cubes(vol)

    ms = timed(mc, max(3, steps // 4))
    ncell = 255 ** 3
    byts = ncell * 8 * 2 + ncell * 8 + ntri * 36  # 2 passes × (tsdf, weight) ≈ 8 B/cell (x-neighbours cached), count+offset, out
    print(json.dumps({"row": "NEXT-4 marching_cubes", "workload": "fused 256^3 volume of 32 C3 views",
                      "ms": ms, "triangles": ntri, "cells_per_s": ncell / (ms * 1e-3),
                      "achieved_GBps": byts / (ms * 1e-3) / 1e9, "peak_GBps": peak,
                      "frac": byts / (ms * 1e-3) / 1e9 / peak,
                      "bytes": "per cell: tsdf+weight read by count and emit passes, 4-B count + 4-B offset, "
                               "36 B per triangle out (includes the host round trip of the count)"}), flush=True)

    # ---- the step with the 3D filter (forward + backward per view, serial)
    g.filter3d = torch.full((g.n,), 0.004, device="cuda")
    grads = g.zeros_like()
    cot = torch.randn((8, H, W), device="cuda")

    def step():
        for cam in cams[:4]:
            P.rd_preprocess(view, g, cam, opts)
            P.rd_bin(view)
            P.rd_render_fwd(view)
            P.rd_render_bwd(view, g, cot[0:3], cot[3], cot[4:7], cot[7], grads)

    for _ in range(3):
        step()
    ms = timed(step, max(3, steps // 4))
    print(json.dumps({"row": "NEXT-3 filter3d", "workload": "C3, f = 0.004 for every Gaussian, 4 views per step, "
                      "one stream", "frames_per_s": 4 / (ms * 1e-3), "ms_per_view": ms / 4}), flush=True)


if __name__ == "__main__":
    main()
