"""Per-tile list-length statistics of the binning (GPU): sizes the per-tile sort's classes.

    python tools/seg_stats.py [C1 C2 C3 C4]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
    for name in cfgs:
        scene, cams, opt = sg.config_scene_and_cameras(name)
        g = P.Gaussians.from_numpy(scene)
        opts = dict(tile=opt.tile, alpha_min=opt.alpha_min, alpha_max=opt.alpha_max, T_min=opt.T_min,
                    median_T=opt.median_T, dilation=opt.dilation, bg=opt.bg, sh_degree=opt.sh_degree, guard_band=opt.guard_band)
        view = P.View()
        lens = []
        for cam in cams[:: max(1, len(cams) // 8)][:8]:
            P.rd_preprocess(view, g, cam, opts)
            P.rd_bin(view)
            _, _, rng = P.rd_debug_binning(view)
            r = rng.cpu().numpy().astype(np.int64)
            lens.append(r[:, 1] - r[:, 0])
        L = np.concatenate(lens)
        q = np.percentile(L, [50, 90, 99, 99.9])
        print(f"{name}: tiles/view={len(lens[0])} mean={L.mean():.0f} p50/90/99/99.9={q.astype(int).tolist()} "
              f"max={L.max()} >1024={np.mean(L > 1024):.3f} >2048={np.mean(L > 2048):.3f} "
              f">4096={np.mean(L > 4096):.4f} >8192={np.mean(L > 8192):.4f} >16384={np.mean(L > 16384):.5f}",
              flush=True)


if __name__ == "__main__":
    main()
