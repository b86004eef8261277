"""Workload for compute-sanitizer (racecheck / synccheck / memcheck / initcheck): the whole hot
path through the C ABI — K1, the binning sorts, K3 (with and without the L_d sums), K4
(blend mask, shared-memory warp reduction, direct atomics), K5a/K5b/K5b64, L_n forward and
backward — on C0 and on a small NeRF-Synthetic-shaped slice (C1 recipe, 20k Gaussians,
800×800, two views), at tile 8 and tile 16. No oracle: this only drives the kernels.

    compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch

import paper_2406_01467_b200 as P
import scenegen as sg


def run(scene, cams, opt, tile):
    g = P.Gaussians.from_numpy(scene)
    grads = g.zeros_like()
    opts = dict(tile=tile, alpha_min=opt.alpha_min, alpha_max=opt.alpha_max, T_min=opt.T_min,
                median_T=opt.median_T, dilation=opt.dilation, bg=opt.bg, sh_degree=opt.sh_degree,
                guard_band=opt.guard_band)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    for k, cam in enumerate(cams):
        H, W = cam.height, cam.width
        cot = torch.randn((9, H, W), generator=gen, device="cuda")
        view = P.View()
        P.rd_preprocess(view, g, cam, opts)
        P.rd_bin(view)
        maps = torch.empty((8, H, W), device="cuda")
        out = dict(color=maps[0:3], depth=maps[3], normal=maps[4:7], alpha=maps[7])
        if k % 2 == 0:
            P.rd_render_fwd_ex(view, out["color"], out["depth"], out["normal"], out["alpha"], distortion=True)
            P.rd_blend_bwd_ex(view, cot[0:3], cot[3], cot[4:7], cot[7], cot[8])
        else:
            P.rd_render_fwd_ex(view, out["color"], out["depth"], out["normal"], out["alpha"])
            P.rd_blend_bwd(view, cot[0:3], cot[3], cot[4:7], cot[7])
        P.rd_preprocess_bwd(view, g, grads)
        Ln, nt = P.rd_normal_consistency(cam, out["depth"], out["alpha"], out["normal"], consistency=True,
                                         depth_normal=True)
        gD, gA, gN = torch.zeros_like(out["depth"]), torch.zeros_like(out["alpha"]), torch.zeros_like(out["normal"])
        P.rd_normal_consistency_bwd(cam, out["depth"], out["normal"], cot[8], gD, gA, gN)
        torch.cuda.synchronize()
        view.close()
    return float(grads.means.abs().sum())


def main():
    torch.cuda.set_device(0)
    c0 = (sg.scene_c0(), [sg.camera_c0()], sg.Options())
    s1, cams1, o1 = sg.config_scene_and_cameras("C1", n_gaussians=20_000)
    for tile in (8, 16):
        for scene, cams, opt in (c0, (s1, cams1[:2], o1)):
            v = run(scene, cams, opt, tile)
            print(f"tile {tile} n {scene.n} views {len(cams)}: |dL/dmu| = {v:.4e}", flush=True)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
