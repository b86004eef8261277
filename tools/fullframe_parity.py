"""Full-frame parity at scale (SURVEY §8(d) "Parity at scale: C1 full frame"): one view of a
config rendered by the CUDA path (C-ABI, bench's 8×8 tiles) and by the fp64 oracle over EVERY
pixel, compared on every unflagged pixel (colour, normal, alpha ≤ 1e-4; depth ≤ 1e-4 where F4/F5
do not apply), the flagged share reported. Runs on the GPU box (the oracle on its host cores);
writes gpurun_out/fullframe_parity_<config>.json (kept under profiles/).

    python tools/fullframe_parity.py [C1] [view]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402

F1, F3, F4, F5 = 1, 4, 8, 16
TOL = 1e-4


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
    vi = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    scene, cams, opt = sg.config_scene_and_cameras(cfg)
    opt.tile = 8
    cam = cams[vi]
    g = P.Gaussians.from_numpy(scene)
    opts = {k: getattr(opt, k) for k in ("tile", "alpha_min", "alpha_max", "T_min", "median_T", "dilation", "bg",
                                          "sh_degree", "guard_band")}
    out, view = P.render(g, cam, opts)
    torch.cuda.synchronize()
    gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
    # bench.py's cpu_baseline extrapolates the oracle's forward from a random-pixel sample
    # (project+sort time + per-pixel time × W·H / n): the full frame below validates it
    rng = np.random.default_rng(0)
    n_s = 2048
    ts = np.zeros(3)
    oracle.render(scene, cam, opt, pixels=rng.choice(cam.width * cam.height, n_s, replace=False), timing=ts)
    extrap = ts[0] + ts[1] * (cam.width * cam.height / n_s)
    tf = np.zeros(3)
    t0 = time.time()
    ref = oracle.render(scene, cam, opt, timing=tf)
    t_or = time.time() - t0
    fl = ref["flags"]
    ok = (fl & (F1 | F3)) == 0
    okd = (fl & (F1 | F3 | F4 | F5)) == 0
    res = {"config": cfg, "view": vi, "width": cam.width, "height": cam.height, "gaussians": int(scene.n),
           "oracle_threads": oracle.num_threads(), "oracle_s": t_or,
           "cpu_baseline_check": {"sample_pixels": n_s, "extrapolated_full_frame_s": extrap,
                                  "full_frame_s": float(tf[0] + tf[1]),
                                  "ratio_extrapolated_over_full": extrap / float(tf[0] + tf[1])},
           "flagged_share_F1_F3": float(1 - ok.mean()), "flagged_share_depth": float(1 - okd.mean()),
           "alpha_mean": float(ref["alpha"].mean()), "tolerance": TOL}
    worst = {}
    for k in ("color", "normal"):
        worst[k] = float(np.abs(gpu[k] - ref[k])[:, ok].max())
    worst["alpha"] = float(np.abs(gpu["alpha"] - ref["alpha"])[ok].max())
    worst["depth"] = float(np.abs(gpu["depth"] - ref["depth"])[okd].max())
    res["max_abs_err"] = worst
    res["pass"] = all(v <= TOL for v in worst.values()) and res["flagged_share_F1_F3"] <= 0.01
    print(json.dumps(res), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)  # (gpurun brings gpurun_out/ back)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"fullframe_parity_{cfg}.json"), "w"), indent=1)
    return 0 if res["pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
