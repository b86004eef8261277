"""Validates bench.py's cpu_baseline extrapolation: the oracle's
forward on the FULL C3 frame (view 0, every pixel) against the extrapolation bench.py makes
from a random-pixel sample (project+sort time + per-pixel time × W·H / n_pix), and the
per-Gaussian dual-gradient cost at two sample sizes. Writes profiles/cpu_baseline_validation.json.

    OMP_NUM_THREADS=... python tools/validate_cpu_baseline.py [n_pix_sample]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import oracle
import scenegen as sg


def main():
    n_pix = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    scene, cams, opt = sg.config_scene_and_cameras("C3")
    cam = cams[0]
    W, H = cam.width, cam.height
    rng = np.random.default_rng(0)
    pix = rng.choice(W * H, n_pix, replace=False)
    ts = np.zeros(3)
    oracle.render(scene, cam, opt, pixels=pix, timing=ts)
    extrap = ts[0] + ts[1] * (W * H / n_pix)
    out = {"config": "C3 view 0 (1237x822, 1.5M Gaussians, guard band 0.15)", "threads": oracle.num_threads(),
           "sample_pixels": n_pix, "sample_project_sort_s": ts[0], "sample_pixel_loop_s": ts[1],
           "extrapolated_full_frame_s": extrap}
    print(json.dumps(out), flush=True)
    tf = np.zeros(3)
    t0 = time.time()
    full = oracle.render(scene, cam, opt, timing=tf)
    out.update({"full_frame_project_sort_s": tf[0], "full_frame_pixel_loop_s": tf[1],
                "full_frame_s": tf[0] + tf[1], "full_frame_wall_s": time.time() - t0,
                "ratio_extrapolated_over_full": extrap / (tf[0] + tf[1]),
                "full_frame_alpha_mean": float(full["alpha"].mean())})
    print(json.dumps(out), flush=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "cpu_baseline_validation.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
