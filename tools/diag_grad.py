"""Diagnostics: per parity case, the worst elementwise gradient entries vs the oracle
(ratio of |Δg| to the bound 1e-3|g| + 1e-3 median|g|), with the Gaussian's footprint."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import oracle
import paper_2406_01467_b200 as P
import scenegen as sg
import test_gpu_parity as T
from gpu_helpers import gpu_grads

names = sys.argv[1:]
cases = [c for c in T.CASES if not names or c[0] in names]
for name, scene, cam, opt in cases:
    ref = oracle.render(scene, cam, opt)
    mask = ref["flags"] == 0
    cot = sg.cotangents(7, cam.width, cam.height)
    cot = {k: (v * mask).astype(np.float32) for k, v in cot.items()}
    _, G, view = gpu_grads(scene, cam, opt, cot)
    pg = oracle.project(scene, cam, opt)
    vis = np.nonzero(pg[:, 0] == 1)[0]
    R = oracle.grad(scene, cam, opt, cot, vis)
    _, _, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    for cname, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                      "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
        a, b = G[vis, sl], R[:, sl]
        med = np.median(np.abs(b[b != 0])) if (b != 0).any() else 0.0
        bound = 1e-3 * np.abs(b) + 1e-3 * med
        ratio = np.abs(a - b) / np.maximum(bound, 1e-300)
        k = np.argsort(-ratio.ravel())[:3]
        for kk in k:
            r, c = np.unravel_index(kk, ratio.shape)
            gid = vis[r]
            s = scene.scales[:, gid]
            print(f"{name:12s} {cname:9s} g{gid:4d} c{c} ratio {ratio[r, c]:8.3f} gpu {a[r, c]: .6e} "
                  f"orc {b[r, c]: .6e} med {med:.2e} touched {touched[gid]} flat {s.min() / s.max():.1e} "
                  f"ndotx {pg[gid, oracle.PG['ndotx']]:.3f} o {scene.opacities[gid]:.3f}", flush=True)
