"""Debug helper: C3 sampled gradients, GPU vs oracle, for the test's candidate choice."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402
from gpu_helpers import grads_to_rows, opts_dict  # noqa: E402

scene, cams, opt = sg.config_scene_and_cameras("C3")
cam = cams[0]
g = P.Gaussians.from_numpy(scene)
out, view = P.render(g, cam, opts_dict(opt))
H, W = cam.height, cam.width
rng = np.random.default_rng(21)
cot = {"color": rng.normal(size=(3, H, W)).astype(np.float32), "depth": rng.normal(size=(H, W)).astype(np.float32),
       "normal": rng.normal(size=(3, H, W)).astype(np.float32), "alpha": rng.normal(size=(H, W)).astype(np.float32)}
c = {k: torch.as_tensor(v).cuda().contiguous() for k, v in cot.items()}
grads = g.zeros_like()
P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
torch.cuda.synchronize()
G = grads_to_rows(grads, g.n)
rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
g2 = P.rd_debug_grads2d(view).cpu().numpy()
small = np.nonzero((touched > 0) & (touched <= 4))[0]
vis = touched > 0
print("g2 nonzero rows (visible)", (np.abs(g2[vis]).sum(1) > 0).sum(), "col5 max", np.nanmax(np.abs(g2[vis, 5])),
      "nan", np.isnan(g2[vis]).sum(), "G nonzero rows", (np.abs(G).sum(1) > 0).sum())
print("small with nonzero G", (np.abs(G[small]).sum(1) > 0).sum())
print("visible", (touched > 0).sum(), "small", len(small), "big", (touched > 64).sum())
cand = small[np.argsort(-np.abs(g2[small, 5]))[:200]]
gids = rng.choice(cand, 6, replace=False)
print("gids", gids, "touched", touched[gids])
print("g2d rows", g2[gids][:, :12])
R = oracle.grad(scene, cam, opt, {k: v.astype(np.float64) for k, v in cot.items()}, gids)
for k, gid in enumerate(gids):
    print(gid, "gpu", np.round(G[gid, :11], 5))
    print(gid, "orc", np.round(R[k, :11], 5))
pg = oracle.project(scene.subset(gids), cam, opt)
print("oracle valid", pg[:, 0], "u", pg[:, 7], "v", pg[:, 8], "z", pg[:, 5], "o", pg[:, 76])
print("gpu u v", rec[gids, 0], rec[gids, 1], "z", rec[gids, 12])
