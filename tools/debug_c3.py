"""Debug helper: backward determinism at C3 scale, and the worst sampled forward pixel."""
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
torch.cuda.synchronize()
H, W = cam.height, cam.width
gen = torch.Generator(device="cuda")
gen.manual_seed(6)
cot = torch.randn((8, H, W), generator=gen, device="cuda")
res = []
g2ds = []
for rep in range(3):
    gr = g.zeros_like()
    P.rd_render_bwd(view, g, cot[0:3], cot[3], cot[4:7], cot[7], gr)
    torch.cuda.synchronize()
    g2ds.append(P.rd_debug_grads2d(view).cpu().numpy())
    res.append(grads_to_rows(gr, g.n))
for sl, name in ((slice(0, 3), "means"), (slice(3, 6), "scales"), (slice(6, 10), "rot"), (slice(10, 11), "opac"),
                 (slice(11, 59), "sh")):
    print(name, "norm", np.linalg.norm(res[0][:, sl]), "d01", np.linalg.norm(res[0][:, sl] - res[1][:, sl]),
          "d02", np.linalg.norm(res[0][:, sl] - res[2][:, sl]))
for k in range(16):
    a, b = g2ds[0][:, k], g2ds[1][:, k]
    print("g2d", k, "norm", np.linalg.norm(a), "diff", np.linalg.norm(a - b), "maxabs", np.abs(a - b).max())
bad = np.nonzero(np.abs(res[0] - res[1]).max(1) > 1e-3 * (np.abs(res[0]).max(1) + 1e-6))[0]
print("rows differing", len(bad), bad[:10])
_, _, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
print("touched of bad", touched[bad[:10]])
for i in bad[:3]:
    print(i, res[0][i, :11], res[1][i, :11])
    print("  g2d", g2ds[0][i], g2ds[1][i])

# worst forward pixel
rng = np.random.default_rng(11)
pix = rng.choice(W * H, 48, replace=False)
ref = oracle.render(scene, cam, opt, pixels=pix)
gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
ys, xs = pix // W, pix % W
for k in ("color", "normal"):
    err = np.abs(gpu[k][:, ys, xs] - ref[k])
    j = np.argmax(err.max(0))
    print(k, "worst px", ys[j], xs[j], "err", err[:, j], "gpu", gpu[k][:, ys[j], xs[j]], "ref", ref[k][:, j],
          "flags", ref["flags"][j], "alpha", ref["alpha"][j], "nblend", ref["nblend"][j])
