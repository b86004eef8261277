"""Debug helper: re-blend one C3 pixel in fp64 from the GPU's own records and list, and
compare per-splat records with the oracle's projection of the same splats."""
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
from gpu_helpers import opts_dict  # noqa: E402

Y, X = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (817, 612)
scene, cams, opt = sg.config_scene_and_cameras("C3")
cam = cams[0]
g = P.Gaussians.from_numpy(scene)
out, view = P.render(g, cam, opts_dict(opt))
torch.cuda.synchronize()
gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(view))
T_, nc, mp = (t.cpu().numpy() for t in P.rd_debug_pixel_state(view))
tiles_x = (cam.width + 15) // 16
t = (Y // 16) * tiles_x + X // 16
lst = ids[ranges[t, 0]:ranges[t, 1]].view(np.uint32)
print("pixel", Y, X, "list", len(lst), "n_contrib", nc[Y, X], "median_pos", mp[Y, X])
pg = oracle.project(scene, cam, opt)
px, py = X + 0.5, Y + 0.5
T = 1.0
N = np.zeros(3)
C = np.zeros(3)
rows = []
for pos, gid in enumerate(lst[:nc[Y, X]]):
    r = rec[gid].astype(np.float64)
    lo = rec[gid, 15:16].copy().view(np.float16).astype(np.float64)
    dx = r[0] + lo[0] - px
    dy = r[1] + lo[1] - py
    e = r[2] * dx * dx + r[3] * dx * dy + r[4] * dy * dy + r[5]
    if e < np.log2(opt.alpha_min):
        continue
    a = min(opt.alpha_max, 2.0 ** e)
    w = a * T
    o = pg[gid]
    dn = np.abs(r[9:12] - o[67:70]).max()
    dc = np.abs(r[6:9] - o[oracle.PG["rgb"]]).max()
    rows.append((pos, gid, w, dn, dc, o[oracle.PG["ndotx"]], rect[gid], touched[gid]))
    N += w * r[9:12]
    C += w * r[6:9]
    T *= 1 - a
print("reblend N", N, "gpu N", gpu["normal"][:, Y, X])
print("reblend C", C, "gpu C", gpu["color"][:, Y, X])
ref = oracle.render(scene, cam, opt, pixels=np.array([Y * cam.width + X]))
print("oracle N", ref["normal"][:, 0], "C", ref["color"][:, 0], "flags", ref["flags"][0], "nblend", ref["nblend"][0])
rows.sort(key=lambda r: -r[2] * r[3])
for r in rows[:8]:
    print("pos %d gid %d w %.4g dnormal %.3g dcolor %.3g ndotx %.3g touched %d" % (r[0], r[1], r[2], r[3], r[4], r[5],
                                                                                    r[7]))
gid = rows[0][1]
print("scales", scene.scales[:, gid], "opacity", scene.opacities[gid])
print("gpu n", rec[gid, 9:12], "oracle n", pg[gid, 67:70])
