"""Tiny forward+backward on C0 and a dense scene (used under RADE_SYNC_CHECK=1 / compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_01467_b200 as P  # noqa: E402
import scenegen as sg  # noqa: E402

for name, scene, cam in (("C0", sg.scene_c0(), sg.camera_c0()),
                         ("C1-small", sg.scene_c1(n=20000), sg.cameras_c1(2)[0])):
    g = P.Gaussians.from_numpy(scene)
    out, view = P.render(g, cam)
    grads = g.zeros_like()
    c = {k: torch.as_tensor(v).cuda() for k, v in sg.cotangents(0, cam.width, cam.height).items()}
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
    torch.cuda.synchronize()
    print(name, "ok M =", P.rd_view_stats(view)["n_duplicates"], float(out["alpha"].mean()))
