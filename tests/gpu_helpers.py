"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI and lay its
results out like the oracle's (numpy fp64)."""
import numpy as np
import torch

import paper_2406_01467_b200 as P


def opts_dict(opt):
    return dict(tile=opt.tile, alpha_min=opt.alpha_min, alpha_max=opt.alpha_max, T_min=opt.T_min,
                median_T=opt.median_T, dilation=opt.dilation, bg=opt.bg, sh_degree=opt.sh_degree,
                guard_band=opt.guard_band)


def gpu_forward(scene, cam, opt, view=None):
    g = P.Gaussians.from_numpy(scene)
    out, view = P.render(g, cam, opts_dict(opt), view=view)
    torch.cuda.synchronize()
    res = {k: v.double().cpu().numpy() for k, v in out.items()}
    return res, view, g


def gpu_grads(scene, cam, opt, cot):
    """Returns (forward outputs, grads laid out [N, 59] like oracle.grad, view)."""
    res, view, g = gpu_forward(scene, cam, opt)
    dev = torch.device("cuda")
    c = {k: torch.as_tensor(np.asarray(v, np.float32)).contiguous().to(dev) for k, v in cot.items()}
    grads = g.zeros_like()
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
    torch.cuda.synchronize()
    return res, grads_to_rows(grads, scene.n), view


def grads_to_rows(grads, n):
    G = np.zeros((n, 59))
    G[:, 0:3] = grads.means.double().cpu().numpy()
    G[:, 3:6] = grads.scales.double().cpu().numpy()
    G[:, 6:10] = grads.rotations.double().cpu().numpy()
    G[:, 10] = grads.opacities.double().cpu().numpy()
    sh = grads.sh.double().cpu().numpy()  # [N, K, 3]
    K = sh.shape[1]
    G[:, 11:11 + 3 * K] = sh.reshape(n, 3 * K)
    return G


def cpu_binning_reference(rect, touched, zkey, tiles_x):
    """Keys built in Gaussian-id order from the GPU's own rect and z_key, then
    std::stable_sort-equivalent (numpy stable argsort) — SURVEY §8(c) binning pin."""
    keys, ids = [], []
    zb = zkey.astype(np.float32).view(np.uint32).astype(np.uint64)
    for i in np.nonzero(touched)[0]:
        r0, r1 = int(rect[i, 0]) & 0xFFFFFFFF, int(rect[i, 1]) & 0xFFFFFFFF
        x0, y0, x1, y1 = r0 & 0xFFFF, r0 >> 16, r1 & 0xFFFF, r1 >> 16
        for ty in range(y0, y1):
            for tx in range(x0, x1):
                keys.append((np.uint64(ty * tiles_x + tx) << np.uint64(32)) | zb[i])
                ids.append(i)
    keys = np.array(keys, dtype=np.uint64)
    ids = np.array(ids, dtype=np.uint32)
    order = np.argsort(keys, kind="stable")
    return keys[order], ids[order]
