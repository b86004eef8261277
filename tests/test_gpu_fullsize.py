"""GPU parity at BASELINE.json's full size, in the launch configuration bench.py times
(C3: 1.5M Gaussians, 1237x822, 8x8 tiles, the views of a step pipelined over one CUDA
stream and one host thread each, their gradient accumulations concurrent).

The oracle cannot render 1M pixels x 1.5M Gaussians in a test, so it is compared on
sampled outputs it computes one by one (random pixels; the gradients of sampled visible
Gaussians), and the binning is checked bit-exactly against a vectorised stable sort of the
64-bit keys built from the GPU's own rects and depth keys."""
import numpy as np
import pytest
import torch

import oracle
import paper_2406_01467_b200 as P
import scenegen as sg
from gpu_helpers import grads_to_rows, opts_dict

pytestmark = pytest.mark.gpu

F1, F3, F4, F5 = 1, 4, 8, 16
TOL = 1e-4


BENCH_TILE = 8  # bench.py's default blend tile


@pytest.fixture(scope="module")
def c3():
    scene, cams, opt = sg.config_scene_and_cameras("C3")
    opt.tile = BENCH_TILE
    cam = cams[0]
    g = P.Gaussians.from_numpy(scene)
    out, view = P.render(g, cam, opts_dict(opt))
    torch.cuda.synchronize()
    gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
    return dict(scene=scene, cams=cams, cam=cam, opt=opt, g=g, view=view, gpu=gpu)


def test_c3_forward_sampled_pixels(c3):
    cam = c3["cam"]
    rng = np.random.default_rng(11)
    pix = rng.choice(cam.width * cam.height, 48, replace=False)
    ref = oracle.render(c3["scene"], cam, c3["opt"], pixels=pix)
    ys, xs = pix // cam.width, pix % cam.width
    gpu = c3["gpu"]
    fl = ref["flags"]
    ok = (fl & (F1 | F3)) == 0
    assert (~ok).sum() <= max(1, 0.01 * len(pix)), (~ok).sum()  # flagged ≤ 1%
    assert (ref["alpha"] > 0.5).mean() > 0.3  # the sample hits the scene
    for k in ("color", "normal"):
        err = np.abs(gpu[k][:, ys, xs] - ref[k])[:, ok]
        assert err.max() <= TOL, (k, err.max())
    err = np.abs(gpu["alpha"][ys, xs] - ref["alpha"])[ok]
    assert err.max() <= TOL, ("alpha", err.max())
    okd = (fl & (F1 | F3 | F4 | F5)) == 0
    err = np.abs(gpu["depth"][ys, xs] - ref["depth"])[okd]
    assert err.max() <= TOL, ("depth", err.max())


def _binning_reference(rect, touched, zkey, tiles_x):
    """Vectorised: keys (tile << 32 | float_bits(z_c)) over the (Gaussian, tile) pairs in id
    order, row-major over each rect, then a stable sort."""
    ids = np.nonzero(touched)[0]
    r0 = rect[ids, 0].astype(np.int64) & 0xFFFFFFFF
    r1 = rect[ids, 1].astype(np.int64) & 0xFFFFFFFF
    x0, y0, x1, y1 = r0 & 0xFFFF, r0 >> 16, r1 & 0xFFFF, r1 >> 16
    w = x1 - x0
    cnt = w * (y1 - y0)
    assert np.array_equal(cnt, touched[ids].astype(np.int64))
    rep = np.repeat(np.arange(len(ids)), cnt)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    li = np.arange(cnt.sum()) - start[rep]
    ty = y0[rep] + li // w[rep]
    tx = x0[rep] + li % w[rep]
    zb = zkey.astype(np.float32).view(np.uint32).astype(np.uint64)
    keys = ((ty * tiles_x + tx).astype(np.uint64) << np.uint64(32)) | zb[ids[rep]]
    order = np.argsort(keys, kind="stable")
    return keys[order], ids[rep][order].astype(np.uint32)


def test_c3_zkey_bits_match_oracle(c3):
    """The sort key (reading S7) of every visible Gaussian at C3, bit for bit against the
    oracle's fp32 z_key; and every Gaussian the GPU keeps is one the oracle keeps."""
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(c3["view"]))
    pg = oracle.project(c3["scene"], c3["cam"], c3["opt"])
    vis = touched > 0
    assert vis.sum() > 500_000 and np.all(pg[vis, 0] == 1)
    zg = np.ascontiguousarray(rec[vis][:, 12]).view(np.uint32)
    zo = pg[vis, oracle.PG["zkey"]].astype(np.float32).view(np.uint32)
    np.testing.assert_array_equal(zg, zo)


def test_c3_binning_bit_exact(c3):
    view = c3["view"]
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(view))
    st = P.rd_view_stats(view)
    rk, ri = _binning_reference(rect, touched, rec[:, 12], st["tiles_x"])
    assert st["n_duplicates"] == len(rk) > 1_000_000
    np.testing.assert_array_equal(keys.view(np.uint64), rk)
    np.testing.assert_array_equal(ids.view(np.uint32), ri)
    T = st["tiles_x"] * st["tiles_y"]
    tiles = (rk >> np.uint64(32)).astype(np.int64)
    first = np.searchsorted(tiles, np.arange(T), side="left")
    last = np.searchsorted(tiles, np.arange(T), side="right")
    exp = np.where((last > first)[:, None], np.stack([first, last], 1), 0)
    np.testing.assert_array_equal(ranges.astype(np.int64), exp)


def _pipelined_grads(g, cams, opt, cots, n_streams, host_threads=False):
    """bench.py's launch configuration: views over n_streams streams (each issued by its own
    host thread when host_threads), every view's K4 and K5 free to overlap the others' (K5
    accumulates with L2 reductions)."""
    import threading
    dev = torch.device("cuda", torch.cuda.current_device())
    grads = g.zeros_like()
    slots = []
    for _ in range(n_streams):
        st = torch.cuda.Stream(dev)
        with torch.cuda.stream(st):
            slots.append((st, P.View(dev)))
    start = torch.cuda.Event()
    start.record()
    for st, _ in slots:
        st.wait_event(start)

    def one(k):
        st, vw = slots[k % n_streams]
        cam, cot = cams[k], cots[k]
        with torch.cuda.stream(st):
            P.rd_preprocess(vw, g, cam, opts_dict(opt), stream=st)
            P.rd_bin(vw, stream=st)
            P.rd_render_fwd(vw, stream=st)
            P.rd_blend_bwd(vw, cot[0:3], cot[3], cot[4:7], cot[7], stream=st)
            P.rd_preprocess_bwd(vw, g, grads, stream=st)

    def worker(si):
        torch.cuda.set_device(dev)
        for k in range(si, len(cams), n_streams):
            one(k)

    if host_threads:
        errs = []

        def guarded(si):
            try:
                worker(si)
            except BaseException as e:  # surfaced below: a dead thread must fail the test
                errs.append(e)

        ths = [threading.Thread(target=guarded, args=(si,)) for si in range(n_streams)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errs, errs
    else:
        for k in range(len(cams)):
            one(k)
    for st, _ in slots:
        torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    return grads_to_rows(grads, g.n)


@pytest.mark.parametrize("n_streams,host_threads", [(2, False), (4, True)])
def test_c3_pipelined_accumulation_matches_sequential(c3, n_streams, host_threads):
    """Four views accumulated through pipelined streams (bench.py's default: one stream and
    one host thread per view of the step) equal the sequential sum (float atomics in K4:
    equal to rounding)."""
    H, W = c3["cam"].height, c3["cam"].width
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    cots = [torch.randn((8, H, W), generator=gen, device="cuda") for _ in range(4)]
    cams = c3["cams"][:4]
    a = _pipelined_grads(c3["g"], cams, c3["opt"], cots, n_streams, host_threads)
    b = _pipelined_grads(c3["g"], cams, c3["opt"], cots, 1)
    for sl in (slice(0, 3), slice(3, 6), slice(6, 10), slice(10, 11), slice(11, 59)):
        nb = np.linalg.norm(b[:, sl])
        assert nb > 0
        assert np.linalg.norm(a[:, sl] - b[:, sl]) <= 1e-5 * nb, sl


def test_c3_split_backward_equals_render_bwd(c3):
    H, W = c3["cam"].height, c3["cam"].width
    gen = torch.Generator(device="cuda")
    gen.manual_seed(6)
    cot = torch.randn((8, H, W), generator=gen, device="cuda")
    g, view = c3["g"], c3["view"]
    ga, gb = g.zeros_like(), g.zeros_like()
    P.rd_render_bwd(view, g, cot[0:3], cot[3], cot[4:7], cot[7], ga)
    P.rd_blend_bwd(view, cot[0:3], cot[3], cot[4:7], cot[7])
    P.rd_preprocess_bwd(view, g, gb)
    torch.cuda.synchronize()
    a, b = grads_to_rows(ga, g.n), grads_to_rows(gb, g.n)
    assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)


def test_c3_sampled_gradients(c3):
    """dL/dθ of sampled visible Gaussians against the oracle's exact (dual-number)
    gradients, L = Σ cot·(C, D, N, A) over the full frame."""
    scene, cam, opt, g, view = c3["scene"], c3["cam"], c3["opt"], c3["g"], c3["view"]
    H, W = cam.height, cam.width
    rng = np.random.default_rng(21)
    cot = {"color": rng.normal(size=(3, H, W)).astype(np.float32),
           "depth": rng.normal(size=(H, W)).astype(np.float32),
           "normal": rng.normal(size=(3, H, W)).astype(np.float32),
           "alpha": rng.normal(size=(H, W)).astype(np.float32)}
    c = {k: torch.as_tensor(v).cuda().contiguous() for k, v in cot.items()}
    grads = g.zeros_like()
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
    torch.cuda.synchronize()
    G = grads_to_rows(grads, g.n)
    _, _, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    # contributing Gaussians (largest opacity gradient) of three footprint classes (the
    # oracle's cost is per covered pixel): small (≤ 4 tiles), medium (16–64 tiles) and big
    # (tile rect > 16 384 px: the fp64 chain rule K5b64)
    t64 = touched.astype(np.int64)
    groups = {"small": ((t64 > 0) & (t64 <= 4), 6), "medium": ((t64 >= 16) & (t64 <= 64), 4),
              "big": (t64 * opt.tile ** 2 > 16384, 2)}
    assert P.rd_view_stats(view)["n_big"] == int(groups["big"][0].sum()) > 0
    for gname, (sel, k) in groups.items():
        ids = np.nonzero(sel)[0]
        if gname == "big":  # the smallest big ones (the oracle walks every covered pixel)
            ids = ids[np.argsort(t64[ids])[:40]]
        cand = ids[np.argsort(-np.abs(G[ids, 10]))[:200]]
        gids = rng.choice(cand, k, replace=False)
        R = oracle.grad(scene, cam, opt, {k_: v.astype(np.float64) for k_, v in cot.items()}, gids)
        A = G[gids]
        for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                         "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
            nb = np.linalg.norm(R[:, sl])
            assert nb > 0, (gname, name)
            rel = np.linalg.norm(A[:, sl] - R[:, sl]) / nb
            assert rel <= 1e-3, (gname, name, rel)


def test_c3_distortion_sampled_pixels(c3):
    """NEXT-1 at full size: the depth-distortion map (S21) at 48 random pixels vs the oracle."""
    cam, g = c3["cam"], c3["g"]
    view = P.View()
    P.rd_preprocess(view, g, cam, opts_dict(c3["opt"]))
    P.rd_bin(view)
    L = P.rd_render_fwd_ex(view, distortion=True)["distortion"]
    torch.cuda.synchronize()
    L = L.double().cpu().numpy()
    rng = np.random.default_rng(12)
    pix = rng.choice(cam.width * cam.height, 48, replace=False)
    ref = oracle.render(c3["scene"], cam, c3["opt"], pixels=pix)
    ys, xs = pix // cam.width, pix % cam.width
    ok = (ref["flags"] & (F1 | F3)) == 0
    assert (~ok).sum() <= max(1, 0.01 * len(pix)) and ref["distortion"].max() > 1e-3
    err = np.abs(L[ys, xs] - ref["distortion"])[ok]
    assert err.max() <= TOL * max(1.0, np.abs(ref["distortion"][ok]).max()), err.max()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_other_configs_forward_sampled_pixels(cfg):
    """The other BASELINE.json configurations at full size (C1 800×800 300k with a white
    background, C2 1600×1200 400k, C4 1237×822 3M): 32 random pixels of view 0 vs the
    oracle."""
    scene, cams, opt = sg.config_scene_and_cameras(cfg)
    opt.tile = BENCH_TILE
    cam = cams[0]
    g = P.Gaussians.from_numpy(scene)
    out, _ = P.render(g, cam, opts_dict(opt))
    torch.cuda.synchronize()
    gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
    rng = np.random.default_rng(13)
    pix = rng.choice(cam.width * cam.height, 32, replace=False)
    ref = oracle.render(scene, cam, opt, pixels=pix)
    ys, xs = pix // cam.width, pix % cam.width
    ok = (ref["flags"] & (F1 | F3)) == 0
    assert (~ok).sum() <= max(1, 0.01 * len(pix))
    for k in ("color", "normal"):
        assert np.abs(gpu[k][:, ys, xs] - ref[k])[:, ok].max() <= TOL, (cfg, k)
    assert np.abs(gpu["alpha"][ys, xs] - ref["alpha"])[ok].max() <= TOL
    okd = (ref["flags"] & (F1 | F3 | F4 | F5)) == 0
    assert np.abs(gpu["depth"][ys, xs] - ref["depth"])[okd].max() <= TOL


def test_c3_guard_band_off_sampled_pixels(c3):
    """C3 with the guard band of reading S6b off (the ABI default): 48 random
    pixels vs the oracle with the same option; the near-camera ground splats then reach
    into the image (the band changes the image: checked, not assumed)."""
    cam = c3["cam"]
    opt = sg.Options(tile=BENCH_TILE, guard_band=0.0)
    out, view = P.render(c3["g"], cam, opts_dict(opt))
    torch.cuda.synchronize()
    gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
    assert P.rd_view_stats(view)["n_visible"] > P.rd_view_stats(c3["view"])["n_visible"]
    rng = np.random.default_rng(14)
    pix = rng.choice(cam.width * cam.height, 48, replace=False)
    ref = oracle.render(c3["scene"], cam, opt, pixels=pix)
    ys, xs = pix // cam.width, pix % cam.width
    ok = (ref["flags"] & (F1 | F3)) == 0
    assert (~ok).sum() <= max(1, 0.01 * len(pix))
    for k in ("color", "normal"):
        assert np.abs(gpu[k][:, ys, xs] - ref[k])[:, ok].max() <= TOL, k
    assert np.abs(gpu["alpha"][ys, xs] - ref["alpha"])[ok].max() <= TOL
    okd = (ref["flags"] & (F1 | F3 | F4 | F5)) == 0
    assert np.abs(gpu["depth"][ys, xs] - ref["depth"])[okd].max() <= TOL
    assert np.abs(gpu["color"] - c3["gpu"]["color"]).max() > 1e-2


def test_c3_batched_k5_equals_per_view_sum(c3):
    """bench.py's default K5 (rd_preprocess_bwd_views over the 4 views of a step) equals the
    per-view rd_preprocess_bwd sum at C3 to fp32 rounding, every parameter class."""
    g, opt = c3["g"], c3["opt"]
    H, W = c3["cam"].height, c3["cam"].width
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    views = []
    for cam in c3["cams"][:4]:
        cot = torch.randn((8, H, W), generator=gen, device="cuda")
        v = P.View()
        P.rd_preprocess(v, g, cam, opts_dict(opt))
        P.rd_bin(v)
        P.rd_render_fwd(v)
        P.rd_blend_bwd(v, cot[0:3], cot[3], cot[4:7], cot[7])
        views.append(v)
    assert sum(P.rd_view_stats(v)["n_big"] for v in views) > 0
    ga, gb, gc = g.zeros_like(), g.zeros_like(), g.zeros_like()
    P.rd_preprocess_bwd_views(views, g, ga)
    for v in views:
        P.rd_preprocess_bwd(v, g, gb)
    for v in views:  # bench --k5 split: geometry per view, then the round's SH part
        P.rd_preprocess_bwd_geometry(v, g, gc)
    P.rd_preprocess_bwd_views_sh(views, g, gc)
    gs = g.zeros_like()  # bench --k5 set: SH rows set (garbage before), the rest accumulated
    gs.sh.fill_(-7.0)
    P.rd_preprocess_bwd_views_ex(views, g, gs, flags=P.rade.RD_K5_SET_SH)
    torch.cuda.synchronize()
    assert torch.equal(gs.sh, ga.sh)
    a, b, c = grads_to_rows(ga, g.n), grads_to_rows(gb, g.n), grads_to_rows(gc, g.n)
    for sl in (slice(0, 3), slice(3, 6), slice(6, 10), slice(10, 11), slice(11, 59)):
        nb = np.linalg.norm(b[:, sl])
        assert nb > 0
        assert np.linalg.norm(a[:, sl] - b[:, sl]) <= 1e-5 * nb, sl
        assert np.linalg.norm(c[:, sl] - b[:, sl]) <= 1e-5 * nb, sl


def _sampled_grad_check(scene, cam, opt, g, view, cot, rng, groups, label):
    """GPU gradients of the sampled Gaussians (per footprint group) vs the oracle's exact dual
    numbers over the full frame; ≤ 1e-3 relative per parameter class."""
    c = {k: torch.as_tensor(v).cuda().contiguous() for k, v in cot.items() if k != "distortion"}
    grads = g.zeros_like()
    if "distortion" in cot:
        P.rd_blend_bwd_ex(view, c["color"], c["depth"], c["normal"], c["alpha"],
                          torch.as_tensor(cot["distortion"]).cuda().contiguous())
        P.rd_preprocess_bwd(view, g, grads)
    else:
        P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
    torch.cuda.synchronize()
    G = grads_to_rows(grads, g.n)
    _, _, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    t64 = touched.astype(np.int64)
    for gname, (lo, hi, k) in groups.items():
        ids = np.nonzero((t64 >= lo) & (t64 <= hi))[0]
        cand = ids[np.argsort(-np.abs(G[ids, 10]))[:200]]
        gids = rng.choice(cand, k, replace=False)
        R = oracle.grad(scene, cam, opt, {k_: v.astype(np.float64) for k_, v in cot.items()}, gids)
        for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                         "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
            nb = np.linalg.norm(R[:, sl])
            assert nb > 0, (label, gname, name)
            rel = np.linalg.norm(G[gids, sl] - R[:, sl]) / nb
            assert rel <= 1e-3, (label, gname, name, rel)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_other_configs_sampled_gradients(cfg):
    """Gradients at the other BASELINE.json configurations (full size, bench tile): small
    and medium Gaussians sampled among the contributing ones vs the oracle."""
    scene, cams, opt = sg.config_scene_and_cameras(cfg)
    opt.tile = BENCH_TILE
    cam = cams[0]
    g = P.Gaussians.from_numpy(scene)
    _, view = P.render(g, cam, opts_dict(opt))
    rng = np.random.default_rng(31)
    H, W = cam.height, cam.width
    cot = {"color": rng.normal(size=(3, H, W)).astype(np.float32), "depth": rng.normal(size=(H, W)).astype(np.float32),
           "normal": rng.normal(size=(3, H, W)).astype(np.float32), "alpha": rng.normal(size=(H, W)).astype(np.float32)}
    _sampled_grad_check(scene, cam, opt, g, view, cot, rng, {"small": (1, 4, 3), "medium": (16, 64, 2)}, cfg)


def test_c3_distortion_sampled_gradients(c3):
    """NEXT-1 at full size: gradients of Σ g·(C, D, N, A, L_d) (ω detached in L_d, S21) of
    sampled C3 Gaussians vs the oracle."""
    scene, cam, opt, g = c3["scene"], c3["cam"], c3["opt"], c3["g"]
    view = P.View()
    P.rd_preprocess(view, g, cam, opts_dict(opt))
    P.rd_bin(view)
    P.rd_render_fwd_ex(view, distortion=True)
    rng = np.random.default_rng(32)
    H, W = cam.height, cam.width
    cot = {"color": rng.normal(size=(3, H, W)).astype(np.float32), "depth": rng.normal(size=(H, W)).astype(np.float32),
           "normal": rng.normal(size=(3, H, W)).astype(np.float32), "alpha": rng.normal(size=(H, W)).astype(np.float32),
           "distortion": (10.0 * rng.normal(size=(H, W))).astype(np.float32)}
    _sampled_grad_check(scene, cam, opt, g, view, cot, rng, {"small": (1, 4, 3), "medium": (16, 64, 2)}, "C3+L_d")


def test_c3_normal_consistency_crop(c3):
    """NEXT-2 at full size: L_n and ñ of the C3 maps (GPU kernel on the full 1237×822 maps) vs
    the oracle's numpy definition on a 96×96 crop of the same maps (interior pixels; stencils
    of ambiguous orientation excluded as in the small-case test)."""
    gpu = c3["gpu"]
    cam = c3["cam"]
    dev = torch.device("cuda")
    t = {k: torch.as_tensor(np.asarray(gpu[k], np.float32)).contiguous().to(dev) for k in ("depth", "alpha", "normal")}
    L, nt = P.rd_normal_consistency(cam, t["depth"], t["alpha"], t["normal"], consistency=True, depth_normal=True)
    torch.cuda.synchronize()
    y0, x0, S = 360, 560, 96
    crop = lambda a: a[..., y0:y0 + S + 1, x0:x0 + S + 1].astype(np.float32).astype(np.float64)
    import copy
    cc = copy.copy(cam)
    cc.cx, cc.cy, cc.width, cc.height = cam.cx - x0, cam.cy - y0, S + 1, S + 1
    Lr, ntr = oracle.normal_consistency(crop(gpu["depth"]), crop(gpu["alpha"]), crop(gpu["normal"]), cc)
    Lg = L.cpu().numpy()[y0:y0 + S, x0:x0 + S]
    ng = nt.cpu().numpy()[:, y0:y0 + S, x0:x0 + S]
    Lr, ntr = Lr[:S, :S], ntr[:, :S, :S]
    xs = (np.arange(S) + 0.5 - cc.cx) / cam.fx
    ys = (np.arange(S) + 0.5 - cc.cy) / cam.fy
    ray = np.stack([np.broadcast_to(xs[None, :], (S, S)), np.broadcast_to(ys[:, None], (S, S)), np.ones((S, S))], 0)
    cosang = np.abs(np.sum(ntr * ray, 0)) / np.linalg.norm(ray, axis=0)
    valid = np.any(ntr != 0, 0)
    ok = ~valid | (cosang > 1e-3)
    assert valid.sum() > 1000
    np.testing.assert_allclose(ng[:, ok], ntr[:, ok], atol=1e-4)
    np.testing.assert_allclose(Lg[ok], Lr[ok], atol=1e-4)
