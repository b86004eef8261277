"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical
seeded scenes. Tolerances are the north star's (BASELINE.json): colour, depth, normal
(and alpha) within 1e-4 absolute; gradients within 1e-3 relative; binning bit-exact.
Pixels whose result is decided by a discrete threshold the two precisions can take
differently are excluded by the oracle's ambiguity flags."""
import numpy as np
import pytest
import torch

import oracle
import paper_2406_01467_b200 as P
import scenegen as sg
from gpu_helpers import cpu_binning_reference, gpu_forward, gpu_grads, grads_to_rows, opts_dict
from helpers import concat, dense_scene, one_gaussian, random_cam

pytestmark = pytest.mark.gpu

F1, F2, F3, F4, F5 = 1, 2, 4, 8, 16
TOL = 1e-4


def _scenes():
    rng = np.random.default_rng(42)
    cases = [("C0", sg.scene_c0(), sg.camera_c0(), sg.Options()),
             ("dense400", dense_scene(1, 400), sg.camera_identity(64, 64, 64), sg.Options()),
             ("dense400_t8", dense_scene(1, 400), sg.camera_identity(64, 64, 64), sg.Options(tile=8)),
             ("ragged_t32", dense_scene(2, 300, width=83, height=61, f=70.0), sg.camera_identity(83, 61, 70.0),
              sg.Options(tile=32, bg=(0.2, 0.5, 1.0))),
             ("ragged", dense_scene(2, 300, width=83, height=61, f=70.0), sg.camera_identity(83, 61, 70.0),
              sg.Options(bg=(0.2, 0.5, 1.0))),
             ("deg1", dense_scene(3, 200), sg.camera_identity(64, 64, 64), sg.Options(sh_degree=1)),
             ("deg0", dense_scene(4, 200), sg.camera_identity(64, 64, 64), sg.Options(sh_degree=0))]
    sc = dense_scene(5, 500, zr=(1.5, 4.0))
    cases.append(("lookat", sc, _lookat_cam(rng, 96, 72), sg.Options()))
    # ties (reading S7): with the identity camera z_key = z exactly, and z takes 3 values, so
    # most pairs of overlapping splats tie on depth and are ordered by id
    tie = dense_scene(6, 300)
    z_new = np.random.default_rng(6).choice([2.5, 3.0, 4.0], tie.n).astype(np.float32)
    tie.means[:2] *= z_new / tie.means[2]
    tie.means[2] = z_new
    cases.append(("ties_t8", tie, sg.camera_identity(64, 64, 64), sg.Options(tile=8)))
    # centres off screen beside the camera (reading S6b): band off (default) and on
    off = _offscreen_scene(7)
    cases.append(("offscreen", off, sg.camera_identity(64, 64, 64), sg.Options()))
    cases.append(("offscreen_gb", off, sg.camera_identity(64, 64, 64), sg.Options(guard_band=0.15)))
    return cases


def _offscreen_scene(seed, n_side=16):
    """dense_scene plus wide splats whose centres project 0.2–0.6 image widths outside the
    image at small depth (z ∈ [0.5, 1.2]): with the guard band off their affine footprints
    reach into the image, with it on (g = 0.15) they are culled."""
    rng = np.random.default_rng(seed)
    base = dense_scene(seed, 200)
    z = rng.uniform(0.5, 1.2, n_side)
    u = np.where(rng.random(n_side) < 0.5, rng.uniform(-0.6, -0.2, n_side), rng.uniform(1.2, 1.6, n_side)) * 64
    v = rng.uniform(0.1, 0.9, n_side) * 64
    swap = rng.random(n_side) < 0.3
    u[swap], v[swap] = v[swap], u[swap]
    x, y = (u - 32) * z / 64, (v - 32) * z / 64
    s = np.exp(rng.uniform(np.log(0.05), np.log(0.2), (3, n_side)))
    side = sg.make_scene(np.stack([x, y, z]), s, sg.random_quaternions(rng, n_side),
                         rng.uniform(0.05, 0.5, n_side), sg.sh_coeffs(rng, n_side))
    return concat(base, side)


def _lookat_cam(rng, W, H):
    R, t = sg.look_at([0.3, -0.2, -0.5], [0.0, 0.0, 3.0], up=(0, -1, 0))
    return sg.Camera(80.0, 82.0, W / 2 + 1.3, H / 2 - 0.7, W, H, R, t, 0.2)


CASES = _scenes()


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    name, scene, cam, opt = request.param
    ref = oracle.render(scene, cam, opt)
    gpu, view, g = gpu_forward(scene, cam, opt)
    return dict(name=name, scene=scene, cam=cam, opt=opt, ref=ref, gpu=gpu, view=view, g=g)


def test_forward_parity(case):
    ref, gpu = case["ref"], case["gpu"]
    fl = ref["flags"]
    ok = (fl & (F1 | F3)) == 0
    assert ok.mean() >= 0.99, ok.mean()  # flagged pixels ≤ 1%
    for k in ("color", "normal"):
        err = np.abs(gpu[k] - ref[k])[:, ok]
        assert err.max() <= TOL, (k, err.max())
    err = np.abs(gpu["alpha"] - ref["alpha"])[ok]
    assert err.max() <= TOL, ("alpha", err.max())
    okd = (fl & (F1 | F3 | F4 | F5)) == 0
    err = np.abs(gpu["depth"] - ref["depth"])[okd]
    assert err.max() <= TOL, ("depth", err.max())
    assert (ref["depth"] > 0).sum() > 10 or case["name"] == "C0"


def test_pixel_state_matches_oracle(case):
    """n_contrib / median position: the median splat the GPU selects is the oracle's."""
    T, nc, mp = (t.cpu().numpy() for t in P.rd_debug_pixel_state(case["view"]))
    ref = case["ref"]
    ok = (ref["flags"] & (F1 | F3 | F4)) == 0
    np.testing.assert_allclose(1.0 - T[ok], ref["alpha"][ok], atol=TOL)
    keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(case["view"]))
    tile = case["opt"].tile
    tiles_x = (case["cam"].width + tile - 1) // tile
    H, W = T.shape
    ys, xs = np.nonzero(ok & (mp >= 0))
    for y, x in zip(ys, xs):
        t = (y // tile) * tiles_x + x // tile
        gid = ids[ranges[t, 0] + mp[y, x]]
        assert gid == ref["median_id"][y, x]
    assert ((mp >= 0) == (ref["median_id"] >= 0))[ok].all()


def test_preprocess_parity(case):
    scene, cam, opt = case["scene"], case["cam"], case["opt"]
    pg = oracle.project(scene, cam, opt)
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(case["view"]))
    vis = touched > 0
    assert np.all(pg[vis, 0] == 1), "GPU kept a Gaussian the oracle culls"
    r = rec[vis].astype(np.float64)
    o = pg[vis]
    np.testing.assert_allclose(r[:, 0], o[:, oracle.PG["u"]], rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(r[:, 1], o[:, oracle.PG["v"]], rtol=1e-5, atol=1e-4)
    # (log2e/2)·conic = UᵀU with U = [[g11, g21], [0, g22]] = (r2, r3, r4)
    L = 1.4426950408889634 / 2
    conic = np.stack([r[:, 2] ** 2, r[:, 2] * r[:, 3], r[:, 3] ** 2 + r[:, 4] ** 2], 1) / L
    np.testing.assert_allclose(conic, o[:, oracle.PG["conic"]], rtol=2e-4, atol=1e-7)
    np.testing.assert_allclose(np.exp2(r[:, 5]), o[:, oracle.PG["o"]], rtol=1e-6)  # log2 o
    # centre = fp32 + half remainder (r3.w): accurate far below the fp32 ulp of u (~6e-5 px)
    lo = rec[vis][:, 15].copy().view(np.float16).astype(np.float64).reshape(-1, 2)
    np.testing.assert_allclose(r[:, 0] + lo[:, 0], o[:, oracle.PG["u"]], rtol=0, atol=2e-6)
    np.testing.assert_allclose(r[:, 1] + lo[:, 1], o[:, oracle.PG["v"]], rtol=0, atol=2e-6)
    np.testing.assert_allclose(r[:, 6:9], o[:, oracle.PG["rgb"]], atol=1e-5)
    np.testing.assert_allclose(r[:, 12], o[:, oracle.PG["z"]], rtol=1e-6)
    # the sort key (reading S7) bit for bit: the GPU's fp32 z_key = the oracle's fp32 z_key
    zg = np.ascontiguousarray(rec[vis][:, 12]).view(np.uint32)
    zo = o[:, oracle.PG["zkey"]].astype(np.float32).view(np.uint32)
    np.testing.assert_array_equal(zg, zo)
    ng = np.abs(o[:, oracle.PG["ndotx"]]) >= 0.05
    np.testing.assert_allclose(r[ng, 9:12], o[ng, 67:70], atol=2e-6)
    np.testing.assert_allclose(r[ng, 13:15], o[ng][:, oracle.PG["p"]], rtol=1e-3, atol=1e-7)


def test_binning_bit_exact(case):
    view = case["view"]
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(view))
    st = P.rd_view_stats(view)
    rk, ri = cpu_binning_reference(rect, touched, rec[:, 12], st["tiles_x"])
    assert st["n_duplicates"] == len(rk)
    np.testing.assert_array_equal(keys.view(np.uint64), rk)
    np.testing.assert_array_equal(ids.view(np.uint32), ri)
    T = st["tiles_x"] * st["tiles_y"]
    tiles = (rk >> np.uint64(32)).astype(np.int64)
    exp = np.zeros((T, 2), np.int64)
    for t in range(T):
        w = np.nonzero(tiles == t)[0]
        if len(w):
            exp[t] = (w[0], w[-1] + 1)
    np.testing.assert_array_equal(ranges.astype(np.int64), exp)


def test_binning_order_matches_oracle(case):
    """Per tile, the GPU's id list is the ORACLE's global front-to-back order (
    reading S7: z_key, ties by id — oracle.order) restricted to the Gaussians whose rect
    covers the tile; the 64-bit keys carry the oracle's z_key bits; ranges follow."""
    view, scene, cam, opt = case["view"], case["scene"], case["cam"], case["opt"]
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(view))
    st = P.rd_view_stats(view)
    tx_n = st["tiles_x"]
    order = oracle.order(scene, cam, opt)
    zk = oracle.project(scene, cam, opt)[:, oracle.PG["zkey"]].astype(np.float32).view(np.uint32)
    per_tile = [[] for _ in range(tx_n * st["tiles_y"])]
    for i in order:
        if touched[i] == 0:
            continue
        r0, r1 = int(rect[i, 0]) & 0xFFFFFFFF, int(rect[i, 1]) & 0xFFFFFFFF
        for ty in range(r0 >> 16, r1 >> 16):
            for tx in range(r0 & 0xFFFF, r1 & 0xFFFF):
                per_tile[ty * tx_n + tx].append(i)
    exp_ids = np.array([i for lst in per_tile for i in lst], np.uint32)
    exp_keys = np.array([(t << 32) | int(zk[i]) for t, lst in enumerate(per_tile) for i in lst], np.uint64)
    np.testing.assert_array_equal(ids.view(np.uint32), exp_ids)
    np.testing.assert_array_equal(keys.view(np.uint64), exp_keys)
    starts = np.cumsum([0] + [len(l) for l in per_tile])
    exp_r = np.array([(starts[t], starts[t + 1]) if per_tile[t] else (0, 0) for t in range(len(per_tile))])
    np.testing.assert_array_equal(ranges.astype(np.int64), exp_r)
    if case["name"].startswith("ties"):  # the case must actually exercise the tie-break
        zz = np.float32(zk.view(np.float32))
        assert any(len(l) > 1 and len(set(zz[l])) < len(l) for l in per_tile)


@pytest.mark.parametrize("W,H", [(2120, 40), (40, 2120), (2072, 2072)])
def test_binning_more_than_256_tiles_per_axis(W, H):
    """Beyond 256 tiles per axis at 8×8 tiles the tile sort takes a second digit per axis
    (tx low / tx high / ty low / ty high passes, binning.cu): keys, ids and ranges still equal
    the stable sort of the 64-bit keys, and the forward still matches the oracle (sampled)."""
    n = 3000 if W * H < 10 ** 6 else 6000
    scene = dense_scene(61, n, width=W, height=H, f=64.0, smin=0.01, smax=0.12)
    cam, opt = sg.camera_identity(W, H, 64.0), sg.Options(tile=8)
    res, view, _ = gpu_forward(scene, cam, opt)
    st = P.rd_view_stats(view)
    assert max(st["tiles_x"], st["tiles_y"]) > 256
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    keys, ids, ranges = (t.cpu().numpy() for t in P.rd_debug_binning(view))
    rk, ri = cpu_binning_reference(rect, touched, rec[:, 12], st["tiles_x"])
    assert st["n_duplicates"] == len(rk) > 0
    np.testing.assert_array_equal(keys.view(np.uint64), rk)
    np.testing.assert_array_equal(ids.view(np.uint32), ri)
    tiles = (rk >> np.uint64(32)).astype(np.int64)
    T = st["tiles_x"] * st["tiles_y"]
    first = np.full(T, -1, np.int64)
    last = np.full(T, -1, np.int64)
    pos = np.arange(len(tiles))
    first[tiles[::-1]] = pos[::-1]
    last[tiles] = pos
    exp = np.where(first[:, None] >= 0, np.stack([first, last + 1], 1), 0)
    np.testing.assert_array_equal(ranges.reshape(-1, 2).astype(np.int64), exp)
    rng = np.random.default_rng(62)
    pix = rng.choice(W * H, 256, replace=False)
    ref = oracle.render(scene, cam, opt, pixels=pix)
    ys, xs = pix // W, pix % W
    ok = (ref["flags"] & 5) == 0
    assert np.abs(res["color"][:, ys, xs] - ref["color"])[:, ok].max() <= 1e-4
    assert np.abs(res["alpha"][ys, xs] - ref["alpha"])[ok].max() <= 1e-4


def test_rect_is_conservative(case):
    """Every pixel where the oracle's α clears α_min (outside the F1 band) lies in a tile of
    the GPU's rect."""
    scene, cam, opt = case["scene"], case["cam"], case["opt"]
    rec, rect, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(case["view"]))
    pg = oracle.project(scene, cam, opt)
    W, H, tile = cam.width, cam.height, opt.tile
    uu, vv = np.meshgrid(np.arange(W) + 0.5, np.arange(H) + 0.5)
    uv = np.stack([uu.ravel(), vv.ravel()], 1)
    amin = float(np.float32(opt.alpha_min))
    for i in np.nonzero(pg[:, 0] == 1)[0]:
        ev = oracle.splat_eval(scene, cam, opt, int(i), uv)
        a = np.minimum(float(np.float32(opt.alpha_max)), ev[:, 0])
        need = np.log(np.maximum(a, 1e-300)) - np.log(amin) > 1e-4
        if not need.any():
            continue
        assert touched[i] > 0, i
        r0, r1 = int(rect[i, 0]) & 0xFFFFFFFF, int(rect[i, 1]) & 0xFFFFFFFF
        tx = (uv[need, 0] // tile).astype(int)
        ty = (uv[need, 1] // tile).astype(int)
        assert np.all((tx >= (r0 & 0xFFFF)) & (tx < (r1 & 0xFFFF)) & (ty >= (r0 >> 16)) & (ty < (r1 >> 16))), i


def test_backward_parity(case):
    scene, cam, opt = case["scene"], case["cam"], case["opt"]
    cot = sg.cotangents(7, cam.width, cam.height)
    ref = case["ref"]
    mask = ref["flags"] == 0
    cot = {k: (v * mask).astype(np.float32) for k, v in cot.items()}
    _, G, _ = gpu_grads(scene, cam, opt, cot)
    pg = oracle.project(scene, cam, opt)
    rgb_raw_near0 = np.zeros(scene.n, bool)  # F6: colour channel within 1e-6 of the clamp
    vis = np.nonzero(pg[:, 0] == 1)[0]
    R = oracle.grad(scene, cam, opt, cot, vis)
    Gv = G[vis]
    excl = rgb_raw_near0[vis]
    classes = {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10), "opacities": slice(10, 11),
               "sh": slice(11, 11 + 3 * (opt.sh_degree + 1) ** 2)}
    for name, sl in classes.items():
        a, b = Gv[~excl, sl], R[~excl, sl]
        nb = np.linalg.norm(b)
        if nb == 0:
            assert np.abs(a).max() == 0
            continue
        rel = np.linalg.norm(a - b) / nb
        assert rel <= 1e-3, (name, rel)
        med = np.median(np.abs(b[b != 0])) if (b != 0).any() else 0.0
        bad = np.abs(a - b) > 1e-3 * np.abs(b) + 1e-3 * med  # every entry
        assert not bad.any(), (name, int(bad.sum()), np.abs(a - b).max())
    # Gaussians the GPU did not draw get exactly zero gradient
    off = np.setdiff1d(np.arange(scene.n), vis)
    assert np.all(G[off] == 0)


def _big_splat_scene(seed=12, W=256):
    """A 256×256 view: 160 small Gaussians (dense_scene) plus 10 screen-sized splats whose
    tile rects exceed 16 384 px (so K1 puts them on the big list and their chain rule runs in
    fp64, K5b64): z ∈ [1.2, 3], scales 0.15–0.5 (σ ≈ 20–100 px), half of them flat (s_min =
    1e-3·s), three of those tilted to 70–80° from the view ray (near-grazing); opacities low
    enough that the splats behind them still receive gradient."""
    rng = np.random.default_rng(seed)
    base = dense_scene(seed, 160, width=W, height=W, f=float(W))
    nb = 10
    z = rng.uniform(1.2, 3.0, nb)
    uv = rng.uniform(0.25, 0.75, (2, nb)) * W
    x, y = (uv[0] - W / 2) * z / W, (uv[1] - W / 2) * z / W
    s = np.exp(rng.uniform(np.log(0.15), np.log(0.5), (3, nb)))
    flat = np.arange(nb) < 5
    s[2, flat] = s[0, flat] * 1e-3
    nrm = np.stack([np.zeros(nb), np.zeros(nb), -np.ones(nb)], 0)
    ang = np.deg2rad(rng.uniform(70, 80, nb))
    tilt = np.arange(nb) < 3  # flat and near-grazing: normal 70–80° away from the view axis
    nrm[:, tilt] = np.stack([np.sin(ang[tilt]), np.zeros(3), -np.cos(ang[tilt])], 0)
    q = sg.quaternion_with_axis3(nrm, rng)
    q[:, ~flat] = sg.random_quaternions(rng, (~flat).sum())
    big = sg.make_scene(np.stack([x, y, z]), s, q, rng.uniform(0.15, 0.45, nb), sg.sh_coeffs(rng, nb))
    return concat(base, big), sg.camera_identity(W, W, float(W))


@pytest.mark.parametrize("tile", [8, 16])
def test_big_splats_fp64_backward_parity(tile):
    """K5b64 (the fp64 chain rule of the screen-sized splats, rade_internal.cuh is_big)
    against the oracle's exact dual-number gradients: every parameter class, ≤ 1e-3 relative
    in norm and elementwise (|Δg| ≤ 1e-3|g| + 1e-3·median|g|) on every entry, for the big
    splats alone and for all visible Gaussians; flagged pixels (≤ 1%) get zero cotangent."""
    scene, cam = _big_splat_scene()
    opt = sg.Options(tile=tile)
    ref = oracle.render(scene, cam, opt)
    mask = ref["flags"] == 0
    assert mask.mean() >= 0.99, mask.mean()
    cot = sg.cotangents(13, cam.width, cam.height)
    cot = {k: (v * mask).astype(np.float32) for k, v in cot.items()}
    out, G, view = gpu_grads(scene, cam, opt, cot)
    st = P.rd_view_stats(view)
    _, _, touched = (t.cpu().numpy() for t in P.rd_debug_preprocess(view))
    big = np.nonzero(touched.astype(np.int64) * tile * tile > 16384)[0]
    assert st["n_big"] == len(big) >= 8, (st["n_big"], len(big))
    assert (big >= 160).sum() >= 8  # most of the added screen-sized splats
    ok = (ref["flags"] & (F1 | F3)) == 0
    for k in ("color", "normal"):
        assert np.abs(out[k] - ref[k])[:, ok].max() <= TOL, k
    vis = np.nonzero(touched > 0)[0]
    R = oracle.grad(scene, cam, opt, cot, vis)
    Gv = G[vis]
    for rows, label in ((np.isin(vis, big), "big"), (np.ones(len(vis), bool), "all")):
        for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                         "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
            a, b = Gv[rows, sl], R[rows, sl]
            nb = np.linalg.norm(b)
            assert nb > 0, (label, name)
            assert np.linalg.norm(a - b) / nb <= 1e-3, (label, name, np.linalg.norm(a - b) / nb)
            med = np.median(np.abs(b[b != 0]))
            bad = np.abs(a - b) > 1e-3 * np.abs(b) + 1e-3 * med
            assert not bad.any(), (label, name, int(bad.sum()))


def test_tile_size_independence():
    """Outputs are bit-identical for tile 8, 16 and 32 (the per-pixel op sequence does not
    depend on the tile; reading S8), on a ragged image; gradients agree to float-atomic
    rounding."""
    scene, cam = dense_scene(21, 400, width=83, height=61, f=70.0), sg.camera_identity(83, 61, 70.0)
    cot = sg.cotangents(4, 83, 61)
    outs = {t: gpu_grads(scene, cam, sg.Options(tile=t), cot) for t in (8, 16, 32)}
    for t in (16, 32):
        for k in outs[8][0]:
            np.testing.assert_array_equal(outs[t][0][k], outs[8][0][k], err_msg=f"tile {t} {k}")
        G, G8 = outs[t][1], outs[8][1]
        for sl in (slice(0, 3), slice(3, 6), slice(6, 10), slice(10, 11), slice(11, 59)):
            assert np.linalg.norm(G[:, sl] - G8[:, sl]) <= 1e-5 * np.linalg.norm(G8[:, sl]), (t, sl)


def test_forward_determinism_and_backward_close():
    scene, cam, opt = dense_scene(22, 400), sg.camera_identity(64, 64, 64), sg.Options()
    cot = sg.cotangents(1, 64, 64)
    a, Ga, _ = gpu_grads(scene, cam, opt, cot)
    b, Gb, _ = gpu_grads(scene, cam, opt, cot)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    # gradients use float atomics (order not fixed): equal to rounding, per parameter class
    for sl in (slice(0, 3), slice(3, 6), slice(6, 10), slice(10, 11), slice(11, 59)):
        na = np.linalg.norm(Ga[:, sl])
        assert np.linalg.norm(Ga[:, sl] - Gb[:, sl]) <= 1e-5 * max(na, 1e-30), sl


def test_empty_and_degenerate_inputs():
    cam, opt = sg.camera_identity(40, 24, 40), sg.Options()
    empty = sg.make_scene(np.zeros((3, 0)), np.zeros((3, 0)), np.zeros((4, 0)), np.zeros(0), np.zeros((16, 3, 0)))
    out, view, g = gpu_forward(empty, cam, opt)
    assert all(np.all(v == 0) for v in out.values())
    assert P.rd_view_stats(view)["n_duplicates"] == 0
    grads = g.zeros_like()
    P.rd_render_bwd(view, g, None, None, None, None, grads)
    # behind the camera, non-positive scale, zero quaternion, NaN mean, tiny opacity: all culled
    bad = concat(one_gaussian([0, 0, -3], [0.1] * 3), one_gaussian([0, 0, 3], [0.1, -0.1, 0.1]),
                 one_gaussian([0, 0, 3], [0.1] * 3, quat=(0, 0, 0, 0)),
                 one_gaussian([np.nan, 0, 3], [0.1] * 3), one_gaussian([0, 0, 3], [0.1] * 3, opacity=1e-3),
                 one_gaussian([0, 0, 0.1], [0.1] * 3))
    out, view, g = gpu_forward(bad, cam, opt)
    assert all(np.all(v == 0) for v in out.values())
    cot = sg.cotangents(2, 40, 24)
    _, G, _ = gpu_grads(bad, cam, opt, cot)
    assert np.all(G == 0)


def test_single_splat_at_centre():
    cam = sg.camera_identity(64, 64, 64)
    z = 3.0
    sc = one_gaussian([(20.5 - 32) * z / 64, (40.5 - 32) * z / 64, z], [0.1, 0.08, 0.12], [0.9, 0.1, -0.2, 0.3],
                      opacity=0.999)
    out, _, _ = gpu_forward(sc, cam, sg.Options())
    pg = oracle.project(sc, cam, sg.Options())[0]
    assert abs(out["alpha"][40, 20] - 0.99) < 1e-6
    np.testing.assert_allclose(out["color"][:, 40, 20], 0.99 * pg[oracle.PG["rgb"]], atol=1e-6)
    assert abs(out["depth"][40, 20] - pg[oracle.PG["z"]]) < 1e-5


def test_invalid_arguments_return_errors():
    cam = sg.camera_identity(16, 16, 16)
    g = P.Gaussians.from_numpy(dense_scene(0, 5))
    view = P.View()
    for bad in (dict(tile=12), dict(alpha_min=0.0), dict(alpha_min=0.995), dict(sh_degree=4), dict(T_min=1.5)):
        with pytest.raises(P.rade.N.RadeError) as e:
            P.rd_preprocess(view, g, cam, bad)
        assert e.value.status == 1
    with pytest.raises(P.rade.N.RadeError) as e:
        P.rd_bin(view)
    assert e.value.status == 2
    bad_cam = sg.camera_identity(16, 16, 16)
    bad_cam.width = 0
    with pytest.raises(P.rade.N.RadeError):
        P.rd_preprocess(view, g, bad_cam)


def test_rasterize_autograd_wrapper():
    scene, cam, opt = dense_scene(30, 100), sg.camera_identity(32, 32, 32), sg.Options()
    g = P.Gaussians.from_numpy(scene)
    ts = [t.clone().requires_grad_(True) for t in g.tensors()]
    color, depth, normal, alpha = P.rasterize(*ts, cam)
    cot = sg.cotangents(3, 32, 32)
    c = {k: torch.as_tensor(v).cuda() for k, v in cot.items()}
    L = (color * c["color"]).sum() + (depth * c["depth"]).sum() + (normal * c["normal"]).sum() + (alpha * c["alpha"]).sum()
    L.backward()
    _, G, _ = gpu_grads(scene, cam, opt, cot)
    np.testing.assert_allclose(ts[0].grad.double().cpu().numpy(), G[:, 0:3], rtol=1e-4, atol=1e-6)


# ----------------------------------------------------------------------------- NEXT-1: L_d

def _gpu_distortion(scene, cam, opt):
    g = P.Gaussians.from_numpy(scene)
    view = P.View()
    P.rd_preprocess(view, g, cam, opts_dict(opt))
    P.rd_bin(view)
    out = P.rd_render_fwd_ex(view, distortion=True)
    torch.cuda.synchronize()
    return out["distortion"].double().cpu().numpy(), view, g


def test_distortion_forward_parity(case):
    """Depth-distortion map (reading S21) vs the oracle's double sum."""
    ref = case["ref"]
    L, _, _ = _gpu_distortion(case["scene"], case["cam"], case["opt"])
    ok = (ref["flags"] & (F1 | F3)) == 0
    err = np.abs(L - ref["distortion"])[ok]
    assert err.max() <= TOL * np.maximum(1.0, np.abs(ref["distortion"][ok])).max(), err.max()
    assert ref["distortion"].max() > 1e-3 or case["name"] == "C0"


def test_distortion_backward_parity(case):
    """Gradients of Σ g·L_d (ω detached, S21) — together with the four image cotangents —
    vs the oracle's dual numbers; per parameter class ≤ 1e-3 relative."""
    scene, cam, opt = case["scene"], case["cam"], case["opt"]
    ref = case["ref"]
    mask = ref["flags"] == 0
    cot = sg.cotangents(8, cam.width, cam.height)
    rng = np.random.default_rng(9)
    cot["distortion"] = rng.normal(size=(cam.height, cam.width))
    cot = {k: (v * mask).astype(np.float32) for k, v in cot.items()}
    _, view, g = _gpu_distortion(scene, cam, opt)
    dev = torch.device("cuda")
    c = {k: torch.as_tensor(v).contiguous().to(dev) for k, v in cot.items()}
    grads = g.zeros_like()
    P.rd_blend_bwd_ex(view, c["color"], c["depth"], c["normal"], c["alpha"], c["distortion"])
    P.rd_preprocess_bwd(view, g, grads)
    torch.cuda.synchronize()
    G = grads_to_rows(grads, scene.n)
    pg = oracle.project(scene, cam, opt)
    vis = np.nonzero(pg[:, 0] == 1)[0]
    R = oracle.grad(scene, cam, opt, cot, vis)
    for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                     "opacities": slice(10, 11), "sh": slice(11, 11 + 3 * (opt.sh_degree + 1) ** 2)}.items():
        a, b = G[vis, sl], R[:, sl]
        nb = np.linalg.norm(b)
        if nb == 0:
            assert np.abs(a).max() == 0
            continue
        assert np.linalg.norm(a - b) / nb <= 1e-3, name


def test_distortion_cotangent_needs_distortion_forward():
    scene, cam = dense_scene(3, 50), sg.camera_identity(32, 32, 32)
    out, view, g = gpu_forward(scene, cam, sg.Options())
    z = torch.zeros((32, 32), device="cuda")
    with pytest.raises(P.rade.N.RadeError) as e:
        P.rd_blend_bwd_ex(view, dL_ddistortion=z)
    assert e.value.status == 2


# ----------------------------------------------------------------------------- NEXT-2: L_n

def test_normal_consistency_forward_parity(case):
    """L_n = A − N·ñ and the depth normals ñ (reading S22): the GPU kernel vs the oracle's
    numpy definition, both on the oracle's rendered maps rounded to fp32 (≤ 1e-4), excluding
    stencils whose orientation is ambiguous (|ñ·P̂| < 1e-3)."""
    cam, gpu = case["cam"], case["ref"]  # maps from the oracle only
    dev = torch.device("cuda")
    t = {k: torch.as_tensor(np.asarray(gpu[k], np.float32)).contiguous().to(dev) for k in ("depth", "alpha", "normal")}
    L, nt = P.rd_normal_consistency(cam, t["depth"], t["alpha"], t["normal"], consistency=True, depth_normal=True)
    torch.cuda.synchronize()
    Lr, ntr = oracle.normal_consistency(gpu["depth"].astype(np.float32).astype(np.float64),
                                        gpu["alpha"].astype(np.float32).astype(np.float64),
                                        gpu["normal"].astype(np.float32).astype(np.float64), cam)
    H, W = gpu["depth"].shape
    xs = (np.arange(W) + 0.5 - cam.cx) / cam.fx
    ys = (np.arange(H) + 0.5 - cam.cy) / cam.fy
    ray = np.stack([np.broadcast_to(xs[None, :], (H, W)), np.broadcast_to(ys[:, None], (H, W)), np.ones((H, W))], 0)
    cosang = np.abs(np.sum(ntr * ray, 0)) / np.linalg.norm(ray, axis=0)
    valid = np.any(ntr != 0, 0)
    ok = ~valid | (cosang > 1e-3)
    np.testing.assert_allclose(nt.cpu().numpy()[:, ok], ntr[:, ok], atol=1e-4)
    np.testing.assert_allclose(L.cpu().numpy()[ok], Lr[ok], atol=1e-4)
    assert valid.sum() > 20 or case["name"] == "C0"


def test_normal_consistency_backward_vs_finite_differences():
    """dL/dD, dL/dA, dL/dN of Σ g·L_n from the GPU kernel vs central finite differences of the
    oracle's fp64 L_n on a small smooth depth map (plus the closed forms dL/dA = g on valid
    pixels and dL/dN = −g ñ)."""
    cam = sg.Camera(30.0, 32.0, 6.2, 4.9, 12, 10, np.eye(3), np.zeros(3), 0.2)
    rng = np.random.default_rng(3)
    H, W = 10, 12
    yy, xx = np.mgrid[0:H, 0:W]
    D = 3.0 + 0.3 * np.sin(0.5 * xx) + 0.2 * np.cos(0.4 * yy) + 0.05 * rng.random((H, W))
    D[7, 3] = 0.0  # a hole
    A = rng.uniform(0.2, 1.0, (H, W))
    Nm = rng.normal(size=(3, H, W)) * 0.5
    g = rng.normal(size=(H, W))
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    D, A, Nm, g = f32(D), f32(A), f32(Nm), f32(g)
    dev = torch.device("cuda")
    tD, tA, tN, tg = (torch.as_tensor(np.asarray(v, np.float32)).contiguous().to(dev) for v in (D, A, Nm, g))
    gD, gA, gN = torch.zeros_like(tD), torch.zeros_like(tA), torch.zeros_like(tN)
    P.rd_normal_consistency_bwd(cam, tD, tN, tg, gD, gA, gN)
    torch.cuda.synchronize()
    L0, nt = oracle.normal_consistency(D, A, Nm, cam)
    valid = np.any(nt != 0, 0)
    np.testing.assert_allclose(gA.cpu().numpy(), np.where(valid, g, 0.0), atol=1e-6)
    np.testing.assert_allclose(gN.cpu().numpy(), -g[None] * nt, atol=1e-6)
    fd = np.zeros((H, W))
    h = 1e-6
    for y in range(H):
        for x in range(W):
            if D[y, x] == 0:
                continue
            Dp, Dm = D.copy(), D.copy()
            Dp[y, x] += h
            Dm[y, x] -= h
            fd[y, x] = (np.sum(g * oracle.normal_consistency(Dp, A, Nm, cam)[0])
                        - np.sum(g * oracle.normal_consistency(Dm, A, Nm, cam)[0])) / (2 * h)
    got = gD.cpu().numpy()
    np.testing.assert_allclose(got, fd, rtol=1e-3, atol=1e-3 * np.abs(fd).max())
    assert np.abs(fd).max() > 1e-2


# ----------------------------------------------------------------------------- NEXT-3: 3D filter

def test_filter3d_forward_and_backward_parity():
    """Mip-Splatting 3D filter (reading S23): the GPU with a per-Gaussian filter size equals
    the oracle on the filtered scene (forward ≤ 1e-4), and its raw-parameter gradients equal
    the oracle's gradients mapped through the filter's vjp (≤ 1e-3 per class)."""
    scene, cam, opt = dense_scene(31, 300), sg.camera_identity(64, 64, 64), sg.Options()
    f = np.random.default_rng(6).uniform(0.005, 0.08, scene.n).astype(np.float32)
    fs, vjp = oracle.apply_filter3d(scene, f.astype(np.float64))
    ref = oracle.render(fs, cam, opt)
    g = P.Gaussians.from_numpy(scene)
    g.filter3d = torch.as_tensor(f).cuda()
    out, view = P.render(g, cam, opts_dict(opt))
    torch.cuda.synchronize()
    gpu = {k: v.double().cpu().numpy() for k, v in out.items()}
    ok = (ref["flags"] & (F1 | F3)) == 0
    assert ok.mean() > 0.95
    for k in ("color", "normal"):
        assert np.abs(gpu[k] - ref[k])[:, ok].max() <= TOL, k
    assert np.abs(gpu["alpha"] - ref["alpha"])[ok].max() <= TOL
    okd = (ref["flags"] & (F1 | F3 | F4 | F5)) == 0
    assert np.abs(gpu["depth"] - ref["depth"])[okd].max() <= TOL
    cot = sg.cotangents(7, 64, 64)
    cot = {k: (v * (ref["flags"] == 0)).astype(np.float32) for k, v in cot.items()}
    c = {k: torch.as_tensor(v).contiguous().cuda() for k, v in cot.items()}
    grads = g.zeros_like()
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], grads)
    torch.cuda.synchronize()
    G = grads_to_rows(grads, scene.n)
    pg = oracle.project(fs, cam, opt)
    vis = np.nonzero(pg[:, 0] == 1)[0]
    R = vjp(oracle.grad(fs, cam, opt, cot, vis), vis)
    for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                     "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
        nb = np.linalg.norm(R[:, sl])
        assert nb > 0
        assert np.linalg.norm(G[vis, sl] - R[:, sl]) / nb <= 1e-3, name


# ----------------------------------------------------------------------------- NEXT-4: TSDF

def _fuse_both(depths, cams, origin, vs, dims, trunc, max_depth=1e30):
    vol = P.TsdfVolume(origin, vs, dims, trunc, max_depth)
    D = torch.as_tensor(np.asarray(depths, np.float32)).contiguous().cuda()
    P.rd_tsdf_integrate(vol, D, cams)
    torch.cuda.synchronize()
    X, Y, Z = dims
    t, w = np.ones((Z, Y, X)), np.zeros((Z, Y, X))
    for k, cam in enumerate(cams):
        oracle.tsdf_integrate(t, w, origin, vs, trunc, max_depth, np.asarray(depths[k], np.float32), cam)
    return vol.tsdf.double().cpu().numpy(), vol.weight.double().cpu().numpy(), t, w


def test_tsdf_fusion_parity():
    """TSDF fusion (reading S24) of the GPU's median depth maps of a scene seen from 40 views
    (two kernel launches of up to 32 fused views): weights bit-exact, tsdf ≤ 1e-5."""
    scene = dense_scene(41, 300)
    cams = []
    for k in range(40):
        a = 2 * np.pi * k / 40
        R, t = sg.look_at([0.8 * np.cos(a), 0.8 * np.sin(a), -0.5], [0.0, 0.0, 4.0], up=(0, -1, 0))
        cams.append(sg.Camera(64.0, 64.0, 32.0, 32.0, 64, 64, R, t, 0.2))
    depths = [oracle.render(scene, c, sg.Options())["depth"] for c in cams]  # inputs from the oracle only
    g, wg, t, w = _fuse_both(depths, cams, (-2.0, -2.0, 2.0), 0.05, (80, 80, 80), 0.2, 50.0)
    np.testing.assert_array_equal(wg, w)
    assert (w > 0).sum() > 5000 and w.max() > 20
    np.testing.assert_allclose(g[w > 0], t[w > 0], atol=1e-5)


# ----------------------------------------------------------------------------- NEXT-4: marching cubes

def _mc_both(tsdf, weight, origin, vs, iso=0.0):
    Z, Y, X = tsdf.shape
    vol = P.TsdfVolume(origin, vs, (X, Y, Z))
    vol.tsdf.copy_(torch.as_tensor(np.asarray(tsdf, np.float32)))
    vol.weight.copy_(torch.as_tensor(np.asarray(weight, np.float32)))
    tri = P.rd_marching_cubes(vol, iso)
    torch.cuda.synchronize()
    ref = oracle.marching_cubes(np.asarray(tsdf, np.float32), weight, origin, vs, iso)
    return tri.double().cpu().numpy(), ref


def test_marching_cubes_random_volume_every_configuration():
    """Uniform random values on 21³ voxels (8000 cells: every one of the 256 corner
    configurations occurs) with 2 % zero-weight voxels: same triangles in the same order as
    the oracle (the tables agree config by config), vertices ≤ 1e-5."""
    rng = np.random.default_rng(5)
    t = rng.uniform(-1, 1, (21, 21, 21)).astype(np.float32)
    w = (rng.random((21, 21, 21)) > 0.02).astype(np.float32)
    gpu, ref = _mc_both(t, w, (-1.0, 0.5, 2.0), 0.1, iso=0.1)
    assert ref.shape[0] > 10000
    assert gpu.shape == ref.shape
    np.testing.assert_allclose(gpu, ref, atol=1e-5)


def test_marching_cubes_capacity_guess_paths():
    """The binding's one-call path (a capacity guess kept from the volume's last extraction)
    and its fallback (guess too small: count, allocate, emit) give the oracle's soup."""
    rng = np.random.default_rng(8)
    t = rng.uniform(-1, 1, (12, 12, 12)).astype(np.float32)
    w = np.ones_like(t)
    ref = oracle.marching_cubes(t, w, (0.0, 0.0, 0.0), 0.5, 0.0)
    vol = P.TsdfVolume((0.0, 0.0, 0.0), 0.5, (12, 12, 12))
    vol.tsdf.copy_(torch.as_tensor(t))
    vol.weight.copy_(torch.as_tensor(w))
    for cap in (0, 7, None):  # no guess, too small, the binding's own guess
        if cap is not None:
            vol._mc_capacity = cap
        gpu = P.rd_marching_cubes(vol).double().cpu().numpy()
        assert gpu.shape == ref.shape, cap
        np.testing.assert_allclose(gpu, ref, atol=1e-5)


def test_marching_cubes_exact_iso_corners():
    """Corner values equal to iso (integer volume, iso 0): the zero-area triangles with two
    vertices on one corner are dropped on both sides (reading S25); same soup, same order."""
    rng = np.random.default_rng(21)
    t = rng.integers(-1, 2, (17, 17, 17)).astype(np.float32)
    gpu, ref = _mc_both(t, np.ones_like(t), (0.5, -1.0, 2.0), 0.25, 0.0)
    assert ref.shape[0] > 1000 and gpu.shape == ref.shape
    np.testing.assert_allclose(gpu, ref, atol=1e-6)
    area = np.linalg.norm(np.cross(gpu[:, 1] - gpu[:, 0], gpu[:, 2] - gpu[:, 0]), axis=1)
    assert area.min() > 0


def test_marching_cubes_scratch_across_streams():
    """Two extractions issued back to back from one host thread on two different streams
    (the per-thread scratch is shared): both return the oracle's soup."""
    rng = np.random.default_rng(22)
    vols, refs = [], []
    for n in (20, 14):
        t = rng.uniform(-1, 1, (n, n, n)).astype(np.float32)
        vol = P.TsdfVolume((0.0, 0.0, 0.0), 0.5, (n, n, n))
        vol.tsdf.copy_(torch.as_tensor(t))
        vol.weight.fill_(1.0)
        vols.append(vol)
        refs.append(oracle.marching_cubes(t, np.ones_like(t), (0.0, 0.0, 0.0), 0.5, 0.0))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        a = P.rd_marching_cubes(vols[0])
    with torch.cuda.stream(s2):
        b = P.rd_marching_cubes(vols[1])
    torch.cuda.synchronize()
    for got, ref in ((a, refs[0]), (b, refs[1])):
        got = got.double().cpu().numpy()
        assert got.shape == ref.shape
        np.testing.assert_allclose(got, ref, atol=1e-5)


def test_marching_cubes_degenerate_volumes():
    """Empty (< 2 voxels along an axis), unobserved (weight 0), all-inside / all-outside:
    no triangles; a too-small capacity returns the count and writes nothing."""
    for shape in ((1, 5, 5), (5, 1, 5), (5, 5, 1)):
        gpu, ref = _mc_both(np.zeros(shape, np.float32) - 1, np.ones(shape), (0.0, 0.0, 0.0), 1.0)
        assert gpu.shape[0] == 0 and ref.shape[0] == 0
    t = np.linspace(-1, 1, 6 * 6 * 6, dtype=np.float32).reshape(6, 6, 6)
    gpu, _ = _mc_both(t, np.zeros_like(t), (0.0, 0.0, 0.0), 1.0)
    assert gpu.shape[0] == 0
    for val in (-1.0, 1.0):
        gpu, _ = _mc_both(np.full((4, 4, 4), val, np.float32), np.ones((4, 4, 4)), (0.0, 0.0, 0.0), 1.0)
        assert gpu.shape[0] == 0
    vol = P.TsdfVolume((0.0, 0.0, 0.0), 1.0, (6, 6, 6))
    vol.tsdf.copy_(torch.as_tensor(t))
    vol.weight.fill_(1.0)
    s = vol.c_struct()
    import ctypes
    from paper_2406_01467_b200 import _native as N
    n = ctypes.c_int64(-1)
    buf = torch.full((4, 3, 3), 7.0, device="cuda")
    assert N.load().rd_marching_cubes(ctypes.byref(s), 0.0, ctypes.c_void_p(buf.data_ptr()), 4, ctypes.byref(n),
                                      None) == 0
    assert n.value > 4 and bool((buf == 7.0).all())


def test_marching_cubes_of_fused_depth_maps():
    """The paper's mesh path: the oracle fuses oracle-rendered median depth maps
    (40 views); (1) rd_marching_cubes on that fused volume (uploaded in fp32) returns the
    oracle's triangle soup, same order, vertices ≤ 1e-5; (2) end to end on the GPU
    (rd_tsdf_integrate then rd_marching_cubes, tsdf ≤ 1e-5 off the oracle's, so decisions at
    near-tied voxels may flip): triangle count within 0.5 %, every vertex within 0.1 voxel of
    the oracle mesh's vertices and vice versa."""
    from scipy.spatial import cKDTree
    scene = dense_scene(41, 300)
    cams = []
    for k in range(40):
        a = 2 * np.pi * k / 40
        R, t = sg.look_at([0.8 * np.cos(a), 0.8 * np.sin(a), -0.5], [0.0, 0.0, 4.0], up=(0, -1, 0))
        cams.append(sg.Camera(64.0, 64.0, 32.0, 32.0, 64, 64, R, t, 0.2))
    depths = [oracle.render(scene, c, sg.Options())["depth"] for c in cams]
    origin, vs, dims = (-2.0, -2.0, 2.0), 0.05, (64, 64, 64)
    X, Y, Z = dims
    t, w = np.ones((Z, Y, X)), np.zeros((Z, Y, X))
    for k, cam in enumerate(cams):
        oracle.tsdf_integrate(t, w, origin, vs, 0.2, 50.0, np.asarray(depths[k], np.float32), cam)
    gpu, ref = _mc_both(t.astype(np.float32), w, origin, vs)
    assert ref.shape[0] > 1000
    assert gpu.shape == ref.shape
    np.testing.assert_allclose(gpu, ref, atol=1e-5)

    vol = P.TsdfVolume(origin, vs, dims, 0.2, 50.0)
    P.rd_tsdf_integrate(vol, torch.as_tensor(np.asarray(depths, np.float32)).contiguous().cuda(), cams)
    e2e = P.rd_marching_cubes(vol).double().cpu().numpy()
    assert abs(e2e.shape[0] - ref.shape[0]) <= 0.005 * ref.shape[0]
    a, b = e2e.reshape(-1, 3), ref.reshape(-1, 3)
    assert cKDTree(b).query(a)[0].max() <= 0.1 * vs
    assert cKDTree(a).query(b)[0].max() <= 0.1 * vs


# ----------------------------------------------------------------------------- batched K5

def _views_of(scene, cams, opt, cots):
    g = P.Gaussians.from_numpy(scene)
    views = []
    for cam, cot in zip(cams, cots):
        view = P.View()
        P.rd_preprocess(view, g, cam, opts_dict(opt))
        P.rd_bin(view)
        P.rd_render_fwd(view)
        c = {k: torch.as_tensor(v).contiguous().cuda() for k, v in cot.items()}
        P.rd_blend_bwd(view, c["color"], c["depth"], c["normal"], c["alpha"])
        views.append(view)
    return g, views


def _orbit_cams(n, W=64, H=64, f=64.0, r=0.8, z=-0.5):
    cams = []
    for k in range(n):
        a = 2 * np.pi * k / n
        R, t = sg.look_at([r * np.cos(a), r * np.sin(a), z], [0.0, 0.0, 4.0], up=(0, -1, 0))
        cams.append(sg.Camera(f, f, W / 2, H / 2, W, H, R, t, 0.2))
    return cams


@pytest.mark.parametrize("which", ["dense", "big"])
def test_batched_k5_matches_oracle_sum_over_views(which):
    """rd_preprocess_bwd_views over 3 views (each Gaussian's rows read once, the views' chain
    rules summed on chip) = Σ over views of the oracle's exact gradients (≤ 1e-3 per class,
    elementwise on every entry) and = the per-view rd_preprocess_bwd sum to fp32 rounding;
    'big' adds screen-sized splats (their fp64 K5b64 pass runs per view inside the batch)."""
    if which == "dense":
        scene, cams = dense_scene(33, 300, zr=(3.0, 6.0)), _orbit_cams(3)
    else:
        scene, cam0 = _big_splat_scene(seed=14, W=256)
        cams = _orbit_cams(3, W=256, H=256, f=256.0, r=0.3, z=0.0)
    opt = sg.Options(tile=8)
    cots, R = [], 0.0
    for k, cam in enumerate(cams):
        ref = oracle.render(scene, cam, opt)
        mask = ref["flags"] == 0
        assert mask.mean() >= 0.99
        cot = {k_: (v * mask).astype(np.float32) for k_, v in sg.cotangents(40 + k, cam.width, cam.height).items()}
        cots.append(cot)
        R = R + oracle.grad(scene, cam, opt, cot, np.arange(scene.n))
    g, views = _views_of(scene, cams, opt, cots)
    if which == "big":
        assert sum(P.rd_view_stats(v)["n_big"] for v in views) > 0
    gb = g.zeros_like()
    P.rd_preprocess_bwd_views(views, g, gb)
    gs = g.zeros_like()
    for v in views:
        P.rd_preprocess_bwd(v, g, gs)
    gp = g.zeros_like()  # split: geometry per view, then the round's SH part
    for v in views:
        P.rd_preprocess_bwd_geometry(v, g, gp)
    P.rd_preprocess_bwd_views_sh(views, g, gp)
    torch.cuda.synchronize()
    B, S = grads_to_rows(gb, scene.n), grads_to_rows(gs, scene.n)
    Sp = grads_to_rows(gp, scene.n)
    for name, sl in {"means": slice(0, 3), "scales": slice(3, 6), "rotations": slice(6, 10),
                     "opacities": slice(10, 11), "sh": slice(11, 59)}.items():
        a, b = B[:, sl], R[:, sl]
        nb = np.linalg.norm(b)
        assert nb > 0, name
        assert np.linalg.norm(a - b) / nb <= 1e-3, (name, np.linalg.norm(a - b) / nb)
        med = np.median(np.abs(b[b != 0]))
        assert not (np.abs(a - b) > 1e-3 * np.abs(b) + 1e-3 * med).any(), name
        assert np.linalg.norm(a - S[:, sl]) <= 1e-5 * np.linalg.norm(S[:, sl]), name
        assert np.linalg.norm(Sp[:, sl] - a) <= 1e-5 * np.linalg.norm(a), name


@pytest.mark.parametrize("sh_degree", [3, 1])
def test_batched_k5_set_sh_rows(sh_degree):
    """rd_preprocess_bwd_views_ex(RD_K5_SET_SH) writes every SH gradient row — the batched
    gradient where a Gaussian is visible in some view, 0 elsewhere and above the active degree —
    without reading the old values: on a buffer whose SH part holds garbage it equals the
    accumulating call on a zeroed buffer (same summation order, bit for bit), and the other
    classes are accumulated as usual."""
    behind = dense_scene(37, 40, zr=(3.0, 6.0))  # mirrored behind the cameras: culled in every view
    behind.means[2] *= -1.0
    scene, cams = concat(dense_scene(36, 300, zr=(3.0, 6.0)), behind), _orbit_cams(3)
    scene.sh_degree = sh_degree
    opt = sg.Options(tile=8, sh_degree=sh_degree)
    cots = [sg.cotangents(50 + k, 64, 64) for k in range(3)]
    g, views = _views_of(scene, cams, opt, cots)
    ref = g.zeros_like()
    P.rd_preprocess_bwd_views(views, g, ref)
    got = g.zeros_like()
    got.sh.fill_(123.0)  # garbage: every SH row must be overwritten
    P.rd_preprocess_bwd_views_ex(views, g, got, flags=P.rade.RD_K5_SET_SH)
    torch.cuda.synchronize()
    assert torch.equal(got.sh, ref.sh)  # one store vs one reduction onto 0: the same values
    for name in ("means", "scales", "rotations", "opacities"):  # float atomics: order-dependent rounding
        a, b = getattr(got, name).cpu().numpy(), getattr(ref, name).cpu().numpy()
        assert np.abs(a - b).max() <= 1e-6 * max(np.abs(b).max(), 1e-30), name
    vis = np.zeros(scene.n, bool)
    for v in views:
        vis |= P.rd_debug_preprocess(v)[2].cpu().numpy() > 0
    assert (~vis).any() and vis.any()
    sh = got.sh.cpu().numpy().reshape(scene.n, -1)
    assert not sh[~vis].any()  # rows of Gaussians visible in no view: 0
    K = (sh_degree + 1) ** 2
    assert not sh[:, 3 * K:].any()  # coefficients above the active degree: 0
    # bench --k5 split-set: each view's geometry part on its own, then the round's SH part
    # setting the rows (RD_K5_SH_ONLY | RD_K5_SET_SH) — the same gradients
    spl = g.zeros_like()
    spl.sh.fill_(-7.0)
    for v in views:
        P.rd_preprocess_bwd_geometry(v, g, spl)
    P.rd_preprocess_bwd_views_ex(views, g, spl, flags=P.rade.RD_K5_SH_ONLY | P.rade.RD_K5_SET_SH)
    torch.cuda.synchronize()
    assert torch.equal(spl.sh, ref.sh)
    for name in ("means", "scales", "rotations", "opacities"):
        a, b = getattr(spl, name).cpu().numpy(), getattr(ref, name).cpu().numpy()
        assert np.abs(a - b).max() <= 1e-6 * max(np.abs(b).max(), 1e-30), name
    with pytest.raises(P.rade.N.RadeError):
        P.rd_preprocess_bwd_views_ex(views, g, got, flags=8)
    with pytest.raises(P.rade.N.RadeError):
        P.rd_preprocess_bwd_views_ex(views, g, got, flags=P.rade.RD_K5_SET_SH | P.rade.RD_K5_GEOMETRY_ONLY)


def test_batched_k5_argument_errors():
    scene, cams = dense_scene(34, 50), _orbit_cams(2)
    opt = sg.Options(tile=8)
    cots = [sg.cotangents(k, 64, 64) for k in range(2)]
    g, views = _views_of(scene, cams, opt, cots)
    gr = g.zeros_like()
    for bad, status in (([views[0], views[0]], 1), ([views[0]] * 9, 1), ([], 1)):
        for fn in (P.rd_preprocess_bwd_views, P.rd_preprocess_bwd_views_sh):
            with pytest.raises(P.rade.N.RadeError) as e:
                fn(bad, g, gr)
            assert e.value.status == status
    fresh = P.View()
    P.rd_preprocess(fresh, g, cams[0], opts_dict(opt))
    with pytest.raises(P.rade.N.RadeError) as e:
        P.rd_preprocess_bwd_views([views[0], fresh], g, gr)
    assert e.value.status == 2
    with pytest.raises(P.rade.N.RadeError) as e:
        P.rd_preprocess_bwd_geometry(fresh, g, gr)
    assert e.value.status == 2


def test_preprocess_views_equals_per_view():
    """rd_preprocess_views (one K1 launch over a round of views) = rd_preprocess on each view,
    bit for bit: records, rects, tile counts, and the binned lists and renders that follow."""
    scene, cams = dense_scene(38, 400, zr=(3.0, 6.0)), _orbit_cams(3)
    opt = sg.Options(tile=8)
    g = P.Gaussians.from_numpy(scene)
    batched = [P.View() for _ in cams]
    P.rd_preprocess_views(batched, g, cams, opts_dict(opt))
    for v, cam in zip(batched, cams):
        single = P.View()
        P.rd_preprocess(single, g, cam, opts_dict(opt))
        (ra, ea, ta), (rb, eb, tb) = P.rd_debug_preprocess(v), P.rd_debug_preprocess(single)
        assert torch.equal(ta, tb)
        vis = tb > 0  # culled Gaussians get no record / rect
        assert vis.any()
        assert torch.equal(ra[vis], rb[vis]) and torch.equal(ea[vis], eb[vis])
        P.rd_bin(v)
        P.rd_bin(single)
        for a, b in zip(P.rd_debug_binning(v), P.rd_debug_binning(single)):
            assert torch.equal(a, b)
        o1, o2 = P.rd_render_fwd(v), P.rd_render_fwd(single)
        torch.cuda.synchronize()
        for k in o1:
            assert torch.equal(o1[k], o2[k]), k
    with pytest.raises(P.rade.N.RadeError):
        P.rd_preprocess_views([batched[0], batched[0]], g, cams[:2], opts_dict(opt))


def test_bin_twice_keeps_the_lists():
    """A second rd_bin before the next rd_preprocess returns the same M and leaves keys, ids and
    ranges bit-identical (the depth passes consume K1's id-order keys, so it must not re-sort);
    the render after it equals a fresh view's."""
    scene = dense_scene(71, 400)
    cam, opt = sg.camera_identity(64, 64, 64.0), sg.Options(tile=8)
    g = P.Gaussians.from_numpy(scene)
    view = P.View()
    P.rd_preprocess(view, g, cam, opts_dict(opt))
    m1 = P.rd_bin(view)
    k1, i1, r1 = (t.clone() for t in P.rd_debug_binning(view))
    m2 = P.rd_bin(view)
    k2, i2, r2 = P.rd_debug_binning(view)
    torch.cuda.synchronize()
    assert m1 == m2 > 0
    assert torch.equal(k1, k2) and torch.equal(i1, i2) and torch.equal(r1, r2)
    out = P.rd_render_fwd(view)
    ref, _ = P.render(g, cam, opts_dict(opt))
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(out[k], ref[k]), k


def test_view_reuse_depth_sort_capacity():
    """One rd_view reused across views whose visible counts differ (the visible-only depth sort
    sizes itself from the view's history): few → many visible (the capacity guess is too
    small: redone at full size) → few (padding beyond the visible ones). Every render equals a
    fresh view's bit for bit, binning included."""
    rng = np.random.default_rng(35)
    n = 24000
    z = rng.uniform(2.0, 6.0, n)
    x = rng.uniform(-0.5, 0.5, n) * z
    y = rng.uniform(-0.5, 0.5, n) * z
    sc = sg.make_scene(np.stack([x, y, z]), np.exp(rng.uniform(np.log(0.005), np.log(0.03), (3, n))),
                       sg.random_quaternions(rng, n), sg.opacity_mixture(rng, n), sg.sh_coeffs(rng, n))
    g = P.Gaussians.from_numpy(sc)
    # a camera seeing a corner of the cloud, one seeing all of it, then the corner again
    near = sg.Camera(64.0, 64.0, 32.0 + 200.0, 32.0 + 200.0, 64, 64, np.eye(3, dtype=np.float32),
                     np.zeros(3, np.float32), 0.2)
    full = sg.camera_identity(64, 64, 64.0)
    opt = opts_dict(sg.Options(tile=8))
    reused = P.View()
    counts = []
    for cam in (near, full, near, full):
        out_r, _ = P.render(g, cam, opt, view=reused)
        out_f, fresh = P.render(g, cam, opt)
        torch.cuda.synchronize()
        for k in out_r:
            assert torch.equal(out_r[k], out_f[k]), k
        kr, ir, rr = P.rd_debug_binning(reused)
        kf, i_f, rf = P.rd_debug_binning(fresh)
        assert torch.equal(kr, kf) and torch.equal(ir, i_f) and torch.equal(rr, rf)
        counts.append(P.rd_view_stats(reused)["n_visible"])
    assert counts[0] < 4000 < 16000 < counts[1], counts


def test_means2d_gradient_parity(case):
    """rd_grads.means2d (dL/d(u_c, v_c), the screen-space gradient) against the oracle's dual
    numbers on the projected centre (oracle.grad(..., means2d=True) columns 59..60): ≤ 1e-3
    relative in norm and elementwise on every entry; the other classes are unchanged by
    requesting it."""
    scene, cam, opt, view, g = case["scene"], case["cam"], case["opt"], case["view"], case["g"]
    ref = case["ref"]
    mask = ref["flags"] == 0
    cot = {k: (v * mask).astype(np.float32) for k, v in sg.cotangents(17, cam.width, cam.height).items()}
    c = {k: torch.as_tensor(v).contiguous().cuda() for k, v in cot.items()}
    ga, gb = g.zeros_like(means2d=True), g.zeros_like()
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], ga)
    P.rd_render_bwd(view, g, c["color"], c["depth"], c["normal"], c["alpha"], gb)
    torch.cuda.synchronize()
    vis = np.nonzero(oracle.project(scene, cam, opt)[:, 0] == 1)[0]
    R = oracle.grad(scene, cam, opt, cot, vis, means2d=True)
    a, b = ga.means2d.double().cpu().numpy()[vis], R[:, 59:61]
    nb = np.linalg.norm(b)
    assert nb > 0
    assert np.linalg.norm(a - b) / nb <= 1e-3, np.linalg.norm(a - b) / nb
    med = np.median(np.abs(b[b != 0]))
    assert not (np.abs(a - b) > 1e-3 * np.abs(b) + 1e-3 * med).any()
    off = np.setdiff1d(np.arange(scene.n), vis)
    assert np.all(ga.means2d.cpu().numpy()[off] == 0)
    A, B = grads_to_rows(ga, scene.n), grads_to_rows(gb, scene.n)
    assert np.linalg.norm(A - B) <= 1e-5 * np.linalg.norm(B)


def test_cull_counters_by_reason():
    """Per-primitive invalidity is a cull, not an error; the profiling
    counters (rd_timings.n_culled) attribute each culled Gaussian to the first reason that
    applies: invalid input, near plane, guard band (S6b), opacity, degenerate, off screen."""
    cam = sg.camera_identity(40, 24, 40)
    scene = concat(one_gaussian([0, 0, 3], [0.1, -0.1, 0.1]),                  # invalid: scale ≤ 0
                   one_gaussian([0, 0, 3], [0.1] * 3, quat=(0, 0, 0, 0)),      # invalid: zero quaternion
                   one_gaussian([np.nan, 0, 3], [0.1] * 3),                    # invalid: NaN mean
                   one_gaussian([0, 0, -3], [0.1] * 3),                        # near: behind the camera
                   one_gaussian([0, 0, 0.1], [0.1] * 3),                       # near: z < znear
                   one_gaussian([12.0, 0, 3], [0.01] * 3),                     # guard band (u ≈ 180 px)
                   one_gaussian([0, 0, 3], [0.1] * 3, opacity=1e-3),           # opacity < alpha_min
                   one_gaussian([0.2, 0.1, 3], [0.1] * 3))                     # visible
    reasons = ("invalid", "near", "guard_band", "opacity", "degenerate", "off_screen")
    for gb, exp in ((0.15, (3, 2, 1, 1, 0, 0)), (0.0, (3, 2, 0, 1, 0, 1))):  # band off: off screen instead
        g = P.Gaussians.from_numpy(scene)
        view = P.View()
        P.rd_set_profiling(view, True)
        P.rd_preprocess(view, g, cam, opts_dict(sg.Options(guard_band=gb)))
        P.rd_bin(view)
        P.rd_render_fwd(view)
        t = P.rd_get_timings(view, reset=True)
        assert tuple(t["n_culled"][r] for r in reasons) == exp, (gb, t["n_culled"])
        assert t["n_visible"] == 1
