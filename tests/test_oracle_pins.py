"""Pins of the fp64 oracle against things other than itself (closed forms, textbook
identities, library routines for sub-steps, brute force on tiny inputs, SPEC examples).

Each test names the PAPER.md lines of the step it pins. None of these call the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import scenegen as sg
from helpers import concat, dense_scene, one_gaussian, quat_to_rot_scipy, random_cam

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
OPT = sg.Options()


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def _pg(O, scene, cam, opt=OPT):
    return O.project(scene, cam, opt)


def _f32cam(cam):
    return O_cam(cam)


def O_cam(cam):
    import oracle
    return oracle._cam_f32(cam)


# ----------------------------------------------------------------------------- Σ

@pytest.mark.parametrize("case", GOLD["covariance"])
def test_covariance_golden(O, case):
    sc = one_gaussian([0, 0, 3], case["scales"], case["quat_wxyz"])
    pg = _pg(O, sc, sg.camera_identity(32, 32, 32))[0]
    assert pg[O.PG["valid"]] == 1
    np.testing.assert_allclose(pg[O.PG["Sigma"]].reshape(3, 3), case["sigma"], atol=1e-7)


def test_covariance_vs_scipy_rotation(O):
    rng = np.random.default_rng(0)
    for _ in range(20):
        q = rng.normal(size=4) * rng.uniform(0.2, 3.0)  # raw, unnormalised (reading S15)
        s = np.exp(rng.uniform(-4, 0, 3))
        sc = one_gaussian([0.1, -0.2, 4.0], s, q)
        pg = _pg(O, sc, sg.camera_identity(32, 32, 32))[0]
        qf = sc.rotations[:, 0].astype(np.float64)
        sf = sc.scales[:, 0].astype(np.float64)
        R = quat_to_rot_scipy(qf)
        ref = R @ np.diag(sf ** 2) @ R.T
        np.testing.assert_allclose(pg[O.PG["Sigma"]].reshape(3, 3), ref, rtol=1e-12, atol=1e-15)


# ----------------------------------------------------------------------------- J

def _uvt(cam, x):
    return np.array([cam.fx * x[0] / x[2] + cam.cx, cam.fy * x[1] / x[2] + cam.cy, np.linalg.norm(x)])


def _fd_jac(cam, x, h=1e-6):
    J = np.zeros((3, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h * max(1.0, abs(x[k]))
        J[:, k] = (_uvt(cam, x + e) - _uvt(cam, x - e)) / (2 * e[k])
    return J


def test_jacobian_vs_finite_differences(O):
    rng = np.random.default_rng(1)
    for _ in range(10):
        cam = O_cam(random_cam(rng))
        sc = one_gaussian(rng.normal(scale=0.3, size=3), [0.1, 0.1, 0.1])
        pg = _pg(O, sc, cam)[0]
        assert pg[0] == 1
        x = pg[O.PG["x"]]
        np.testing.assert_allclose(pg[O.PG["J"]].reshape(3, 3), _fd_jac(cam, x), rtol=1e-7, atol=1e-9)
        # the pinhole projection itself: (u_c, v_c, t_c) equal the (u, v, t) map at x_c
        np.testing.assert_allclose([pg[O.PG["u"]], pg[O.PG["v"]], pg[O.PG["tc"]]], _uvt(cam, x), rtol=1e-13)


# ----------------------------------------------------------------------------- Σ′, q̂, t*

def _independent_sigma_prime(cam, sc):
    """Σ′ = J W Σ Wᵀ Jᵀ built from scipy's rotation and a finite-difference J."""
    q = sc.rotations[:, 0].astype(float)
    s = sc.scales[:, 0].astype(float)
    R = quat_to_rot_scipy(q)
    Sig = R @ np.diag(s ** 2) @ R.T
    W = np.asarray(cam.R, float)
    x = W @ sc.means[:, 0].astype(float) + np.asarray(cam.t, float)
    Sc = W @ Sig @ W.T
    J = _fd_jac(cam, x)
    return J @ Sc @ J.T, x, Sc


def _argmax_1d(f, lo, hi):
    """Brute-force maximiser of a 1-D function: dense grid, then golden section."""
    ts = np.linspace(lo, hi, 20001)
    vals = f(ts)
    k = int(np.argmax(vals))
    a, b = ts[max(k - 1, 0)], ts[min(k + 1, len(ts) - 1)]
    g = (np.sqrt(5) - 1) / 2
    for _ in range(200):
        c, d = b - g * (b - a), a + g * (b - a)
        if f(np.array([c]))[0] > f(np.array([d]))[0]:
            b = d
        else:
            a = c
    return 0.5 * (a + b)


def test_sigma_prime_and_ray_space_maximum_bruteforce(O):
    """PAPER:413-416 (Eq.2) and PAPER:497-522 (Eq.9-13): the closed-form t* is the maximiser
    of the ray-space 1D Gaussian G′¹(t) (Eq.10), checked by brute-force search."""
    rng = np.random.default_rng(2)
    for trial in range(6):
        cam = O_cam(random_cam(rng))
        flat = [1.0, 0.3, 0.05][trial % 3]
        sc = one_gaussian(rng.normal(scale=0.3, size=3), np.array([0.2, 0.1, 0.2 * flat]), rng.normal(size=4))
        pg = _pg(O, sc, cam)[0]
        assert pg[0] == 1
        Sp, x, _ = _independent_sigma_prime(cam, sc)
        np.testing.assert_allclose(pg[O.PG["Sp"]].reshape(3, 3), Sp, rtol=2e-6, atol=1e-9 * np.abs(Sp).max())
        Spi = np.linalg.inv(Sp)
        uc = np.array([pg[O.PG["u"]], pg[O.PG["v"]], pg[O.PG["tc"]]])
        sd = np.sqrt(Sp[2, 2])
        pts = uc[:2] + rng.normal(scale=2.0, size=(8, 2)) * np.sqrt(np.diag(Sp)[:2])
        ev = O.splat_eval(sc, cam, OPT, 0, pts)
        # α = o·exp(−½ Δᵀ (Σ′[0:2,0:2] + hI)⁻¹ Δ) (readings S1, S5)
        A2 = Sp[:2, :2] + float(np.float32(0.3)) * np.eye(2)
        dl = uc[:2][None, :] - pts
        a_ref = float(sc.opacities[0]) * np.exp(-0.5 * np.einsum("ni,ij,nj->n", dl, np.linalg.inv(A2), dl))
        np.testing.assert_allclose(ev[:, 0], a_ref, rtol=1e-5)
        for k, (u, v) in enumerate(pts):
            def G(t):
                w = np.stack([np.full_like(t, u - uc[0]), np.full_like(t, v - uc[1]), t - uc[2]], 0)
                return np.exp(-np.einsum("in,ij,jn->n", w, Spi, w))
            tb = _argmax_1d(G, uc[2] - 30 * sd, uc[2] + 30 * sd)
            assert abs(ev[k, 1] - tb) <= 1e-6 * uc[2], (ev[k, 1], tb)
            # Eq.15: d = (z_c/t_c) t*
            assert abs(ev[k, 2] - pg[O.PG["z"]] / uc[2] * ev[k, 1]) <= 1e-12 * uc[2]


def test_conditional_mean_identity(O):
    """The maximum of a Gaussian along t at fixed (u, v) is the conditional mean
    t_c + Σ′_{t,uv} Σ′_{uv,uv}⁻¹ (uv − uv_c) (textbook), i.e. q = −Σ′_{uv,uv}⁻¹ Σ′_{uv,t}."""
    rng = np.random.default_rng(3)
    for _ in range(10):
        cam = O_cam(random_cam(rng))
        sc = one_gaussian(rng.normal(scale=0.3, size=3), np.exp(rng.uniform(-3, -1, 3)), rng.normal(size=4))
        pg = _pg(O, sc, cam)[0]
        Sp, _, _ = _independent_sigma_prime(cam, sc)
        A = Sp[:2, :2]
        q_ref = -np.linalg.solve(A, Sp[:2, 2])
        np.testing.assert_allclose(pg[O.PG["q"]], q_ref, rtol=1e-5, atol=1e-9)


def test_qhat_normalisation_and_q_p_relation(O):
    """q̂·v′ = 1, p = (z_c/t_c) q."""
    rng = np.random.default_rng(4)
    cam = O_cam(random_cam(rng))
    sc = dense_scene(4, 50)
    pg = _pg(O, sc, sg.camera_identity(64, 64, 64))
    v = pg[:, 0] == 1
    np.testing.assert_allclose(pg[v, 62], 1.0, rtol=0, atol=1e-15)
    zt = (pg[v, O.PG["z"]] / pg[v, O.PG["tc"]])[:, None]
    np.testing.assert_allclose(pg[v][:, O.PG["p"]], zt * pg[v][:, O.PG["q"]], rtol=1e-15)


def test_centre_identity_and_planarity(O):
    """d(u_c, v_c) = z_c (PAPER:535-550 and appendix); the ray-space
    intersection points lie on the plane (q, 1)·(𝐮 − 𝐮_c) = 0."""
    rng = np.random.default_rng(5)
    for _ in range(10):
        cam = O_cam(random_cam(rng))
        sc = one_gaussian(rng.normal(scale=0.3, size=3), np.exp(rng.uniform(-4, -1, 3)), rng.normal(size=4))
        pg = _pg(O, sc, cam)[0]
        uc, vc, tc, z = pg[O.PG["u"]], pg[O.PG["v"]], pg[O.PG["tc"]], pg[O.PG["z"]]
        ev = O.splat_eval(sc, cam, OPT, 0, [[uc, vc]])
        assert abs(ev[0, 1] - tc) <= 1e-13 * tc
        assert abs(ev[0, 2] - z) <= 1e-13 * tc
        pts = np.array([uc, vc]) + rng.normal(scale=5.0, size=(50, 2))
        ev = O.splat_eval(sc, cam, OPT, 0, pts)
        q = pg[O.PG["q"]]
        res = q[0] * (pts[:, 0] - uc) + q[1] * (pts[:, 1] - vc) + (ev[:, 1] - tc)
        assert np.abs(res).max() <= 1e-9 * tc


# ----------------------------------------------------------------------------- normal

def test_normal_is_conjugate_direction(O):
    """n = Jᵀ n′ normalised equals −Σ_c⁻¹x_c/‖·‖ (derived: q̂ J ∝ x_cᵀΣ_c⁻¹),
    computed here from scipy's rotation, independent of J and the intrinsics."""
    rng = np.random.default_rng(6)
    for _ in range(20):
        cam = O_cam(random_cam(rng))
        sc = one_gaussian(rng.normal(scale=0.3, size=3), np.exp(rng.uniform(-4, -1, 3)), rng.normal(size=4))
        pg = _pg(O, sc, cam)[0]
        _, x, Sc = _independent_sigma_prime(cam, sc)
        m = -np.linalg.solve(Sc, x)
        m /= np.linalg.norm(m)
        n = pg[O.PG["n"]]
        assert np.linalg.norm(n - m) < 1e-8
        assert np.dot(n, x) < 0  # toward the image plane


def test_isotropic_gaussian(O):
    """Isotropic: Σ′ has v′ as eigenvector ⇒ q = p = 0, d ≡ z_c, n = −x̂_c; at the centre
    pixel the rasterized depth equals the perspective ray maximum of Eq.7."""
    g = GOLD["isotropic_on_axis"]
    sc = one_gaussian(g["mean"], g["scales"])
    pg = _pg(O, sc, sg.camera_identity(64, 64, 64))[0]
    np.testing.assert_allclose(pg[O.PG["q"]], g["q"], atol=1e-15)
    np.testing.assert_allclose(pg[O.PG["p"]], g["p"], atol=1e-15)
    np.testing.assert_allclose(pg[O.PG["n"]], g["n"], atol=1e-15)
    rng = np.random.default_rng(7)
    for _ in range(10):
        # W = I exactly (an fp32 look-at rotation is orthonormal only to 1e-7, which would
        # make W Σ Wᵀ slightly anisotropic)
        cam = sg.Camera(rng.uniform(40, 80), rng.uniform(40, 80), rng.uniform(20, 40), rng.uniform(20, 30), 64, 48,
                        np.eye(3, dtype=np.float32), np.zeros(3, np.float32), 0.2)
        s = np.exp(rng.uniform(-4, -1))
        z = rng.uniform(2, 6)
        sc = one_gaussian([rng.uniform(-0.4, 0.4) * z, rng.uniform(-0.3, 0.3) * z, z], [s, s, s], rng.normal(size=4))
        pg = _pg(O, sc, cam)[0]
        x = pg[O.PG["x"]]
        assert np.abs(pg[O.PG["q"]]).max() < 1e-12 * pg[O.PG["tc"]]
        np.testing.assert_allclose(pg[O.PG["n"]], -x / np.linalg.norm(x), atol=1e-12)
        uc, vc = pg[O.PG["u"]], pg[O.PG["v"]]
        ev = O.splat_eval(sc, cam, OPT, 0, [[uc, vc], [uc + 3.0, vc - 2.0]])
        assert abs(ev[0, 4] - pg[O.PG["z"]]) < 1e-12 * pg[O.PG["tc"]]  # perspective depth at centre
        assert abs(ev[0, 2] - pg[O.PG["z"]]) < 1e-12 * pg[O.PG["tc"]]  # rasterized depth at centre
        assert abs(ev[1, 2] - pg[O.PG["z"]]) < 1e-12 * pg[O.PG["tc"]]  # d ≡ z_c off-centre too


def test_flattened_gaussian_normal_converges_to_splat_normal(O):
    """As s_min/s_max → 0 the rasterized normal → ±R_c e_min: the angle
    decreases quadratically with the flatness."""
    rng = np.random.default_rng(8)
    for _ in range(5):
        cam = O_cam(random_cam(rng))
        q = rng.normal(size=4)
        mean = rng.normal(scale=0.3, size=3)
        q32 = q.astype(np.float32).astype(float)  # the value the scene stores
        Rc = np.asarray(cam.R, float) @ quat_to_rot_scipy(q32 / np.linalg.norm(q32))
        e = Rc[:, 2]
        x = np.asarray(cam.R, float) @ mean + np.asarray(cam.t, float)
        if abs(np.dot(e, x / np.linalg.norm(x))) < 0.3:  # avoid near-grazing splats
            continue
        angs = []
        for eps in (1e-1, 1e-2, 1e-3):
            sc = one_gaussian(mean, [0.2, 0.15, 0.2 * eps], q)
            n = _pg(O, sc, cam)[0][O.PG["n"]]
            angs.append(np.degrees(np.arctan2(np.linalg.norm(np.cross(n, e)), abs(np.dot(n, e)))))
        assert angs[0] < 5.0 and angs[2] < 1e-3
        # quadratic convergence: each 10x flatter splat cuts the angle ~100x
        assert angs[1] < 0.02 * angs[0] and angs[2] < 0.02 * angs[1]


# ----------------------------------------------------------------------------- SH

def _real_sh_scipy(l, m, d):
    from scipy.special import sph_harm_y
    x, y, z = d
    theta = np.arccos(np.clip(z, -1, 1))
    phi = np.arctan2(y, x)
    Y = sph_harm_y(l, abs(m), theta, phi)  # includes the Condon-Shortley phase
    if m < 0:
        return np.sqrt(2) * (-1) ** m * Y.imag
    if m > 0:
        return np.sqrt(2) * (-1) ** m * Y.real
    return Y.real


def test_sh_basis_vs_scipy(O):
    rng = np.random.default_rng(9)
    for _ in range(50):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        B = O.sh_basis(d)
        for l in range(4):
            for m in range(-l, l + 1):
                # reading S14: 3DGS basis = (−1)^m × standard real SH
                ref = (-1) ** m * _real_sh_scipy(l, m, d)
                assert abs(B[l * l + l + m] - ref) < 1e-12, (l, m)


def test_sh_degree0_and_zero_dc(O):
    cam = sg.camera_identity(32, 32, 32)
    sc0 = one_gaussian([0, 0, 3], [0.1] * 3, dc=(0, 0, 0))
    np.testing.assert_allclose(_pg(O, sc0, cam)[0][O.PG["rgb"]], GOLD["sh_zero_dc"]["rgb"], atol=0)
    rgbs = []
    for mean in ([0, 0, 3], [1, 0.5, 3], [-1, -1, 4]):
        sc = one_gaussian(mean, [0.1] * 3, dc=(0.7, -0.3, 0.2))
        rgbs.append(_pg(O, sc, cam, sg.Options(sh_degree=0))[0][O.PG["rgb"]])
    np.testing.assert_allclose(rgbs[0], rgbs[1], atol=1e-15)
    np.testing.assert_allclose(rgbs[0], rgbs[2], atol=1e-15)


# ----------------------------------------------------------------------------- blending / median

def _empty_scene():
    return sg.make_scene(np.zeros((3, 0)), np.zeros((3, 0)), np.zeros((4, 0)), np.zeros(0), np.zeros((16, 3, 0)))


def test_empty_scene_renders_zeros(O):
    r = O.render(_empty_scene(), sg.camera_identity(16, 8, 16), OPT)
    for k in ("color", "depth", "normal", "alpha"):
        assert np.all(r[k] == 0)


@pytest.mark.parametrize("case", GOLD["alpha_at_centre"]["cases"])
def test_single_splat_at_centre(O, case):
    """Pixel whose centre is the splat centre: C = c·min(o, α_max)."""
    cam = sg.camera_identity(64, 64, 64)
    z = 3.0
    # u_c = fx x/z + cx = 20.5 (centre of pixel 20), v_c = 40.5
    mean = [(20.5 - 32) * z / 64, (40.5 - 32) * z / 64, z]
    sc = one_gaussian(mean, [0.1, 0.08, 0.12], [0.9, 0.1, -0.2, 0.3], opacity=case["opacity"])
    pg = _pg(O, sc, cam)[0]
    r = O.render(sc, cam, OPT)
    a = case["alpha"]
    np.testing.assert_allclose(r["alpha"][40, 20], a, rtol=1e-7)
    np.testing.assert_allclose(r["color"][:, 40, 20], a * pg[O.PG["rgb"]], rtol=1e-7)
    np.testing.assert_allclose(r["normal"][:, 40, 20], a * pg[O.PG["n"]], rtol=1e-7, atol=1e-12)
    if a > 0.5:
        np.testing.assert_allclose(r["depth"][40, 20], pg[O.PG["z"]], rtol=1e-12)


def test_two_opaque_layers_median(O):
    """Median depth (reading S9) selects, not averages: with fronto-parallel flat
    splats on the principal axis (q = 0 ⇒ d = z_c), D = 2.0 where α₁ > 0.5 and 3.0 where
    only the two together cross 0.5."""
    g = GOLD["two_opaque_layers"]
    cam = sg.camera_identity(64, 64, 64)
    o = g["opacity"]
    front = one_gaussian([0, 0, g["front_depth"]], [0.15, 0.15, 1e-3], opacity=o)
    back = one_gaussian([0, 0, g["back_depth"]], [0.6, 0.6, 1e-3], opacity=o)
    sc = concat(front, back)
    pg = _pg(O, sc, cam)
    np.testing.assert_allclose(pg[:, 63:67], 0.0, atol=1e-15)  # q = p = 0
    r = O.render(sc, cam, OPT)
    D = r["depth"]
    assert abs(D[32, 32] - g["median_at_centre"]) < 1e-12
    # analytic α of an isotropic screen Gaussian: σ² = (f s / z)² + h
    ii, jj = np.meshgrid(np.arange(64) + 0.5, np.arange(64) + 0.5)
    r2 = (ii - 32) ** 2 + (jj - 32) ** 2
    s1, s2 = float(front.scales[0, 0]), float(back.scales[0, 0])
    h = float(np.float32(0.3))
    a1 = np.minimum(0.99, o * np.exp(-0.5 * r2 / ((64 * s1 / 2.0) ** 2 + h)))
    a2 = np.minimum(0.99, o * np.exp(-0.5 * r2 / ((64 * s2 / 3.0) ** 2 + h)))
    a1 = np.where(a1 >= 1 / 255, a1, 0.0)
    a2 = np.where(a2 >= 1 / 255, a2, 0.0)
    T1 = 1 - a1
    T2 = T1 * (1 - a2)
    expect = np.where(T1 <= 0.5, 2.0, np.where(T2 <= 0.5, 3.0, 0.0))
    ok = (np.abs(T1 - 0.5) > 1e-6) & (np.abs(T2 - 0.5) > 1e-6)
    np.testing.assert_allclose(D[ok], expect[ok], rtol=0, atol=1e-12)
    assert (expect == 3.0).sum() > 20 and (expect == 2.0).sum() > 20
    mean_depth = (2.0 * 0.99 + 3.0 * 0.01 * 0.99) / (0.99 + 0.0099)
    assert abs(mean_depth - g["expected_depth_at_centre_if_mean"]) < 1e-4


def test_weights_sum_identity_and_median_property(O):
    """Σω + T_final = 1 (telescoping Eq.3): with every colour = 1 and bg = 0
    the colour channel equals α = 1 − T. When D ≠ 0 it equals d (Eq.15) of exactly the
    median splat at that pixel."""
    sc = dense_scene(10, 300)
    sc.sh[:] = 0
    sc.sh[0] = 0.5 / 0.28209479177387814  # rgb = 1
    cam = sg.camera_identity(64, 64, 64)
    r = O.render(sc, cam, OPT)
    for c in range(3):
        np.testing.assert_allclose(r["color"][c], r["alpha"], atol=1e-12)
    assert r["nblend"].mean() > 3
    ys, xs = np.nonzero(r["depth"])
    assert len(ys) > 100
    rng = np.random.default_rng(0)
    for k in rng.choice(len(ys), 40, replace=False):
        y, x = ys[k], xs[k]
        gid = int(r["median_id"][y, x])
        ev = O.splat_eval(sc, cam, OPT, gid, [[x + 0.5, y + 0.5]])
        assert ev[0, 2] == pytest.approx(r["depth"][y, x], rel=1e-13)


def test_tile_free_subset_render_matches_full(O):
    """Rendering a pixel subset gives the same values as the full frame (pure per-pixel
    definition; no tiling anywhere in the oracle)."""
    sc = dense_scene(11, 120)
    cam = sg.camera_identity(64, 64, 64)
    full = O.render(sc, cam, OPT)
    pix = np.array([0, 5, 64 * 10 + 3, 64 * 63 + 63, 2000])
    sub = O.render(sc, cam, OPT, pixels=pix)
    for k in ("color", "normal"):
        np.testing.assert_array_equal(sub[k], full[k].reshape(3, -1)[:, pix])
    for k in ("depth", "alpha", "flags", "nblend"):
        np.testing.assert_array_equal(sub[k], full[k].reshape(-1)[pix])


# ----------------------------------------------------------------------------- gradients

def _loss(O, sc, cam, cot, opt=OPT):
    return O.loss(O.render(sc, cam, opt), cot)


def _set_param(sc, j, gid, value):
    if j < 3:
        sc.means[j, gid] = value
    elif j < 6:
        sc.scales[j - 3, gid] = value
    elif j < 10:
        sc.rotations[j - 6, gid] = value
    elif j == 10:
        sc.opacities[gid] = value
    else:
        k = j - 11
        sc.sh[k // 3, k % 3, gid] = value


def _get_param(sc, j, gid):
    if j < 3:
        return sc.means[j, gid]
    if j < 6:
        return sc.scales[j - 3, gid]
    if j < 10:
        return sc.rotations[j - 6, gid]
    if j == 10:
        return sc.opacities[gid]
    k = j - 11
    return sc.sh[k // 3, k % 3, gid]


def _double_scene(sc):
    d = sc.copy()
    for k in ("means", "scales", "rotations", "opacities", "sh"):
        setattr(d, k, getattr(d, k).astype(np.float64))
    return d


def test_dual_gradient_vs_central_fd(O):
    """The oracle's forward-mode dual gradient equals central finite differences of its own
    render, away from the flagged kinks."""
    sc = _double_scene(dense_scene(12, 40, smin=0.05))
    cam = sg.camera_identity(48, 48, 48)
    cot = sg.cotangents(3, 48, 48)
    r = O.render(sc, cam, OPT)
    m = r["flags"] == 0
    for k in cot:
        cot[k] = cot[k] * m
    pg = _pg(O, sc, cam)
    cand = [i for i in range(sc.n) if pg[i, 0] == 1 and not pg[i, 73:76].any()]
    gids = np.array(cand[:4])
    G = O.grad(sc, cam, OPT, cot, gids)
    params = list(range(11)) + [11, 13, 14, 16, 30, 58]
    checked = 0
    for gk, gid in enumerate(gids):
        for j in params:
            x0 = _get_param(sc, j, gid)
            h = 1e-6 * max(abs(x0), 0.05)
            _set_param(sc, j, gid, x0 + h)
            Lp = _loss(O, sc, cam, cot)
            _set_param(sc, j, gid, x0 - h)
            Lm = _loss(O, sc, cam, cot)
            _set_param(sc, j, gid, x0)
            fd = (Lp - Lm) / (2 * h)
            scale = max(abs(G[gk, j]), 1e-3 * np.abs(G[gk]).max(), 1e-6)
            assert abs(fd - G[gk, j]) <= 2e-5 * scale + 1e-7, (gid, j, fd, G[gk, j])
            checked += 1
    assert checked > 50


def test_zero_cotangent_gives_zero_gradient(O):
    sc = dense_scene(13, 30)
    cam = sg.camera_identity(32, 32, 32)
    z = {k: np.zeros_like(v) for k, v in sg.cotangents(0, 32, 32).items()}
    G = O.grad(sc, cam, OPT, z, np.arange(30))
    assert np.all(G == 0)


# ----------------------------------------------------------------------------- guard band (S6b)

@pytest.mark.parametrize("axis", [0, 1])
def test_guard_band_cull(O, axis):
    """Reading S6b (optional, rd_options.guard_band = 0.15): a centre projecting outside
    [−0.15, 1.15]× the image is culled. Pinned by placing a wide splat just inside / just
    outside each edge (closed-form pixel position u = fx·x/z + cx) and checking that it is
    kept and reaches into the image, or culled and contributes nothing; with the band off
    (the default) every one of them is kept and reaches into the image."""
    cam = sg.camera_identity(64, 48, 60.0)
    OPT_G = sg.Options(guard_band=0.15)
    size = (cam.width, cam.height)[axis]
    f = (cam.fx, cam.fy)[axis]
    c = (cam.cx, cam.cy)[axis]
    z = 3.0
    lo, hi = -0.15 * size, 1.15 * size
    for target in (hi - 0.5, hi + 0.5, lo + 0.5, lo - 0.5):
        keep = lo <= target <= hi
        pos = [0.0, 0.0, z]
        pos[axis] = (target - c) * z / f
        sc = one_gaussian(pos, [1.0, 1.0, 1.0], opacity=0.9)
        pg = O.project(sc, cam, OPT_G)
        assert (pg[0, 0] == 1) == keep, (axis, target)
        out = O.render(sc, cam, OPT_G)
        if keep:
            assert out["alpha"].max() > 0.05  # σ ≈ 20 px: its footprint reaches into the image
        else:
            assert out["alpha"].max() == 0.0
        assert O.project(sc, cam, OPT)[0, 0] == 1  # band off: kept
        assert O.render(sc, cam, OPT)["alpha"].max() > 0.05


# ----------------------------------------------------------------------------- L_d

def _two_layers(o=0.9):
    """Fronto-parallel flat splats on the principal axis (q = p = 0 ⇒ d = z_c at every pixel),
    depths 2 and 3; at the centre pixel α = o exactly for both."""
    front = one_gaussian([0, 0, 2.0], [0.15, 0.15, 1e-3], opacity=o)
    back = one_gaussian([0, 0, 3.0], [0.6, 0.6, 1e-3], opacity=o)
    return concat(front, back)


def _two_layer_alphas(r2):
    """Analytic α of the two isotropic screen Gaussians: σ² = (f s / z)² + h (S5), with the
    fp32 values the renderer receives."""
    h = float(np.float32(0.3))
    o, s1, s2 = (float(np.float32(x)) for x in (0.9, 0.15, 0.6))
    a1 = o * np.exp(-0.5 * r2 / ((64 * s1 / 2.0) ** 2 + h))
    a2 = o * np.exp(-0.5 * r2 / ((64 * s2 / 3.0) ** 2 + h))
    return a1, a2


def test_depth_distortion_two_layers_closed_form(O):
    """L_d = Σ_i Σ_j ω_i ω_j (d_i − d_j)² with ω = (α₁, α₂(1 − α₁)) and
    d = (2, 3): 2·ω₁·ω₂·1² (the double sum counts (i, j) and (j, i)) at every pixel, with
    the α of the analytic isotropic screen Gaussians."""
    cam = sg.camera_identity(64, 64, 64)
    r = O.render(_two_layers(), cam, OPT)
    ii, jj = np.meshgrid(np.arange(64) + 0.5, np.arange(64) + 0.5)
    r2 = (ii - 32) ** 2 + (jj - 32) ** 2
    a1, a2 = _two_layer_alphas(r2)
    a1 = np.where(a1 >= 1 / 255, a1, 0.0)
    a2 = np.where(a2 >= 1 / 255, a2, 0.0)
    expect = 2 * a1 * (1 - a1) * a2 * 1.0
    np.testing.assert_allclose(r["distortion"], expect, rtol=1e-9, atol=1e-14)
    assert expect[32, 32] > 0.17


def test_depth_distortion_gradient_detached_weights(O):
    """Reading S21 (ω detached): dL_d/dμ_z of the back layer at a pixel is
    ∂L_d/∂d₂ = 4 ω₂ (A d₂ − D₁) with A = Σω, D₁ = Σωd, since d₂ = z_c moves one-for-one
    with μ_z (q = p = 0, centre on the axis) and the weights carry no derivative."""
    cam = sg.camera_identity(64, 64, 64)
    sc = _two_layers()
    zero = {"color": np.zeros((3, 64, 64)), "depth": np.zeros((64, 64)), "normal": np.zeros((3, 64, 64)),
            "alpha": np.zeros((64, 64)), "distortion": np.zeros((64, 64))}
    zero["distortion"][32, 32] = 1.0
    G = O.grad(sc, cam, OPT, zero, [0, 1])
    a1, a2 = _two_layer_alphas(0.5)
    w1, w2, d1, d2 = a1, a2 * (1 - a1), 2.0, 3.0
    A, D1 = w1 + w2, w1 * d1 + w2 * d2
    assert G[1, 2] == pytest.approx(4 * w2 * (A * d2 - D1), rel=1e-9)
    assert G[0, 2] == pytest.approx(4 * w1 * (A * d1 - D1), rel=1e-9)
    assert abs(G[1, 10]) < 1e-12  # opacity enters only through ω: detached


def test_depth_distortion_one_pass_identity(O):
    """Σ_ij ω_i ω_j (d_i − d_j)² = 2 (A·D₂ − D₁²) (expansion of the square), and
    L_d ≥ 0: checked on a dense random scene through per-pixel (ω, d) lists rebuilt from the
    oracle's own per-splat evaluation."""
    sc = dense_scene(12, 120)
    cam = sg.camera_identity(32, 32, 32)
    r = O.render(sc, cam, OPT)
    assert (r["distortion"] >= -1e-12).all() and r["distortion"].max() > 1e-3
    pg = O.project(sc, cam, OPT)
    order = [i for i in np.lexsort((np.arange(sc.n), pg[:, 1])) if pg[i, 0] == 1]
    rng = np.random.default_rng(1)
    for _ in range(20):
        y, x = rng.integers(0, 32, 2)
        T, A, D1, D2 = 1.0, 0.0, 0.0, 0.0
        for gid in order:
            ev = O.splat_eval(sc, cam, OPT, int(gid), [[x + 0.5, y + 0.5]])
            a = min(0.99, ev[0, 0])
            if a < 1 / 255:
                continue
            if T * (1 - a) < 1e-4:
                break
            w = a * T
            A, D1, D2 = A + w, D1 + w * ev[0, 2], D2 + w * ev[0, 2] ** 2
            T *= 1 - a
        assert r["distortion"][y, x] == pytest.approx(2 * (A * D2 - D1 * D1), rel=1e-7, abs=1e-10)


# ----------------------------------------------------------------------------- L_n

def test_depth_normal_planes(O):
    """Reading S22: finite-difference normals of an analytically rendered
    plane. Fronto-parallel → (0, 0, −1) everywhere interior; a tilted plane n·X = c →
    ±n (oriented so ñ·P < 0) to rounding; the last row/column are 0."""
    cam = sg.Camera(50.0, 55.0, 20.3, 14.7, 40, 30, np.eye(3), np.zeros(3), 0.2)
    D = np.full((30, 40), 3.5)
    nt = O.depth_normal(D, cam)
    np.testing.assert_allclose(nt[:, :-1, :-1], np.broadcast_to(np.array([0, 0, -1.0])[:, None, None], (3, 29, 39)),
                               atol=1e-12)
    assert np.all(nt[:, -1, :] == 0) and np.all(nt[:, :, -1] == 0)
    n = np.array([0.3, -0.2, -0.9])
    n /= np.linalg.norm(n)
    c = -4.0  # n·X = c, in front of the camera (X_z > 0)
    fx, fy, cx, cy = 50.0, 55.0, 20.3, 14.7
    xs = (np.arange(40) + 0.5 - cx) / fx
    ys = (np.arange(30) + 0.5 - cy) / fy
    r = np.stack([np.broadcast_to(xs[None, :], (30, 40)), np.broadcast_to(ys[:, None], (30, 40)),
                  np.ones((30, 40))], 0)
    D = c / np.einsum("k,kyx->yx", n, r)
    assert (D > 0).all()
    nt = O.depth_normal(D, cam)
    expect = n if (n @ r[:, 5, 5]) * D[5, 5] < 0 else -n
    np.testing.assert_allclose(nt[:, :-1, :-1], np.broadcast_to(expect[:, None, None], (3, 29, 39)), atol=1e-9)


def test_depth_normal_holes(O):
    """A hole (D = 0) removes the normals of the three stencils that use it."""
    cam = sg.camera_identity(16, 12, 20.0)
    D = np.full((12, 16), 2.0)
    D[5, 7] = 0.0
    nt = O.depth_normal(D, cam)
    zero = np.all(nt == 0, 0)
    assert zero[5, 7] and zero[5, 6] and zero[4, 7]
    assert zero.sum() == 3 + 12 + 16 - 1


def test_normal_consistency_flat_splat_is_zero(O):
    """A fronto-parallel flat splat has n = (0, 0, −1) = ñ of its constant depth, so
    L_n = A − N·ñ = A − A = 0 wherever it alone is blended; L_n ∈ [0, 2A] always."""
    cam = sg.camera_identity(32, 32, 32)
    sc = one_gaussian([0, 0, 2.0], [0.6, 0.6, 1e-4], opacity=0.8)
    r = O.render(sc, cam, OPT)
    L, nt = O.normal_consistency(r["depth"], r["alpha"], r["normal"], cam)
    valid = np.any(nt != 0, 0)
    assert valid.sum() > 200
    np.testing.assert_allclose(L[valid], 0.0, atol=1e-9)
    sc2 = dense_scene(14, 150, width=32, height=32, f=32.0)
    r2 = O.render(sc2, cam, OPT)
    L2, nt2 = O.normal_consistency(r2["depth"], r2["alpha"], r2["normal"], cam)
    v2 = np.any(nt2 != 0, 0)
    assert v2.sum() > 50
    assert (L2[v2] >= -1e-12).all() and (L2[v2] <= 2 * r2["alpha"][v2] + 1e-12).all()


# ----------------------------------------------------------------------------- 3D filter (S23)

def test_filter3d_covariance_and_mass(O):
    """Reading S23 (Mip-Splatting 3D filter): the filtered Gaussian's Σ' equals Σ + f²I
    (checked through the oracle's own Σ of both scenes), and o·√det Σ — the integral of
    o·exp(−½xᵀΣ⁻¹x) up to (2π)^{3/2} — is preserved."""
    sc = dense_scene(21, 20)
    f = np.random.default_rng(2).uniform(0.01, 0.2, sc.n)
    fs, _ = O.apply_filter3d(sc, f)
    cam = sg.camera_identity(64, 64, 64)
    A, B = O.project(sc, cam, OPT), O.project(fs, cam, OPT)
    both = (A[:, 0] == 1) & (B[:, 0] == 1)
    assert both.sum() > 10
    Sa = A[both][:, 9:18].reshape(-1, 3, 3)
    Sb = B[both][:, 9:18].reshape(-1, 3, 3)
    np.testing.assert_allclose(Sb, Sa + (f[both] ** 2)[:, None, None] * np.eye(3), rtol=1e-12, atol=1e-14)
    mass_a = sc.opacities[both].astype(np.float64) * np.sqrt(np.linalg.det(Sa))
    mass_b = fs.opacities[both] * np.sqrt(np.linalg.det(Sb))
    np.testing.assert_allclose(mass_b, mass_a, rtol=1e-9)


def test_filter3d_gradient_vjp_vs_finite_differences(O):
    """The raw-parameter gradient (dual-number gradient of the filtered scene mapped through
    apply_filter3d's vjp) vs central differences of the filtered render in the raw scales
    and opacity."""
    sc = dense_scene(22, 30)
    cam = sg.camera_identity(32, 32, 32)
    f = np.random.default_rng(4).uniform(0.02, 0.1, sc.n)
    cot = sg.cotangents(5, 32, 32)
    fs, vjp = O.apply_filter3d(sc, f)
    pg = O.project(fs, cam, OPT)
    gid = int(np.nonzero(pg[:, 0] == 1)[0][3])
    G = vjp(O.grad(fs, cam, OPT, cot, [gid]), [gid])[0]

    def loss(scene):
        return O.loss(O.render(O.apply_filter3d(scene, f)[0], cam, OPT), cot)

    for j, (arr, idx) in enumerate([("scales", (0, gid)), ("scales", (2, gid)), ("opacities", (gid,))]):
        h = 1e-6
        sp, sm = sc.copy(), sc.copy()
        for s_, sgn in ((sp, 1), (sm, -1)):
            a = getattr(s_, arr).astype(np.float64)
            a[idx] += sgn * h
            setattr(s_, arr, a)
        fd = (loss(sp) - loss(sm)) / (2 * h)
        col = {0: 3, 1: 5, 2: 10}[j]
        assert G[col] == pytest.approx(fd, rel=2e-4, abs=1e-7), (arr, idx)


# ----------------------------------------------------------------------------- TSDF (S24)

def _tsdf_cam():
    return sg.Camera(60.0, 60.0, 32.0, 24.0, 64, 48, np.eye(3, dtype=np.float32), np.zeros(3, np.float32), 0.2)


def test_tsdf_plane_zero_crossing(O):
    """Reading S24: fusing the depth map of a fronto-parallel plane at depth d
    gives tsdf = (d − z)/τ exactly wherever |d − z| < τ, so each z-column's zero crossing
    lies at d (within ½ voxel of the voxel centres)."""
    cam = _tsdf_cam()
    d, vs = 2.03, 0.02
    tau = 4 * vs
    dims = (40, 10, 12)  # Z, Y, X
    tsdf, w = np.ones(dims), np.zeros(dims)
    origin = (-0.12, -0.1, 1.6)
    O.tsdf_integrate(tsdf, w, origin, vs, tau, 100.0, np.full((48, 64), d), cam)
    zc = origin[2] + (np.arange(dims[0]) + 0.5) * vs
    band = np.abs(d - zc) < tau
    assert (w[band] == 1).all()
    np.testing.assert_allclose(tsdf[band], np.broadcast_to(((d - zc[band]) / tau)[:, None, None],
                                                           (band.sum(), 10, 12)), atol=1e-6)
    col = tsdf[:, 5, 6]
    k = np.nonzero((col[:-1] > 0) & (col[1:] <= 0))[0][0]
    zero = zc[k] + col[k] / (col[k] - col[k + 1]) * vs
    assert abs(zero - d) < 0.5 * vs
    assert (w[zc < d - tau - 1e-6] == 1).all() and (w[zc > d + tau + 1e-6] == 0).all()


def test_tsdf_holes_twice_and_order(O):
    """Holes leave the volume unchanged; the same map twice gives the same tsdf and doubled
    weights; the weighted average does not depend on the view order."""
    cam = _tsdf_cam()
    rng = np.random.default_rng(0)
    dims, vs = (20, 12, 14), 0.05
    origin = (-0.35, -0.3, 1.5)
    t0, w0 = np.ones(dims), np.zeros(dims)
    O.tsdf_integrate(t0, w0, origin, vs, 0.2, 100.0, np.zeros((48, 64)), cam)
    assert (w0 == 0).all() and (t0 == 1).all()
    D1 = 2.0 + 0.1 * rng.random((48, 64))
    D2 = 2.1 + 0.1 * rng.random((48, 64))
    a, wa = np.ones(dims), np.zeros(dims)
    O.tsdf_integrate(a, wa, origin, vs, 0.2, 100.0, D1, cam)
    b, wb = a.copy(), wa.copy()
    O.tsdf_integrate(b, wb, origin, vs, 0.2, 100.0, D1, cam)
    np.testing.assert_allclose(b, a, atol=1e-15)
    np.testing.assert_array_equal(wb, 2 * wa)
    c, wc = np.ones(dims), np.zeros(dims)
    d, wd = np.ones(dims), np.zeros(dims)
    for D in (D1, D2):
        O.tsdf_integrate(c, wc, origin, vs, 0.2, 100.0, D, cam)
    for D in (D2, D1):
        O.tsdf_integrate(d, wd, origin, vs, 0.2, 100.0, D, cam)
    np.testing.assert_allclose(c, d, atol=1e-12)
    np.testing.assert_array_equal(wc, wd)
    assert (wc == 2).sum() > 100


# ----------------------------------------------------------------------------- marching cubes (S25)

def _sphere_volume(n=28, vs=0.1, R=0.9, center=(0.03, -0.02, 0.05)):
    origin = (-1.4, -1.4, -1.4)
    c = origin[0] + (np.arange(n) + 0.5) * vs
    Zc, Yc, Xc = np.meshgrid(c, c, c, indexing="ij")
    sdf = np.sqrt((Xc - center[0]) ** 2 + (Yc - center[1]) ** 2 + (Zc - center[2]) ** 2) - R
    tau = 4 * vs
    return np.clip(sdf / tau, -1, 1).astype(np.float32), np.ones((n, n, n), np.float32), origin, vs, R, center


def test_mc_sphere_accuracy_and_watertight(O):
    """Reading S25: the iso-surface of an analytic sphere's truncated SDF lies on
    the sphere (mean |d| < 0.05 voxel, max < 0.25 voxel; SPEC's bars are 0.5 / 1.5), and the
    triangle soup is a closed, consistently oriented surface: after merging equal vertices
    every directed edge occurs exactly once and its reverse exactly once; normals point out."""
    ts, w, origin, vs, R, ctr = _sphere_volume()
    m = O.marching_cubes(ts, w, origin, vs)
    assert len(m) > 1000
    d = np.linalg.norm(m.reshape(-1, 3) - np.array(ctr), axis=1) - R
    assert np.abs(d).mean() < 0.05 * vs and np.abs(d).max() < 0.25 * vs
    key = {tuple(np.round(p, 9)) for p in m.reshape(-1, 3)}
    idx = {p: k for k, p in enumerate(sorted(key))}
    tri = np.array([[idx[tuple(np.round(p, 9))] for p in t] for t in m])
    directed = {}
    for a, b, c in tri:
        for e in ((a, b), (b, c), (c, a)):
            directed[e] = directed.get(e, 0) + 1
    assert all(v == 1 for v in directed.values())
    assert all(directed.get((b, a), 0) == 1 for (a, b) in directed)
    nrm = np.cross(m[:, 1] - m[:, 0], m[:, 2] - m[:, 0])
    outward = np.einsum("ij,ij->i", nrm, m.mean(1) - np.array(ctr))
    assert (outward > 0).all()


def test_mc_plane_and_degenerate(O):
    """A planar SDF gives triangles whose normals are parallel to the plane normal; an
    all-positive volume and zero-weight corners give nothing."""
    n, vs = 12, 0.1
    origin = (0.0, 0.0, 0.0)
    c = origin[0] + (np.arange(n) + 0.5) * vs
    Zc, Yc, Xc = np.meshgrid(c, c, c, indexing="ij")
    nrm = np.array([0.2, -0.3, 0.93])
    nrm /= np.linalg.norm(nrm)
    sdf = (Xc * nrm[0] + Yc * nrm[1] + Zc * nrm[2] - 0.55).astype(np.float32)
    m = O.marching_cubes(sdf, np.ones_like(sdf), origin, vs)
    assert len(m) > 50
    tn = np.cross(m[:, 1] - m[:, 0], m[:, 2] - m[:, 0])
    tn /= np.linalg.norm(tn, axis=1, keepdims=True)
    np.testing.assert_allclose(tn, np.broadcast_to(nrm, tn.shape), atol=1e-6)
    assert len(O.marching_cubes(np.ones_like(sdf), np.ones_like(sdf), origin, vs)) == 0
    assert len(O.marching_cubes(sdf, np.zeros_like(sdf), origin, vs)) == 0


# ----------------------------------------------------------------------------- sort key and order (S7)

def _round_f32(q):
    """Round a rational to the nearest binary32 value, ties to even (normal range only):
    an fp32 rounding written from its definition, independent of any float hardware."""
    from fractions import Fraction
    if q == 0:
        return np.float32(0.0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()  # 2^e ≤ a < 2^(e+2)
    while a >= Fraction(2) ** (e + 1):
        e += 1
    while a < Fraction(2) ** e:
        e -= 1
    assert -126 <= e <= 127
    scaled = a / Fraction(2) ** (e - 23)  # in [2^23, 2^24)
    m = scaled.numerator // scaled.denominator
    rem = scaled - m
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and m % 2 == 1):
        m += 1
    v = Fraction(m) * Fraction(2) ** (e - 23)
    return np.float32(sign * float(v))  # exactly representable


def _fma_f32(a, b, c):
    """IEEE fused multiply-add in binary32: a·b + c computed exactly, rounded once."""
    from fractions import Fraction
    return _round_f32(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def test_zkey_fp32_fma_chain_exact(O):
    """Reading S7: the sort key is z_key = fma(W20, μx, fma(W21, μy, fma(W22, μz, t2))) in
    IEEE fp32. The oracle's value (C fmaf) equals, bit for bit, the chain evaluated with exact
    rational arithmetic and one round-to-nearest-even per fma (written from the IEEE
    definition here), over random cameras and Gaussians including near-tie values."""
    rng = np.random.default_rng(17)
    for trial in range(6):
        cam = O_cam(random_cam(rng))
        n = 200
        mu = rng.normal(scale=1.5, size=(3, n))
        mu[:, :20] = mu[:, 20:40] * (1 + 1e-7)  # near-equal keys
        sc = sg.make_scene(mu, np.full((3, n), 0.05), sg.random_quaternions(rng, n), np.full(n, 0.9),
                           np.zeros((16, 3, n)))
        pg = O.project(sc, cam, OPT)
        R = np.asarray(cam.R, np.float32).reshape(9)
        t = np.asarray(cam.t, np.float32)
        for i in range(n):
            m = sc.means[:, i]
            z = _fma_f32(R[6], m[0], _fma_f32(R[7], m[1], _fma_f32(R[8], m[2], t[2])))
            got = np.float32(pg[i, O.PG["zkey"]])
            assert got.view(np.uint32) == z.view(np.uint32), (trial, i, got, z)


def test_round_f32_helper_matches_numpy_on_exact_cases():
    """The helper itself: on values whose binary32 rounding numpy does in one step (float64
    inputs converted once), the two agree — including ties to even."""
    from fractions import Fraction
    rng = np.random.default_rng(3)
    for x in rng.normal(scale=10, size=200):
        assert _round_f32(Fraction(float(x))) == np.float32(x)
    one = Fraction(1)
    ulp = Fraction(1, 2 ** 23)
    assert _round_f32(one + ulp / 2) == np.float32(1.0)            # tie → even (1.0)
    assert _round_f32(one + 3 * ulp / 2) == np.float32(1.0 + 2 ** -22)  # tie → even (odd mantissa rounds up)


def test_order_tie_break_by_index(O):
    """PAPER:422 orders by depth; equal keys break by Gaussian index (reading S7; SPEC:168,
    172). Two co-located splats with different colours and opacities: at their common centre
    the blended colour is c_a·α_a + c_b·α_b·(1 − α_a) with a the LOWER id (closed form), and
    swapping the ids swaps the roles; oracle.order lists the lower id first."""
    cam = sg.camera_identity(32, 32, 32)
    pos = [(15.5 - 16) * 3.0 / 32, (15.5 - 16) * 3.0 / 32, 3.0]
    a = one_gaussian(pos, [0.2, 0.2, 0.2], opacity=0.6, dc=(1.0, 0.0, 0.0))
    b = one_gaussian(pos, [0.2, 0.2, 0.2], opacity=0.5, dc=(0.0, 1.0, 0.0))
    for first, second in ((a, b), (b, a)):
        sc = concat(first, second)
        assert list(O.order(sc, cam, OPT)) == [0, 1]
        pg = O.project(sc, cam, OPT)
        assert pg[0, O.PG["zkey"]] == pg[1, O.PG["zkey"]]
        out = O.render(sc, cam, OPT)
        a0, a1 = float(np.float32(first.opacities[0])), float(np.float32(second.opacities[0]))
        c0, c1 = pg[0, O.PG["rgb"]], pg[1, O.PG["rgb"]]
        np.testing.assert_allclose(out["color"][:, 15, 15], c0 * a0 + c1 * a1 * (1 - a0), rtol=1e-12)
    # many ties: the order is (z_key, id) — pinned against a plain sort of (z_key, id) tuples
    rng = np.random.default_rng(4)
    sc = dense_scene(9, 300)
    sc.means[2] = rng.choice([2.5, 3.0, 4.0], sc.n)  # identity camera: z_key = z exactly
    pg = O.project(sc, cam, OPT)
    ok = np.nonzero(pg[:, 0] == 1)[0]
    exp = [i for _, i in sorted((np.float32(pg[i, O.PG["zkey"]]), i) for i in ok)]
    assert list(O.order(sc, cam, OPT)) == exp
    assert len(set(np.float32(pg[ok, O.PG["zkey"]]))) == 3


def test_mc_exact_iso_corners_no_degenerate_triangles(O):
    """Reading S25: corner values equal to iso put vertices exactly on cube corners; every
    triangle that would have two vertices on one corner (zero area) is dropped, and all the
    others keep a positive area. Integer-valued volume with iso = 0 hits this everywhere."""
    rng = np.random.default_rng(21)
    t = rng.integers(-1, 2, (9, 9, 9)).astype(np.float32)
    tri = O.marching_cubes(t, np.ones_like(t), (0.0, 0.0, 0.0), 1.0, 0.0)
    assert tri.shape[0] > 100
    area = 0.5 * np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)
    assert area.min() > 1e-6
    # the table alone (no drop) would emit more: some were degenerate
    table = O.mc_table()
    n_all = 0
    for k in range(8):
        for j in range(8):
            for i in range(8):
                cfg = sum(1 << c for c in range(8) if t[k + (c >> 2 & 1), j + (c >> 1 & 1), i + (c & 1)] < 0)
                n_all += len(table[cfg]) if 0 < cfg < 255 else 0
    assert n_all > tri.shape[0]


def test_means2d_gradient_single_splat_closed_form(O):
    """The oracle's dL/d(u_c, v_c) (dual slots 59..60: the projected centre moved with every
    other per-splat quantity fixed) for ONE splat and colour + alpha cotangents equals the
    closed form Σ_px g(px)·∂α/∂u_c with α = o·exp(−½ΔᵀCΔ), Δ = centre − pixel, so
    ∂α/∂(u_c, v_c) = −α·CΔ (S1, S4) — C and α from the oracle's projection,
    pixels near the α_min / α_max kinks excluded."""
    cam = sg.camera_identity(48, 40, 50.0)
    sc = one_gaussian([0.13, -0.07, 2.5], [0.12, 0.07, 0.2], quat=(0.9, 0.2, -0.3, 0.1), opacity=0.7,
                      dc=(0.4, -0.1, 0.25))
    rng = np.random.default_rng(5)
    cot = {"color": rng.normal(size=(3, 40, 48)), "depth": np.zeros((40, 48)), "normal": np.zeros((3, 40, 48)),
           "alpha": rng.normal(size=(40, 48))}
    pg = O.project(sc, cam, OPT)[0]
    conic = pg[O.PG["conic"]]
    C = np.array([[conic[0], conic[1]], [conic[1], conic[2]]])
    rgb = pg[O.PG["rgb"]]
    uu, vv = np.meshgrid(np.arange(48) + 0.5, np.arange(40) + 0.5)
    d = np.stack([pg[O.PG["u"]] - uu, pg[O.PG["v"]] - vv], -1)
    a = float(np.float32(0.7)) * np.exp(-0.5 * np.einsum("hwi,ij,hwj->hw", d, C, d))
    amin, amax = float(np.float32(1 / 255)), float(np.float32(0.99))
    ok = (a >= amin * (1 + 1e-4)) & (a < amax)
    assert (a >= amax).sum() == 0 and ok.sum() > 100
    g = cot["alpha"] + np.einsum("c,chw->hw", rgb, cot["color"])  # dL/dα per pixel (single splat)
    dadu = -a[..., None] * np.einsum("ij,hwj->hwi", C, d)
    exp = np.einsum("hw,hwi->i", np.where(ok, g, 0.0), dadu)
    cot_m = {k: (v * ok if v.ndim == 2 else v * ok[None]) for k, v in cot.items()}
    got = O.grad(sc, cam, OPT, cot_m, [0], means2d=True)[0, 59:61]
    np.testing.assert_allclose(got, exp, rtol=1e-10, atol=1e-12)
