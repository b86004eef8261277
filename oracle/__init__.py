"""RaDe-GS CPU oracle (fp64) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package. The product path (paper_2406_01467_b200/) never imports
it and shares no code with it. See oracle/rade_oracle.cpp for what is computed and the
PAPER.md lines each step follows.

Parity status of each oracle function:
  project      pinned (tests/test_oracle_pins.py: Σ examples + scipy rotation, Jacobian vs
               finite differences, Σ′/t* vs brute-force 1D maximisation, isotropic and
               flattened closed forms, q̂·v′ = 1, centre identity, planarity)
  sh_basis     pinned (scipy real spherical harmonics with Condon-Shortley phase)
  splat_eval   pinned (brute-force 1D search; perspective Eq.7 vs isotropic closed form)
  render       pinned (two opaque layers, single splat, empty scene, Σω + T = 1, median
               property, tile-free brute force by construction)
  grad         pinned (central finite differences of render)
  distortion   pinned (two-layer closed form; detached-weight gradient closed form;
               one-pass identity on per-splat evaluations)
  depth_normal, normal_consistency (NEXT-2, image space, plain numpy fp64)
               pinned (fronto-parallel and tilted planes: analytic normals; holes;
               Σω(1 − n·ñ) = A − N·ñ on the oracle's own blend)
  Constants chosen by convention (readings S1, S5, S6, S8, S14) are parity unpinned
  against the paper: the paper fixes none of them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rade_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

PG_STRIDE = 96
PG = dict(valid=0, zkey=1, x=slice(2, 5), z=5, tc=6, u=7, v=8, Sigma=slice(9, 18), Sc=slice(18, 27),
          J=slice(27, 36), Sp=slice(36, 45), Spi=slice(45, 54), A2=slice(54, 57), conic=slice(57, 60),
          qhat=slice(60, 63), q=slice(63, 65), p=slice(65, 67), n=slice(67, 70), rgb=slice(70, 73),
          rgb_clamped=slice(73, 76), o=76, ndotx=77)
NPARAM = 59
NDUAL = 61  # + dL/d(u_c, v_c) (or_grad columns 59, 60)

# default ambiguity bands: F1 α-cutoff, F2 α-clamp (|Δ ln α|),
# F3 T-stop (relative), F4 median crossing (|T′ − median_T|), F5 grazing |n·x̂_c|
DEFAULT_EPS = (1e-5, 1e-5, 1e-4, 1e-5, 0.05)


def build(force=False):
    """Compile the oracle (g++ -O2 -fopenmp, no fast-math, no FP contraction)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", _SRC, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            common = [i64, dp, dp, dp, dp, dp, ctypes.c_int, dp, dp]
            L.or_project.argtypes = common + [dp]
            L.or_splat_eval.argtypes = common + [i64, i64, dp, dp]
            L.or_render.argtypes = common + [i64, ctypes.c_void_p, dp, dp, dp, dp, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, dp]
            L.or_grad.argtypes = common + [dp, i64, ctypes.c_void_p, dp, dp]
            L.or_order.argtypes = common + [ctypes.c_void_p, ctypes.c_void_p]
            L.or_sh_basis.argtypes = [dp, dp]
            L.or_sh_basis.restype = None
            L.or_num_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _scene_args(scene):
    means = np.ascontiguousarray(scene.means, np.float64)
    scales = np.ascontiguousarray(scene.scales, np.float64)
    rot = np.ascontiguousarray(scene.rotations, np.float64)
    opac = np.ascontiguousarray(scene.opacities, np.float64)
    sh = np.ascontiguousarray(scene.sh, np.float64).reshape(scene.sh.shape[0] * 3, scene.n)
    keep = (means, scales, rot, opac, sh)
    return keep, [ctypes.c_int64(scene.n), _dp(means), _dp(scales), _dp(rot), _dp(opac), _dp(sh),
                  ctypes.c_int(int(scene.sh.shape[0]))]


def _cam_vec(cam):
    v = np.zeros(19, np.float64)
    v[0:6] = [cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]
    v[6:15] = np.asarray(cam.R, np.float64).reshape(9)
    v[15:18] = np.asarray(cam.t, np.float64).reshape(3)
    v[18] = cam.znear
    return v


def _opt_vec(opt, eps=DEFAULT_EPS):
    """Options are taken at their fp32 values: both sides see the same float inputs."""
    f = lambda x: float(np.float32(x))
    v = np.zeros(15, np.float64)
    v[0:5] = [f(opt.alpha_min), f(opt.alpha_max), f(opt.T_min), f(opt.median_T), f(opt.dilation)]
    v[5:8] = [f(b) for b in opt.bg]
    v[8] = opt.sh_degree
    v[9:14] = eps
    v[14] = f(getattr(opt, "guard_band", 0.0))  # reading S6b: 0 = off
    return v


def _cam_f32(cam):
    """Camera values as the fp32 numbers the GPU receives."""
    import copy
    c = copy.copy(cam)
    c.fx, c.fy, c.cx, c.cy, c.znear = (float(np.float32(x)) for x in (cam.fx, cam.fy, cam.cx, cam.cy, cam.znear))
    c.R = np.asarray(cam.R, np.float32)
    c.t = np.asarray(cam.t, np.float32)
    return c


def project(scene, cam, opt):
    """Per-Gaussian projection, array [N, 96] indexed by oracle.PG."""
    keep, sargs = _scene_args(scene)
    cv, ov = _cam_vec(_cam_f32(cam)), _opt_vec(opt)
    out = np.zeros((scene.n, PG_STRIDE), np.float64)
    lib().or_project(*sargs, _dp(cv), _dp(ov), _dp(out))
    return out


def splat_eval(scene, cam, opt, gid, uv):
    """Per (Gaussian gid, point uv[k]) -> [k, 6]: α_raw, t*_ray, d, t*_persp, depth_persp, power."""
    keep, sargs = _scene_args(scene)
    cv, ov = _cam_vec(_cam_f32(cam)), _opt_vec(opt)
    uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
    out = np.zeros((uv.shape[0], 6), np.float64)
    rc = lib().or_splat_eval(*sargs, _dp(cv), _dp(ov), ctypes.c_int64(gid), ctypes.c_int64(uv.shape[0]),
                             _dp(uv), _dp(out))
    if rc != 0:
        raise ValueError(f"splat {gid} culled (rc={rc})")
    return out


def render(scene, cam, opt, pixels=None, eps=DEFAULT_EPS, timing=None):
    """Brute-force render. pixels=None: full frame, outputs shaped [C][H][W] / [H][W];
    else a 1-D array of linear pixel indices, outputs shaped [C][k] / [k].
    timing (optional float64[3]) receives: project+sort s, per-pixel loop s, survivors."""
    keep, sargs = _scene_args(scene)
    cv, ov = _cam_vec(_cam_f32(cam)), _opt_vec(opt, eps)
    W, H = cam.width, cam.height
    if pixels is None:
        npix, pix = W * H, None
    else:
        pix = np.ascontiguousarray(pixels, np.int64)
        npix = pix.shape[0]
    color = np.zeros(3 * npix)
    depth = np.zeros(npix)
    normal = np.zeros(3 * npix)
    alpha = np.zeros(npix)
    flags = np.zeros(npix, np.uint8)
    nblend = np.zeros(npix, np.int32)
    mid = np.zeros(npix, np.int64)
    dist = np.zeros(npix)
    lib().or_render(*sargs, _dp(cv), _dp(ov), ctypes.c_int64(npix),
                    None if pix is None else pix.ctypes.data, _dp(color), _dp(depth), _dp(normal),
                    _dp(alpha), flags.ctypes.data, nblend.ctypes.data, mid.ctypes.data, _dp(dist),
                    None if timing is None else _dp(timing))
    shape = (H, W) if pixels is None else (npix,)
    return dict(color=color.reshape((3,) + shape), depth=depth.reshape(shape), normal=normal.reshape((3,) + shape),
                alpha=alpha.reshape(shape), flags=flags.reshape(shape), nblend=nblend.reshape(shape),
                median_id=mid.reshape(shape), distortion=dist.reshape(shape))


def grad(scene, cam, opt, cot, gids, eps=DEFAULT_EPS, timing=None, means2d=False):
    """Exact dL/dθ for the listed Gaussians, L = Σ_px cot·(C, D, N, A[, L_d]) (cot["distortion"]
    optional; ω detached in L_d, S21). Returns [len(gids), 59] (μ 0..2, s 3..5, q 6..9, o 10,
    sh 11 + coeff*3 + ch); with means2d=True [len(gids), 61], columns 59..60 = dL/d(u_c, v_c)
    (the projected centre, every other per-splat quantity fixed)."""
    keep, sargs = _scene_args(scene)
    cv, ov = _cam_vec(_cam_f32(cam)), _opt_vec(opt, eps)
    W, H = cam.width, cam.height
    c = np.zeros((9, H, W), np.float64)
    c[0:3] = cot["color"]
    c[3] = cot["depth"]
    c[4:7] = cot["normal"]
    c[7] = cot["alpha"]
    if cot.get("distortion") is not None:
        c[8] = cot["distortion"]
    c = np.ascontiguousarray(c)
    gids = np.ascontiguousarray(gids, np.int64)
    out = np.zeros((gids.shape[0], NDUAL), np.float64)
    lib().or_grad(*sargs, _dp(cv), _dp(ov), _dp(c), ctypes.c_int64(gids.shape[0]), gids.ctypes.data, _dp(out),
                  None if timing is None else _dp(timing))
    return out if means2d else np.ascontiguousarray(out[:, :NPARAM])


def order(scene, cam, opt):
    """Ids of the surviving Gaussians in the oracle's global front-to-back order (
    reading S7: fp32 z_key ascending, ties by id)."""
    keep, sargs = _scene_args(scene)
    cv, ov = _cam_vec(_cam_f32(cam)), _opt_vec(opt)
    out = np.zeros(scene.n, np.int64)
    cnt = np.zeros(1, np.int64)
    lib().or_order(*sargs, _dp(cv), _dp(ov), out.ctypes.data, cnt.ctypes.data)
    return out[:int(cnt[0])]


def sh_basis(direction):
    d = np.ascontiguousarray(direction, np.float64)
    out = np.zeros(16)
    lib().or_sh_basis(_dp(d), _dp(out))
    return out


def loss(outputs, cot, bg=None):
    """L = Σ_px cot·(C, D, N, A) from a render() result (fp64)."""
    return float(np.sum(outputs["color"] * cot["color"]) + np.sum(outputs["depth"] * cot["depth"])
                 + np.sum(outputs["normal"] * cot["normal"]) + np.sum(outputs["alpha"] * cot["alpha"]))


def apply_filter3d(scene, filt):
    """The Mip-Splatting 3D filter ("incorporate the 3D filter proposed in
    Mip-Splatting"; reading S23): Σ ← Σ + f²I per Gaussian, which for Σ = R S²Rᵀ is the
    Gaussian with scales s' = √(s² + f²) and the same rotation, and o ← o·√(det Σ / det Σ')
    = o·Π_k s_k/s'_k. Returns (filtered scene, vjp) where vjp maps the gradient rows of the
    filtered scene ([n, 59]) to the raw scales and opacities (f is a constant)."""
    f = np.asarray(filt, np.float64)
    s = np.asarray(scene.scales, np.float64)
    sp = np.sqrt(s * s + f[None, :] ** 2)
    ratio = np.prod(s / sp, axis=0)
    out = scene.copy()
    out.scales = sp
    out.opacities = np.asarray(scene.opacities, np.float64) * ratio
    op = out.opacities

    def vjp(G, gids):
        G = np.array(G, np.float64, copy=True)
        gids = np.asarray(gids)
        d_op = G[:, 10].copy()
        for k in range(3):
            sk, spk = s[k, gids], sp[k, gids]
            G[:, 3 + k] = G[:, 3 + k] * sk / spk + d_op * op[gids] * (1.0 / sk - sk / spk ** 2)
        G[:, 10] = d_op * op[gids] / np.asarray(scene.opacities, np.float64)[gids]
        return G

    return out, vjp


def tsdf_integrate(tsdf, weight, origin, voxel, trunc, max_depth, depth, cam):
    """One view of TSDF fusion of the median depth map ("render depth maps for
    all training views and construct a TSDF"; reading S24 = SPEC:418-423): voxel (i, j, k)
    of the [Z][Y][X] grid has its centre at origin + (i+½, j+½, k+½)·voxel; in camera space
    X_c = R X + t; it is updated when z_c > znear, its projection (u, v) falls in the image
    (pixel ⌊u⌋, ⌊v⌋), the depth D there is a sample (0 < D ≤ max_depth) and
    sdf = D − z_c > −trunc: tsdf ← (w·tsdf + clamp(sdf/trunc, −1, 1))/(w + 1), w ← w + 1.
    The voxel centre, X_c and (u, v) are formed in fp32 in a fixed operation order (no fused
    multiply-add), so the pixel choice is the same decision on both sides; the update is
    fp64 (so is sdf = D − z_c and its truncation test, a decision). tsdf, weight: float64
    [Z, Y, X] updated in place."""
    f = np.float32
    Z, Y, X = tsdf.shape
    o = np.asarray(origin, f)
    vs = f(voxel)
    ix = (np.arange(X, dtype=f) + f(0.5)) * vs + o[0]
    iy = (np.arange(Y, dtype=f) + f(0.5)) * vs + o[1]
    iz = (np.arange(Z, dtype=f) + f(0.5)) * vs + o[2]
    Xw = np.broadcast_to(ix[None, None, :], (Z, Y, X))
    Yw = np.broadcast_to(iy[None, :, None], (Z, Y, X))
    Zw = np.broadcast_to(iz[:, None, None], (Z, Y, X))
    R = np.asarray(cam.R, f).reshape(3, 3)
    t = np.asarray(cam.t, f)
    xc = ((R[0, 0] * Xw + R[0, 1] * Yw) + R[0, 2] * Zw) + t[0]
    yc = ((R[1, 0] * Xw + R[1, 1] * Yw) + R[1, 2] * Zw) + t[1]
    zc = ((R[2, 0] * Xw + R[2, 1] * Yw) + R[2, 2] * Zw) + t[2]
    ok = zc > f(cam.znear)
    zs = np.where(ok, zc, f(1))
    u = (f(cam.fx) * xc) / zs + f(cam.cx)
    v = (f(cam.fy) * yc) / zs + f(cam.cy)
    ok &= (u >= 0) & (v >= 0) & (u < f(cam.width)) & (v < f(cam.height))
    px = np.where(ok, np.floor(u), 0).astype(np.int64)
    py = np.where(ok, np.floor(v), 0).astype(np.int64)
    D = np.asarray(depth, f)[py, px]
    ok &= (D > 0) & (D <= f(max_depth))
    sdf = D - zc  # fp32, the one decision both sides take in the same precision
    ok &= sdf > -f(trunc)
    new = np.clip(sdf.astype(np.float64) / trunc, -1.0, 1.0)
    tsdf[ok] = (weight[ok] * tsdf[ok] + new[ok]) / (weight[ok] + 1.0)
    weight[ok] += 1.0


# Marching cubes ("with the Marching Cube algorithm"; reading S25). The cube's corner
# c ∈ 0..7 sits at (c & 1, c >> 1 & 1, c >> 2 & 1); inside = value < iso.
_MC_EDGES = [(0, 1), (2, 3), (4, 5), (6, 7), (0, 2), (1, 3), (4, 6), (5, 7), (0, 4), (1, 5), (2, 6), (3, 7)]
# faces as corner cycles, counter-clockwise seen from outside the cube
_MC_FACES = [(0, 4, 6, 2), (1, 3, 7, 5), (0, 1, 5, 4), (2, 6, 7, 3), (0, 2, 3, 1), (4, 5, 7, 6)]
_mc_cache = None


def mc_table():
    """Triangles (as edge triples) of every corner configuration, built by walking the cube
    faces: on each face, every maximal run of inside corners is cut off by one segment from
    the crossing entering the run to the crossing leaving it (so diagonal inside corners are
    separated, a choice that depends on the face alone and so agrees between the two cubes
    sharing it — watertight); the segments chain into loops through the crossing edges;
    each loop is fanned into triangles, oriented so their normal points from the inside
    corners to the outside ones. Returns a list of 256 lists of (e0, e1, e2)."""
    global _mc_cache
    if _mc_cache is not None:
        return _mc_cache
    pos = np.array([[c & 1, (c >> 1) & 1, (c >> 2) & 1] for c in range(8)], np.float64)
    eid = {}
    for k, (a, b) in enumerate(_MC_EDGES):
        eid[(a, b)] = eid[(b, a)] = k
    mid = np.array([(pos[a] + pos[b]) / 2 for a, b in _MC_EDGES])
    table = []
    for cfg in range(256):
        ins = [(cfg >> c) & 1 == 1 for c in range(8)]
        nxt = {}
        for f in _MC_FACES:
            for i in range(4):
                if ins[f[i]] and not ins[f[i - 1]]:  # a run of inside corners starts at f[i]
                    enter = eid[(f[i - 1], f[i])]
                    j = i
                    while ins[f[(j + 1) % 4]]:
                        j += 1
                    leave = eid[(f[j % 4], f[(j + 1) % 4])]
                    nxt[enter] = leave
        tris = []
        seen = set()
        inside_c = pos[[c for c in range(8) if ins[c]]].mean(0) if any(ins) else None
        outside_c = pos[[c for c in range(8) if not ins[c]]].mean(0) if not all(ins) else None
        for start in sorted(nxt):
            if start in seen:
                continue
            loop = [start]
            seen.add(start)
            e = nxt[start]
            while e != start:
                loop.append(e)
                seen.add(e)
                e = nxt[e]
            pts = mid[loop]
            nrm = np.zeros(3)  # Newell normal of the loop
            for k in range(len(loop)):
                p, q = pts[k], pts[(k + 1) % len(loop)]
                nrm += np.array([(p[1] - q[1]) * (p[2] + q[2]), (p[2] - q[2]) * (p[0] + q[0]),
                                 (p[0] - q[0]) * (p[1] + q[1])])
            if nrm @ (outside_c - inside_c) < 0:
                loop = loop[::-1]
            for k in range(1, len(loop) - 1):
                tris.append((loop[0], loop[k], loop[k + 1]))
        table.append(tris)
    _mc_cache = table
    return table


def marching_cubes(tsdf, weight, origin, voxel, iso=0.0):
    """Triangle soup of the iso-surface of a [Z][Y][X] volume (reading S25): cells between
    voxel centres (origin + (i+½)·voxel), skipped when a corner has weight 0; per cell the
    table's triangles, each vertex linearly interpolated on its edge,
    p = p_a + (iso − v_a)/(v_b − v_a)·(p_b − p_a). Order: cells with x fastest, then y, z;
    triangles in table order; a triangle with two vertices on the same cube corner (a corner
    value equal to iso makes s exactly 0 or 1) has zero area and is dropped. Returns float64
    [T, 3, 3] (vertex positions)."""
    table = mc_table()
    t = np.asarray(tsdf, np.float32)
    w = np.asarray(weight)
    Z, Y, X = t.shape
    out = []
    cx = lambda i: origin[0] + (i + 0.5) * voxel
    cy = lambda j: origin[1] + (j + 0.5) * voxel
    cz = lambda k: origin[2] + (k + 0.5) * voxel
    corners = [(c & 1, (c >> 1) & 1, (c >> 2) & 1) for c in range(8)]
    for k in range(Z - 1):
        for j in range(Y - 1):
            for i in range(X - 1):
                vals, ok, cfg = [], True, 0
                for c, (dx, dy, dz) in enumerate(corners):
                    if w[k + dz, j + dy, i + dx] == 0:
                        ok = False
                        break
                    v = float(t[k + dz, j + dy, i + dx])
                    vals.append(v)
                    if v < iso:
                        cfg |= 1 << c
                if not ok or cfg == 0 or cfg == 255:
                    continue
                for tri in table[cfg]:
                    tv, at = [], []
                    for e in tri:
                        a, b = _MC_EDGES[e]
                        pa = np.array([cx(i + corners[a][0]), cy(j + corners[a][1]), cz(k + corners[a][2])])
                        pb = np.array([cx(i + corners[b][0]), cy(j + corners[b][1]), cz(k + corners[b][2])])
                        s = (iso - vals[a]) / (vals[b] - vals[a])
                        tv.append(pa + s * (pb - pa))
                        at.append(a if s == 0.0 else b if s == 1.0 else -1 - len(at))  # corner it sits on
                    if len(set(at)) < 3:  # two vertices on one corner: zero area, dropped (S25)
                        continue
                    out.append(tv)
    return np.array(out, np.float64).reshape(-1, 3, 3)


def depth_normal(depth, cam):
    """Normal from the depth map by finite differences ("applying finite
    difference on the depth map"; reading S22 = SPEC:309-316): back-project the pixel centre
    and its right and lower neighbours, P = D·((x+½−cx)/fx, (y+½−cy)/fy, 1);
    ñ = normalize((P_right − P) × (P_down − P)), flipped so that ñ·P < 0; 0 where the pixel
    or either neighbour is a hole (D = 0) or missing (last column / row).
    depth [H, W] → ñ [3, H, W] (fp64)."""
    D = np.asarray(depth, np.float64)
    H, W = D.shape
    fx, fy, cx, cy = (float(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    xs = (np.arange(W) + 0.5 - cx) / fx
    ys = (np.arange(H) + 0.5 - cy) / fy
    P = np.stack([D * xs[None, :], D * ys[:, None], D], 0)
    out = np.zeros((3, H, W))
    for y in range(H - 1):
        for x in range(W - 1):
            if D[y, x] == 0 or D[y, x + 1] == 0 or D[y + 1, x] == 0:
                continue
            a = P[:, y, x + 1] - P[:, y, x]
            b = P[:, y + 1, x] - P[:, y, x]
            m = np.cross(a, b)
            nm = np.linalg.norm(m)
            if nm == 0:
                continue
            n = m / nm
            if n @ P[:, y, x] > 0:
                n = -n
            out[:, y, x] = n
    return out


def normal_consistency(depth, alpha, normal, cam):
    """Per-pixel normal consistency (reading S22): L_n = Σ_i ω_i (1 − n_iᵀñ)
    = A − Nᵀñ with A = Σω (alpha) and N = Σωn (the normal map), ñ = depth_normal; 0 where
    ñ is undefined. Returns (L_n [H, W], ñ [3, H, W])."""
    nt = depth_normal(depth, cam)
    valid = np.any(nt != 0, axis=0)
    L = np.where(valid, np.asarray(alpha, np.float64) - np.sum(np.asarray(normal, np.float64) * nt, 0), 0.0)
    return L, nt


def num_threads():
    return int(lib().or_num_threads())
