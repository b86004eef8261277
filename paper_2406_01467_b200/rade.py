"""Thin Python binding of the C ABI (include/rade.h): same names, argument marshalling only.

Every step of the path runs in librade.so's CUDA kernels; this module only turns torch
tensors (device memory, owned by the caller) and the current CUDA stream into the ABI's
plain pointers, and supplies a torch-backed allocator callback for the view's scratch.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _native as N

_DEF = None


def default_options():
    """rd_options_default() as a dict."""
    lib = N.load()
    o = N.RdOptions()
    N.check(lib.rd_options_default(ctypes.byref(o)), "rd_options_default")
    return dict(tile=o.tile, alpha_min=o.alpha_min, alpha_max=o.alpha_max, T_min=o.T_min, median_T=o.median_T,
                dilation=o.dilation, bg=tuple(o.bg), sh_degree=o.sh_degree, guard_band=o.guard_band)


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_f32(name, t, shape=None):
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


@dataclass
class Gaussians:
    """Device parameters, one row per Gaussian (include/rade.h rd_gaussians): means [N,3],
    scales [N,3] (activated), rotations [N,4] (raw w,x,y,z), opacities [N] (activated),
    sh [N,K,3] — the tensor layout of a 3DGS trainer; optional filter3d [N] (the Mip-Splatting
    3D filter size, NEXT-3: a constant input, it has no gradient)."""
    means: torch.Tensor
    scales: torch.Tensor
    rotations: torch.Tensor
    opacities: torch.Tensor
    sh: torch.Tensor
    filter3d: Optional[torch.Tensor] = None
    means2d: Optional[torch.Tensor] = None  # as a gradient holder only: dL/d(u_c, v_c) [N, 2] (optional)

    @property
    def n(self):
        return int(self.opacities.shape[0])

    def validate(self):
        n = self.n
        _check_f32("means", self.means, (n, 3))
        _check_f32("scales", self.scales, (n, 3))
        _check_f32("rotations", self.rotations, (n, 4))
        _check_f32("opacities", self.opacities, (n,))
        _check_f32("sh", self.sh)
        if self.sh.dim() != 3 or self.sh.shape[0] != n or self.sh.shape[2] != 3:
            raise ValueError("sh must be [N, K, 3]")
        if self.filter3d is not None:
            _check_f32("filter3d", self.filter3d, (n,))

    def c_struct(self):
        self.validate()
        return N.RdGaussians(self.n, int(self.sh.shape[1]), self.means.data_ptr(), self.scales.data_ptr(),
                             self.rotations.data_ptr(), self.opacities.data_ptr(), self.sh.data_ptr(),
                             None if self.filter3d is None else self.filter3d.data_ptr())

    @staticmethod
    def from_numpy(scene, device="cuda"):
        """From a scenegen.Scene (whose arrays are [3][N], [4][N], [K][3][N])."""
        f = lambda a: torch.as_tensor(a, dtype=torch.float32).contiguous().to(device)
        return Gaussians(f(scene.means.T), f(scene.scales.T), f(scene.rotations.T), f(scene.opacities),
                         f(scene.sh.transpose(2, 0, 1)))

    def zeros_like(self, means2d: bool = False):
        """A zeroed gradient holder; means2d=True adds the [N, 2] screen-space gradient."""
        g = Gaussians(*(torch.zeros_like(t) for t in (self.means, self.scales, self.rotations, self.opacities,
                                                          self.sh)))
        if means2d:
            g.means2d = torch.zeros((self.n, 2), dtype=torch.float32, device=self.means.device)
        return g

    def tensors(self):
        return (self.means, self.scales, self.rotations, self.opacities, self.sh)


def camera_struct(cam):
    """Any object with fx, fy, cx, cy, width, height, R (3x3), t (3), znear."""
    c = N.RdCamera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    R = [float(x) for row in (cam.R.tolist() if hasattr(cam.R, "tolist") else cam.R) for x in row]
    t = [float(x) for x in (cam.t.tolist() if hasattr(cam.t, "tolist") else cam.t)]
    for k in range(9):
        c.R[k] = R[k]
    for k in range(3):
        c.t[k] = t[k]
    c.znear = float(getattr(cam, "znear", 0.2))
    return c


def options_struct(opt=None):
    o = N.RdOptions()
    N.check(N.load().rd_options_default(ctypes.byref(o)), "rd_options_default")
    if opt is None:
        return o
    get = (lambda k, d: opt.get(k, d)) if isinstance(opt, dict) else (lambda k, d: getattr(opt, k, d))
    o.tile = int(get("tile", o.tile))
    o.alpha_min = float(get("alpha_min", o.alpha_min))
    o.alpha_max = float(get("alpha_max", o.alpha_max))
    o.T_min = float(get("T_min", o.T_min))
    o.median_T = float(get("median_T", o.median_T))
    o.dilation = float(get("dilation", o.dilation))
    bg = get("bg", tuple(o.bg))
    for k in range(3):
        o.bg[k] = float(bg[k])
    o.sh_degree = int(get("sh_degree", o.sh_degree))
    o.guard_band = float(get("guard_band", o.guard_band))
    return o


class View:
    """Owns an rd_view* and the torch tensors backing its scratch buffers."""

    def __init__(self, device=None):
        self.lib = N.load()
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self._bufs = {}

        def _alloc(nbytes, ctx):
            try:
                t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            except Exception:  # noqa: BLE001 - reported to C as a NULL pointer -> RD_ERR_ALLOC
                return None
            self._bufs[t.data_ptr()] = t
            return t.data_ptr()

        def _free(ptr, ctx):
            self._bufs.pop(ptr, None)

        self._alloc_cb = N.ALLOC_FN(_alloc)
        self._free_cb = N.FREE_FN(_free)
        h = ctypes.c_void_p()
        N.check(self.lib.rd_view_create(ctypes.byref(h), self._alloc_cb, self._free_cb, None), "rd_view_create")
        self.handle = h
        self.camera = None
        self.options = None
        self.n = 0

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rd_view_destroy(self.handle)
            self.handle = None
            self._bufs.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def rd_view_create(device=None) -> View:
    return View(device)


def rd_view_destroy(view: View):
    view.close()


def rd_preprocess(view: View, gaussians: Gaussians, camera, options=None, stream=None):
    g = gaussians.c_struct()
    c = camera_struct(camera)
    o = options_struct(options)
    N.check(view.lib.rd_preprocess(view.handle, ctypes.byref(g), ctypes.byref(c), ctypes.byref(o),
                                   _stream_ptr(stream)), "rd_preprocess")
    view.camera, view.options, view.n = c, o, gaussians.n


def rd_preprocess_views(views, gaussians: Gaussians, cameras, options=None, stream=None):
    """K1 for a round of views (≤ 8) of the same Gaussians in one launch on `stream`
    (parameter and SH rows read once); = rd_preprocess on each view."""
    views = list(views)
    if len(cameras) != len(views):
        raise ValueError("one camera per view")
    arr = (ctypes.c_void_p * len(views))(*[v.handle for v in views])
    g = gaussians.c_struct()
    cs = [camera_struct(c) for c in cameras]
    carr = (N.RdCamera * len(cs))(*cs)
    o = options_struct(options)
    N.check(N.load().rd_preprocess_views(arr, len(views), ctypes.byref(g), carr, ctypes.byref(o),
                                         _stream_ptr(stream)), "rd_preprocess_views")
    for v, c in zip(views, cs):
        v.camera, v.options, v.n = c, o, gaussians.n


def rd_bin(view: View, stream=None) -> int:
    m = ctypes.c_int64(0)
    N.check(view.lib.rd_bin(view.handle, ctypes.byref(m), _stream_ptr(stream)), "rd_bin")
    return int(m.value)


def rd_render_fwd(view: View, color=None, depth=None, normal=None, alpha=None, stream=None, allocate=True):
    """Renders into the given tensors; missing ones are allocated if `allocate`."""
    H, W = view.camera.height, view.camera.width
    dev = view.device
    if allocate:
        color = torch.empty((3, H, W), dtype=torch.float32, device=dev) if color is None else color
        depth = torch.empty((H, W), dtype=torch.float32, device=dev) if depth is None else depth
        normal = torch.empty((3, H, W), dtype=torch.float32, device=dev) if normal is None else normal
        alpha = torch.empty((H, W), dtype=torch.float32, device=dev) if alpha is None else alpha
    for name, t, shp in (("color", color, (3, H, W)), ("depth", depth, (H, W)), ("normal", normal, (3, H, W)),
                         ("alpha", alpha, (H, W))):
        if t is not None:
            _check_f32(name, t, shp)
    N.check(view.lib.rd_render_fwd(view.handle, _ptr(color), _ptr(depth), _ptr(normal), _ptr(alpha),
                                   _stream_ptr(stream)), "rd_render_fwd")
    return dict(color=color, depth=depth, normal=normal, alpha=alpha)


def rd_render_fwd_ex(view: View, color=None, depth=None, normal=None, alpha=None, distortion=None, stream=None):
    """rd_render_fwd plus the depth-distortion map L_d (reading S21) when `distortion` is a
    [H, W] float32 tensor (or True: allocated). Returns the dict of the given maps."""
    H, W = view.camera.height, view.camera.width
    if distortion is True:
        distortion = torch.empty((H, W), dtype=torch.float32, device=view.device)
    for name, t, shp in (("color", color, (3, H, W)), ("depth", depth, (H, W)), ("normal", normal, (3, H, W)),
                         ("alpha", alpha, (H, W)), ("distortion", distortion, (H, W))):
        if t is not None:
            _check_f32(name, t, shp)
    m = N.RdFwdMaps(*(None if t is None else t.data_ptr() for t in (color, depth, normal, alpha, distortion)))
    N.check(view.lib.rd_render_fwd_ex(view.handle, ctypes.byref(m), _stream_ptr(stream)), "rd_render_fwd_ex")
    return dict(color=color, depth=depth, normal=normal, alpha=alpha, distortion=distortion)


def rd_blend_bwd_ex(view: View, dL_dcolor=None, dL_ddepth=None, dL_dnormal=None, dL_dalpha=None,
                    dL_ddistortion=None, stream=None):
    """rd_blend_bwd plus the cotangent of the distortion map (ω detached, S21)."""
    _check_cot(view, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha)
    if dL_ddistortion is not None:
        _check_f32("dL_ddistortion", dL_ddistortion, (view.camera.height, view.camera.width))
    c = N.RdBwdCotangents(*(None if t is None else t.data_ptr()
                            for t in (dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, dL_ddistortion)))
    N.check(view.lib.rd_blend_bwd_ex(view.handle, ctypes.byref(c), _stream_ptr(stream)), "rd_blend_bwd_ex")


def rd_normal_consistency(camera, depth, alpha=None, normal=None, consistency=True, depth_normal=False,
                          stream=None):
    """NEXT-2 (reading S22): the normal-consistency map A − N·ñ and/or the depth normals ñ
    from rendered maps. consistency / depth_normal: tensors, True (allocate) or None/False."""
    depth = depth.contiguous()
    H, W = depth.shape
    dev = depth.device
    if consistency is True:
        consistency = torch.empty((H, W), dtype=torch.float32, device=dev)
    if depth_normal is True:
        depth_normal = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    consistency = consistency if isinstance(consistency, torch.Tensor) else None
    depth_normal = depth_normal if isinstance(depth_normal, torch.Tensor) else None
    for name, t, shp in (("depth", depth, (H, W)), ("alpha", alpha, (H, W)), ("normal", normal, (3, H, W)),
                         ("consistency", consistency, (H, W)), ("depth_normal", depth_normal, (3, H, W))):
        if t is not None:
            _check_f32(name, t, shp)
    c = camera_struct(camera)
    N.check(N.load().rd_normal_consistency(ctypes.byref(c), _ptr(depth), _ptr(alpha), _ptr(normal), _ptr(consistency),
                                           _ptr(depth_normal), _stream_ptr(stream)), "rd_normal_consistency")
    return consistency, depth_normal


def rd_normal_consistency_bwd(camera, depth, normal, dL_dconsistency, dL_ddepth=None, dL_dalpha=None,
                              dL_dnormal=None, stream=None):
    """Adds the backward of Σ dL_dconsistency·consistency into the given map cotangents."""
    H, W = depth.shape
    for name, t, shp in (("depth", depth, (H, W)), ("normal", normal, (3, H, W)),
                         ("dL_dconsistency", dL_dconsistency, (H, W)), ("dL_ddepth", dL_ddepth, (H, W)),
                         ("dL_dalpha", dL_dalpha, (H, W)), ("dL_dnormal", dL_dnormal, (3, H, W))):
        if t is not None:
            _check_f32(name, t, shp)
    c = camera_struct(camera)
    N.check(N.load().rd_normal_consistency_bwd(ctypes.byref(c), _ptr(depth), _ptr(normal), _ptr(dL_dconsistency),
                                               _ptr(dL_ddepth), _ptr(dL_dalpha), _ptr(dL_dnormal),
                                               _stream_ptr(stream)), "rd_normal_consistency_bwd")


class TsdfVolume:
    """NEXT-4: a TSDF volume on the device ([Z][Y][X] fp32 tsdf and weight; reading S24)."""

    def __init__(self, origin, voxel_size, dims_xyz, truncation=None, max_depth=1e30, device="cuda"):
        self.origin = tuple(float(v) for v in origin)
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(v) for v in dims_xyz)
        self.truncation = float(truncation if truncation is not None else 4 * voxel_size)
        self.max_depth = float(max_depth)
        X, Y, Z = self.dims
        self.tsdf = torch.ones((Z, Y, X), dtype=torch.float32, device=device)
        self.weight = torch.zeros((Z, Y, X), dtype=torch.float32, device=device)
        self._mc_capacity = 0  # triangle buffer size guess for rd_marching_cubes (last count + 25%)

    def c_struct(self):
        s = N.RdTsdf()
        for k in range(3):
            s.origin[k] = self.origin[k]
            s.dims[k] = self.dims[k]
        s.voxel_size, s.truncation, s.max_depth = self.voxel_size, self.truncation, self.max_depth
        s.tsdf, s.weight = self.tsdf.data_ptr(), self.weight.data_ptr()
        return s


def rd_tsdf_integrate(volume: TsdfVolume, depths, cameras, stream=None):
    """Fuses depth maps [V, H, W] (device fp32, 0 = hole) rendered from `cameras` (V)."""
    depths = depths.contiguous()
    if depths.dim() == 2:
        depths = depths[None]
    _check_f32("depths", depths)
    V = depths.shape[0]
    if len(cameras) != V:
        raise ValueError("one camera per depth map")
    cams = (N.RdCamera * max(V, 1))(*[camera_struct(c) for c in cameras])
    s = volume.c_struct()
    N.check(N.load().rd_tsdf_integrate(ctypes.byref(s), _ptr(depths), cams, V, _stream_ptr(stream)),
            "rd_tsdf_integrate")
    return volume


def rd_marching_cubes(volume: TsdfVolume, iso=0.0, stream=None):
    """NEXT-4: the iso-surface of the fused volume as a triangle soup [T, 3, 3] (device fp32),
    cells in x-fastest order (reading S25). Two calls through the C-ABI: count, then emit."""
    s = volume.c_struct()
    n = ctypes.c_int64(0)
    lib = N.load()
    # one call when the buffer of the volume's previous extraction (+25%) is large enough
    cap = getattr(volume, "_mc_capacity", 0)
    buf = torch.empty((cap, 3, 3), dtype=torch.float32, device=volume.tsdf.device) if cap else None
    N.check(lib.rd_marching_cubes(ctypes.byref(s), float(iso), _ptr(buf) if cap else None, cap, ctypes.byref(n),
                                  _stream_ptr(stream)), "rd_marching_cubes")
    if cap and n.value <= cap:
        return buf[:n.value]
    volume._mc_capacity = int(n.value * 1.25) + 1024
    tris = torch.empty((n.value, 3, 3), dtype=torch.float32, device=volume.tsdf.device)
    if n.value:
        N.check(lib.rd_marching_cubes(ctypes.byref(s), float(iso), _ptr(tris), n.value, ctypes.byref(n),
                                      _stream_ptr(stream)), "rd_marching_cubes")
    return tris


def _check_cot(view, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha):
    H, W = view.camera.height, view.camera.width
    for name, t, shp in (("dL_dcolor", dL_dcolor, (3, H, W)), ("dL_ddepth", dL_ddepth, (H, W)),
                         ("dL_dnormal", dL_dnormal, (3, H, W)), ("dL_dalpha", dL_dalpha, (H, W))):
        if t is not None:
            _check_f32(name, t, shp)


def _grads_struct(grads):
    if grads is None:
        raise ValueError("grads is required")
    grads.validate()
    if grads.means2d is not None:
        _check_f32("means2d", grads.means2d, (grads.n, 2))
    return N.RdGrads(grads.means.data_ptr(), grads.scales.data_ptr(), grads.rotations.data_ptr(),
                     grads.opacities.data_ptr(), grads.sh.data_ptr(),
                     None if grads.means2d is None else grads.means2d.data_ptr())


def rd_render_bwd(view: View, gaussians: Gaussians, dL_dcolor=None, dL_ddepth=None, dL_dnormal=None,
                  dL_dalpha=None, grads: Gaussians = None, stream=None):
    """Accumulates (+=) parameter gradients into `grads` (same layout as `gaussians`)."""
    _check_cot(view, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha)
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(view.lib.rd_render_bwd(view.handle, ctypes.byref(g), _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(dL_dnormal),
                                   _ptr(dL_dalpha), ctypes.byref(gr), _stream_ptr(stream)), "rd_render_bwd")
    return grads


def rd_blend_bwd(view: View, dL_dcolor=None, dL_ddepth=None, dL_dnormal=None, dL_dalpha=None, stream=None):
    """K4 only: the per-Gaussian 2-D gradients of the view (first half of rd_render_bwd)."""
    _check_cot(view, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha)
    N.check(view.lib.rd_blend_bwd(view.handle, _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(dL_dnormal), _ptr(dL_dalpha),
                                  _stream_ptr(stream)), "rd_blend_bwd")


def rd_preprocess_bwd_views(views, gaussians: Gaussians, grads: Gaussians, stream=None):
    """K5 of up to 8 views of the same Gaussians in one pass (rows read and reduced once).
    The caller orders `stream` after every view's rd_blend_bwd."""
    views = list(views)
    arr = (_VP_T * len(views))(*[v.handle for v in views])
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(N.load().rd_preprocess_bwd_views(arr, len(views), ctypes.byref(g), ctypes.byref(gr), _stream_ptr(stream)),
            "rd_preprocess_bwd_views")
    return grads


_VP_T = ctypes.c_void_p


def rd_preprocess_bwd_geometry(view: View, gaussians: Gaussians, grads: Gaussians, stream=None):
    """K5 geometry part of one view (K5b64 + K5b), right after its rd_blend_bwd; the SH part of
    the round follows with rd_preprocess_bwd_views_sh."""
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(view.lib.rd_preprocess_bwd_geometry(view.handle, ctypes.byref(g), ctypes.byref(gr), _stream_ptr(stream)),
            "rd_preprocess_bwd_geometry")
    return grads


RD_K5_SH_ONLY, RD_K5_GEOMETRY_ONLY, RD_K5_SET_SH = 1, 2, 4


def rd_preprocess_bwd_views_ex(views, gaussians: Gaussians, grads: Gaussians, flags: int = 0, stream=None):
    """rd_preprocess_bwd_views with flags (RD_K5_SH_ONLY, RD_K5_GEOMETRY_ONLY, RD_K5_SET_SH: the SH
    gradient rows are set, 0 where visible in none of the views, instead of accumulated)."""
    views = list(views)
    arr = (_VP_T * len(views))(*[v.handle for v in views])
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(N.load().rd_preprocess_bwd_views_ex(arr, len(views), ctypes.byref(g), ctypes.byref(gr), int(flags),
                                                _stream_ptr(stream)), "rd_preprocess_bwd_views_ex")
    return grads


def rd_preprocess_bwd_views_sh(views, gaussians: Gaussians, grads: Gaussians, stream=None):
    """K5 SH part of a round of views (rows read and reduced once), after their geometry parts
    may already have run."""
    views = list(views)
    arr = (_VP_T * len(views))(*[v.handle for v in views])
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(N.load().rd_preprocess_bwd_views_sh(arr, len(views), ctypes.byref(g), ctypes.byref(gr),
                                                _stream_ptr(stream)), "rd_preprocess_bwd_views_sh")
    return grads


def rd_preprocess_bwd(view: View, gaussians: Gaussians, grads: Gaussians, stream=None):
    """K5 only: accumulates (+=) parameter gradients from the last rd_blend_bwd of the view."""
    g = gaussians.c_struct()
    gr = _grads_struct(grads)
    N.check(view.lib.rd_preprocess_bwd(view.handle, ctypes.byref(g), ctypes.byref(gr), _stream_ptr(stream)),
            "rd_preprocess_bwd")
    return grads


def rd_view_stats(view: View) -> dict:
    s = N.RdStats()
    N.check(view.lib.rd_view_stats(view.handle, ctypes.byref(s)), "rd_view_stats")
    return {k: getattr(s, k) for k, _ in N.RdStats._fields_}


def rd_set_profiling(view: View, enabled: bool = True):
    N.check(view.lib.rd_set_profiling(view.handle, 1 if enabled else 0), "rd_set_profiling")


def rd_get_timings(view: View, reset: bool = False) -> dict:
    t = N.RdTimings()
    N.check(view.lib.rd_get_timings(view.handle, ctypes.byref(t), 1 if reset else 0), "rd_get_timings")
    d = {k: getattr(t, k) for k, _ in N.RdTimings._fields_ if k not in ("ms", "launches", "n_culled")}
    d["n_culled"] = dict(zip(("invalid", "near", "guard_band", "opacity", "degenerate", "off_screen"), t.n_culled))
    d["ms"] = {name: t.ms[i] for i, name in enumerate(N.KERNEL_NAMES)}
    d["launches"] = {name: t.launches[i] for i, name in enumerate(N.KERNEL_NAMES)}
    return d


def rd_debug_binning(view: View, stream=None):
    st = rd_view_stats(view)
    M, T = st["n_duplicates"], st["tiles_x"] * st["tiles_y"]
    keys = torch.empty(max(M, 1), dtype=torch.int64, device=view.device)
    ids = torch.empty(max(M, 1), dtype=torch.int32, device=view.device)
    ranges = torch.empty(2 * T, dtype=torch.int32, device=view.device)
    N.check(view.lib.rd_debug_binning(view.handle, _ptr(keys), _ptr(ids), _ptr(ranges), _stream_ptr(stream)),
            "rd_debug_binning")
    return keys[:M], ids[:M], ranges.view(T, 2)


def rd_debug_preprocess(view: View, stream=None):
    n = view.n
    rec = torch.empty((max(n, 1), 16), dtype=torch.float32, device=view.device)
    rect = torch.empty((max(n, 1), 2), dtype=torch.int32, device=view.device)
    touched = torch.empty(max(n, 1), dtype=torch.int32, device=view.device)
    N.check(view.lib.rd_debug_preprocess(view.handle, _ptr(rec), _ptr(rect), _ptr(touched), _stream_ptr(stream)),
            "rd_debug_preprocess")
    return rec[:n], rect[:n], touched[:n]


def rd_debug_pixel_state(view: View, stream=None):
    H, W = view.camera.height, view.camera.width
    T = torch.empty((H, W), dtype=torch.float32, device=view.device)
    nc = torch.empty((H, W), dtype=torch.int32, device=view.device)
    mp = torch.empty((H, W), dtype=torch.int32, device=view.device)
    N.check(view.lib.rd_debug_pixel_state(view.handle, _ptr(T), _ptr(nc), _ptr(mp), _stream_ptr(stream)),
            "rd_debug_pixel_state")
    return T, nc, mp


def rd_debug_grads2d(view: View, stream=None):
    g = torch.empty((max(view.n, 1), 16), dtype=torch.float32, device=view.device)
    N.check(view.lib.rd_debug_grads2d(view.handle, _ptr(g), _stream_ptr(stream)), "rd_debug_grads2d")
    return g[:view.n]


def rd_version() -> str:
    return N.load().rd_version().decode()


# ----------------------------------------------------------------------------- convenience

def render(gaussians: Gaussians, camera, options=None, view: View = None, stream=None):
    """One forward pass through all three forward stages. Returns (outputs, view)."""
    view = View() if view is None else view
    rd_preprocess(view, gaussians, camera, options, stream)
    rd_bin(view, stream)
    out = rd_render_fwd(view, stream=stream)
    return out, view


def render_backward(view: View, gaussians: Gaussians, cot: dict, grads: Gaussians, stream=None):
    return rd_render_bwd(view, gaussians, cot.get("color"), cot.get("depth"), cot.get("normal"), cot.get("alpha"),
                         grads, stream)


class RadeRasterize(torch.autograd.Function):
    """torch.autograd wrapper: (means, scales, rotations, opacities, sh) -> (color, depth,
    normal, alpha). Marshalling only; forward and backward are the C-ABI calls."""

    @staticmethod
    def forward(ctx, means, scales, rotations, opacities, sh, camera, options=None):
        g = Gaussians(means.contiguous(), scales.contiguous(), rotations.contiguous(), opacities.contiguous(),
                      sh.contiguous())
        out, view = render(g, camera, options)
        ctx.view, ctx.g = view, g
        return out["color"], out["depth"], out["normal"], out["alpha"]

    @staticmethod
    def backward(ctx, gc, gd, gn, ga):
        g = ctx.g
        grads = g.zeros_like()
        f = lambda t: None if t is None else t.contiguous()
        rd_render_bwd(ctx.view, g, f(gc), f(gd), f(gn), f(ga), grads)
        return grads.means, grads.scales, grads.rotations, grads.opacities, grads.sh, None, None


def rasterize(means, scales, rotations, opacities, sh, camera, options=None):
    return RadeRasterize.apply(means, scales, rotations, opacities, sh, camera, options)
