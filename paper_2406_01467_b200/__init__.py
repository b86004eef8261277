"""B200-native RaDe-GS rasterizer hot path (arXiv 2406.01467).

The compute lives in librade.so (hand-written sm_100a CUDA behind the C ABI of
include/rade.h). This package is the thin Python binding (`rade`), the in-tree build
(`build`) and the view-parallel multi-GPU driver (`parallel`).
"""
from .rade import (Gaussians, RadeRasterize, TsdfVolume, View, camera_struct, default_options, options_struct, rasterize,
                   rd_bin, rd_blend_bwd, rd_blend_bwd_ex, rd_debug_binning, rd_debug_grads2d, rd_debug_pixel_state,
                   rd_debug_preprocess, rd_get_timings, rd_normal_consistency, rd_normal_consistency_bwd, rd_preprocess, rd_preprocess_views, rd_preprocess_bwd, rd_preprocess_bwd_geometry, rd_preprocess_bwd_views, rd_preprocess_bwd_views_ex, rd_preprocess_bwd_views_sh, rd_render_bwd,
                   rd_marching_cubes, rd_render_fwd, rd_render_fwd_ex, rd_set_profiling, rd_tsdf_integrate, rd_version, rd_view_create, rd_view_destroy, rd_view_stats,
                   render, render_backward)

__all__ = ["Gaussians", "RadeRasterize", "TsdfVolume", "View", "camera_struct", "default_options", "options_struct", "rasterize",
           "rd_bin", "rd_blend_bwd", "rd_blend_bwd_ex", "rd_debug_binning", "rd_debug_grads2d", "rd_debug_pixel_state",
           "rd_debug_preprocess", "rd_get_timings", "rd_normal_consistency", "rd_normal_consistency_bwd", "rd_preprocess", "rd_preprocess_views", "rd_preprocess_bwd", "rd_preprocess_bwd_geometry", "rd_preprocess_bwd_views", "rd_preprocess_bwd_views_ex", "rd_preprocess_bwd_views_sh", "rd_render_bwd",
           "rd_marching_cubes", "rd_render_fwd", "rd_render_fwd_ex", "rd_set_profiling", "rd_tsdf_integrate", "rd_version", "rd_view_create", "rd_view_destroy", "rd_view_stats",
           "render", "render_backward"]
