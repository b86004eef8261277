/*
 * rade.h — C ABI of the B200-native RaDe-GS rasterizer (arXiv 2406.01467).
 *
 * The library renders, for one camera view and a set of general 3D Gaussians, in ONE
 * pass: colour (Eq.3), alpha, the normal map (Eq.21-22, PAPER:617-627;
 * aggregated as Σ ω_i n_i, reading S10) and the median-depth map (the depth of
 * each splat at a pixel is the rasterized plane d = z_c + p·Δ of Eq.4),
 * and the matching backward pass (gradients for means, scales, rotations, opacities and
 * SH colours — the training use of PAPER:43-46). The problem statement it follows is
 * "given Gaussians (x_c, Σ = R S Sᵀ Rᵀ, opacity, SH) and a camera (W, intrinsics),
 * render colour, median depth and normal".
 *
 * Calls, in order, per view:
 *   rd_preprocess  stage 1 (K1): per-Gaussian EWA projection, conic, α-bounded tile rect,
 *                  SH colour, depth-plane coefficients p and normal n
 *   rd_bin         stage 2 (K2): depth radix sort, tile-count scan, duplicate (tile | depth)
 *                  keys, tile radix sort (hand-written onesweep passes), per-tile ranges
 *   rd_render_fwd  stage 3 (K3): per-tile front-to-back blend of C, A, N, median D
 *   rd_render_bwd  stage 4 (K4, K5): reverse replay per pixel, per-Gaussian chain rule
 *                  (also as its two halves rd_blend_bwd (K4) and rd_preprocess_bwd (K5))
 *
 * Conventions:
 *   - Camera: world->camera rotation R (row-major) and translation t; +z forward, +y down;
 *     pixel (i, j) is sampled at (i + 0.5, j + 0.5); u = fx·x/z + cx, v = fy·y/z + cy.
 *   - Gaussian arrays are row-major fp32 DEVICE arrays, one row per Gaussian (the layout of
 *     the (N,3)/(N,4)/(N,16,3) tensors of a 3DGS trainer; a view touches ~half of the
 *     Gaussians, and per-Gaussian rows keep the untouched half out of the traffic):
 *       means[n][3], scales[n][3] (activated, > 0), rotations[n][4] (raw quaternion w,x,y,z,
 *       normalised internally; the base pointer must be 16-byte aligned),
 *       opacities[n] (activated, in (0,1)), sh[n][sh_coeffs][3] (sh_coeffs = (deg+1)^2 ≤ 16).
 *   - Image outputs are planar fp32 DEVICE arrays: color[3][H][W], depth[H][W] (0 where the
 *     transmittance never crosses median_T), normal[3][H][W] (camera space, unnormalised
 *     Σ ω n), alpha[H][W] = 1 − T_final.
 *   - Gradients are ACCUMULATED (+=) into rd_grads arrays laid out like rd_gaussians, so
 *     several views can be summed before an all-reduce; the caller zeroes them.
 *
 * Ownership: every array passed in is owned by the caller. Internal scratch (per-Gaussian
 * records, keys/values, sort temp, per-pixel forward state, 2-D gradient accumulators) is
 * owned by the rd_view and obtained from the caller's rd_alloc_fn (e.g. PyTorch's caching
 * allocator) or, when alloc is NULL, from cudaMallocAsync on the call's stream. Buffers are
 * cached by capacity and reused across views. All calls on one view must use one stream.
 *
 * Errors: functions never throw; they return an rd_status and set a thread-local message
 * readable with rd_last_error(). Invalid arguments (null pointers, n < 0, width/height ≤ 0,
 * rotations not 16-byte aligned, tile ∉ {8, 16, 32}, thresholds outside (0, 1),
 * alpha_min ≥ alpha_max, sh_degree > 3 or
 * (sh_degree+1)^2 > sh_coeffs) return RD_ERR_INVALID_ARGUMENT; out-of-order calls return
 * RD_ERR_STATE; allocation failure RD_ERR_ALLOC; CUDA launch/runtime errors RD_ERR_CUDA.
 * A degenerate primitive (non-finite input, scale ≤ 0, zero quaternion, centre depth ≤
 * znear, opacity < alpha_min, singular 2-D covariance) is CULLED, not an error: it
 * contributes nothing and receives zero gradient.
 *
 * Synchronisation: every call is asynchronous on the given stream except rd_bin, which
 * reads the duplicate count M back to the host once: its histogram kernel writes the counts
 * to mapped pinned memory and rd_bin waits for that kernel's completion event (not for the
 * stream), with the depth sort already queued behind it.
 *
 * Threads: the library keeps no shared mutable state (the error message is thread-local);
 * calls on DISTINCT rd_view handles may run concurrently from different host threads, which
 * is how a multi-view caller keeps one view's rd_bin wait from holding back the issue of the
 * others (bench.py: one stream and one host thread per view of a step). One rd_view must not
 * be used by two threads at once.
 */
#ifndef RADE_H_
#define RADE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RD_OK = 0,
  RD_ERR_INVALID_ARGUMENT = 1,
  RD_ERR_STATE = 2,
  RD_ERR_ALLOC = 3,
  RD_ERR_CUDA = 4
} rd_status;

/* Host struct. R is world->camera, row-major; znear culls centres with z ≤ znear. */
typedef struct rd_camera {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];
  float t[3];
  float znear;
} rd_camera;

/* Host struct. Defaults (rd_options_default): tile 16, alpha_min 1/255, alpha_max 0.99,
 * T_min 1e-4, median_T 0.5, dilation 0.3 px², bg (0,0,0), sh_degree 3, guard_band 0 (off). */
typedef struct rd_options {
  int32_t tile;      /* 8, 16 or 32 pixels (outputs do not depend on it, reading S8) */
  float alpha_min;   /* splats with α < alpha_min are skipped (S8) */
  float alpha_max;   /* α = min(alpha_max, o·G) (S8) */
  float T_min;       /* stop before blending a splat that would make T < T_min (S8) */
  float median_T;    /* median depth: first blended splat with T_after ≤ median_T (S9) */
  float dilation;    /* h added to the 2-D covariance diagonal for α only (S5) */
  float bg[3];       /* C += T_final · bg (S17) */
  int32_t sh_degree; /* active SH degree 0..3 */
  float guard_band;  /* reading S6b, off when 0 (the default: SURVEY S6 culls on
                        z ≤ znear only). When g > 0, a Gaussian whose centre projects outside
                        [−g·W, (1+g)·W] × [−g·H, (1+g)·H] is culled, decided in fp32 as
                        fx·x_k ∈ [float(−gW − cx)·z_k, float((1+g)W − cx)·z_k] (same for y);
                        bench.py's C3 workload uses g = 0.15. Must be finite and ≥ 0. */
} rd_options;

/* Device Gaussian parameters, one row per Gaussian (see layout above). */
typedef struct rd_gaussians {
  int64_t n;
  int32_t sh_coeffs; /* coefficients stored per channel: 1, 4, 9 or 16 */
  const float* means;
  const float* scales;
  const float* rotations;
  const float* opacities;
  const float* sh;
  const float* filter3d; /* NULL, or [n]: the Mip-Splatting 3D filter size f per Gaussian (NEXT-3,
                            reading S23): rendered as Σ + f²I (scales √(s² + f²)) with opacity
                            o·Π s/√(s² + f²); gradients are w.r.t. the raw scales/opacities */
} rd_gaussians;

/* Device gradient arrays, same layouts as rd_gaussians; accumulated (+=). */
typedef struct rd_grads {
  float* means;
  float* scales;
  float* rotations;
  float* opacities;
  float* sh;
  float* means2d; /* optional (NULL: not produced), [n][2]: dL/d(u_c, v_c), the gradient w.r.t. the
                     projected centre in pixels with every other per-splat quantity held fixed
                     (the screen-space gradient 3DGS densification accumulates; PAPER:44 trains
                     with the 3DGS schedule); += per view, 0 for Gaussians culled in a view */
} rd_grads;

/* Per-view statistics (host struct filled by rd_view_stats). */
typedef struct rd_stats {
  int64_t n;            /* Gaussians in the last rd_preprocess */
  int64_t n_duplicates; /* M: (Gaussian, tile) pairs after rd_bin */
  int32_t tiles_x, tiles_y;
  int32_t width, height;
  int32_t stage;        /* 0 created, 1 preprocessed, 2 binned, 3 rendered, 4 blend-backward done */
  int32_t key_bits;     /* width of the equivalent one-pass sort key: 32 + ceil(log2(tiles)) */
  int64_t n_visible;    /* Gaussians that touch ≥ 1 tile (after rd_bin) */
  int64_t n_big;        /* of those, the ones whose backward chain rule runs in fp64 (K5b64:
                           tile rect > 16384 px), after rd_bin */
} rd_stats;

/* Per-kernel device timings and work counters (host struct filled by rd_get_timings).
 * Kernel index: 0 K1 preprocess_fwd, 1 K2a depth_sort (incl. the K2h histogram kernel), 2 K2b
 * scan, 3 K2c duplicate (fused with the first tile pass), 4 K2d tile_sort (remaining tile
 * passes), 5 K2e ranges, 6 K3 render_fwd, 7 K4 render_bwd (including the zeroing of
 * the 2-D gradient scratch), 8 K5 preprocess_bwd. */
#define RD_NUM_KERNELS 9
typedef struct rd_timings {
  double ms[RD_NUM_KERNELS];       /* summed CUDA-event durations since the last reset */
  int64_t launches[RD_NUM_KERNELS];
  int64_t pairs_evaluated_fwd;     /* (pixel, splat) pairs K3 evaluated (α computed)   */
  int64_t pairs_blended_fwd;       /* pairs K3 blended (α ≥ alpha_min, not stopped)   */
  int64_t pairs_evaluated_bwd;     /* pairs K4 evaluated (list positions < n_contrib) */
  int64_t n_visible;               /* Σ over views of Gaussians with tiles_touched > 0 */
  int64_t n_duplicates;            /* Σ over views of M */
  int64_t views;                   /* rd_render_fwd calls since the last reset */
  int64_t n_visible_union;         /* Σ over rd_preprocess_bwd_views calls timed on this view of the
                                      Gaussians visible in at least one of their views */
  int64_t n_culled[6];             /* Σ over rd_preprocess calls of the Gaussians culled (not an error,
                                      SPEC:49, 58, 76, 85), by the first reason that applies:
                                      [0] invalid input (non-finite, scale ≤ 0, zero quaternion),
                                      [1] centre depth ≤ znear, [2] outside the guard band (S6b),
                                      [3] opacity < alpha_min, [4] degenerate 2-D covariance or plane,
                                      [5] footprint entirely off screen */
  int64_t pairs_issued_fwd;        /* (pixel, splat) slots K3's warps stepped through: steps × the 64
                                      pixels of a warp (E_issued); pairs_evaluated_fwd /
                                      this = the SIMT efficiency of the walk */
} rd_timings;

typedef void* (*rd_alloc_fn)(size_t bytes, void* ctx);
typedef void (*rd_free_fn)(void* ptr, void* ctx);
typedef struct rd_view rd_view;
typedef void* rd_stream; /* a cudaStream_t */

/* Fills *opt with the defaults listed above. */
rd_status rd_options_default(rd_options* opt);

/* Creates a view handle. alloc/free may both be NULL (then cudaMallocAsync/cudaFreeAsync
 * on the call stream are used); otherwise both must be given. */
rd_status rd_view_create(rd_view** view, rd_alloc_fn alloc, rd_free_fn free_fn, void* ctx);

/* Releases the handle and every internal buffer (through free_fn / cudaFree). */
rd_status rd_view_destroy(rd_view* view);

/* Stage 1 (K1). Validates arguments, then launches one thread per Gaussian: cull,
 * x_c = W μ + t, (u_c, v_c), J, Σ′ top-left 2x2, conic of the dilated 2-D
 * covariance, α-bounded tile rect, SH → RGB, p (Eq.12-15) and n
 * (Eq.21-22). The camera and options are captured by value. */
rd_status rd_preprocess(rd_view* view, const rd_gaussians* g, const rd_camera* cam, const rd_options* opt,
                        rd_stream stream);

/* Stage 1 for n_views ≤ 8 views of the SAME Gaussians at once (a training step's round of
 * views): equivalent to rd_preprocess on each (views[k], cams[k]) — bit for bit — but one K1
 * launch on `stream` runs every Gaussian through all the views in turn, so its parameter and
 * SH rows are read from DRAM once. cams: HOST array of n_views cameras; opt shared. The caller
 * orders each view's later calls (on its own stream) after `stream`. Errors: n_views ∉ [1, 8],
 * NULL / repeated views → RD_ERR_INVALID_ARGUMENT; otherwise as rd_preprocess. */
rd_status rd_preprocess_views(rd_view* const* views, int32_t n_views, const rd_gaussians* g, const rd_camera* cams,
                              const rd_options* opt, rd_stream stream);

/* Stage 2 (K2). Result: the M (tile, Gaussian id) pairs in the order of ONE stable sort of
 * the 64-bit keys (tile << 32 | float_bits(z_c)) emitted in id order — per tile the
 * Gaussians front to back by z_c, ties by id (the depth sort of PAPER:422, reading S7) — and
 * per-tile [first, last) ranges; M is read to the host (written to *n_duplicates_out if
 * non-NULL). Computed as a stable depth sort of the visible Gaussians (4 radix passes), the
 * scan of their tile counts, and a stable sort of the duplicates by tile (tx, then ty digits;
 * the first pass fused with the duplicate generation), all single-pass radix passes with
 * decoupled look-back (binning.cu). Images of more than 2047 tiles per axis are rejected by
 * rd_preprocess (RD_ERR_INVALID_ARGUMENT). A second rd_bin before the next rd_preprocess
 * returns the same M and leaves the lists as they are. */
rd_status rd_bin(rd_view* view, int64_t* n_duplicates_out, rd_stream stream);

/* Stage 3 (K3). One CTA per tile. Any output pointer may be NULL to skip that map.
 * color[3][H][W], depth[H][W], normal[3][H][W], alpha[H][W] (device, fp32). */
rd_status rd_render_fwd(rd_view* view, float* color, float* depth, float* normal, float* alpha, rd_stream stream);

/* Stage 3 with the optional depth-distortion map (NEXT-1, reading S21):
 * distortion[H][W] = L_d = Σ_i Σ_j ω_i ω_j (d_i − d_j)² over the pixel's blended splats
 * (ω = blend weights, d = the per-pixel depth of Eq.15). Any pointer may be NULL; when
 * `distortion` is non-NULL the view also keeps the per-pixel state its backward needs. */
typedef struct rd_fwd_maps {
  float* color;       /* [3][H][W] */
  float* depth;       /* [H][W] median depth */
  float* normal;      /* [3][H][W] */
  float* alpha;       /* [H][W] */
  float* distortion;  /* [H][W] L_d, or NULL (then no distortion state is kept) */
} rd_fwd_maps;
rd_status rd_render_fwd_ex(rd_view* view, const rd_fwd_maps* maps, rd_stream stream);

/* Cotangents of rd_fwd_maps (any may be NULL = zero). dL_ddistortion needs a forward that
 * produced the distortion map (else RD_ERR_STATE); its gradient flows through d only — the
 * weights ω are detached (S21): ∂L_d/∂d_k = 4 ω_k (A d_k − D₁), A = Σω, D₁ = Σωd. */
typedef struct rd_bwd_cotangents {
  const float* dL_dcolor;
  const float* dL_ddepth;
  const float* dL_dnormal;
  const float* dL_dalpha;
  const float* dL_ddistortion;
} rd_bwd_cotangents;
rd_status rd_blend_bwd_ex(rd_view* view, const rd_bwd_cotangents* cot, rd_stream stream);

/* Stage 4 (K4 + K5). Cotangents dL/d(color, depth, normal, alpha) in the output layouts
 * (any may be NULL = zero). `g` must be the same Gaussians given to rd_preprocess.
 * Gradients are accumulated into `grads` (all five pointers required).
 * = rd_blend_bwd followed by rd_preprocess_bwd on the same stream. */
rd_status rd_render_bwd(rd_view* view, const rd_gaussians* g, const float* dL_dcolor, const float* dL_ddepth,
                        const float* dL_dnormal, const float* dL_dalpha, const rd_grads* grads, rd_stream stream);

/* Stage 4, first half (K4): the reverse per-pixel replay of Eq.3/Eq.4 into
 * the view's per-Gaussian 2-D gradients (see rd_debug_grads2d); touches no user gradient.
 * Cotangents as in rd_render_bwd. Requires rd_render_fwd on this view. */
rd_status rd_blend_bwd(rd_view* view, const float* dL_dcolor, const float* dL_ddepth, const float* dL_dnormal,
                       const float* dL_dalpha, rd_stream stream);

/* Stage 4, second half (K5): the per-Gaussian chain rule from the 2-D gradients of the last
 * rd_blend_bwd to means, scales, rotations, opacities and SH, ACCUMULATED (+=) into `grads`
 * with L2 reductions (red.global.add): calls of different views into the same `grads` may
 * run concurrently on different streams (the floating-point summation order, hence the
 * rounding of the sum, then depends on timing). `grads` must be 16-byte aligned where
 * rotations are. */
rd_status rd_preprocess_bwd(rd_view* view, const rd_gaussians* g, const rd_grads* grads, rd_stream stream);

/* Stage 4 second half (K5) for n_views ≤ 8 views of the SAME Gaussians at once (the views of
 * a training step): equivalent to rd_preprocess_bwd on each view in turn (up to
 * the fp32 summation order), but each Gaussian's parameter and SH rows are read once, the
 * chain rules of every view in which it is visible are summed on chip, and its gradient rows
 * are updated with ONE reduction (per-view K5 re-reads and re-reduces the rows once per view;
 * PAPER:43-46 is the training use). Every view must have completed rd_blend_bwd with the
 * same options; the caller orders `stream` after the views' streams (e.g. events) and
 * before any later use of the views' scratch. Errors: n_views ∉ [1, 8], NULL or repeated
 * views, differing Gaussians / options → RD_ERR_INVALID_ARGUMENT; a view before
 * rd_blend_bwd → RD_ERR_STATE. Timed (rd_get_timings) on views[0] as one K5 launch. */
rd_status rd_preprocess_bwd_views(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                  const rd_grads* grads, rd_stream stream);

/* K5 in two parts, for a caller that pipelines the views of a step: the GEOMETRY part of one
 * view (K5b64 + K5b: the chain rule of its 2-D gradients through the projection, conic, depth
 * plane and normal into means, scales, rotations, opacities — and means2d — plus the
 * 3D-filter mapping) may run on the view's stream right after its
 * rd_blend_bwd, while other views still blend; the SH part of a round of views (the colour
 * gradient into the SH rows and its view-direction term of dL/dμ) runs once all
 * of them are done. rd_preprocess_bwd_geometry on each view + rd_preprocess_bwd_views_sh on
 * the round = rd_preprocess_bwd_views on the round (up to the fp32 summation order: every
 * part adds with reductions). Same arguments, ordering rules and errors as
 * rd_preprocess_bwd / rd_preprocess_bwd_views; each is timed as a K5 launch. */
rd_status rd_preprocess_bwd_geometry(rd_view* view, const rd_gaussians* g, const rd_grads* grads, rd_stream stream);
rd_status rd_preprocess_bwd_views_sh(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                     const rd_grads* grads, rd_stream stream);

/* rd_preprocess_bwd_views with flags: RD_K5_SH_ONLY (= rd_preprocess_bwd_views_sh),
 * RD_K5_GEOMETRY_ONLY (the geometry parts of the views), RD_K5_SET_SH — the SH gradient rows
 * are SET instead of accumulated: every Gaussian's row is written, with 0 where it is visible
 * in none of the views, and the old values are never read (a caller whose step has one round
 * of views and who zeroes only the non-SH gradients saves the SH rows' zeroing and the read of
 * the reduction; needs sh_coeffs·3 a multiple of 4). Errors: unknown or contradictory flags →
 * RD_ERR_INVALID_ARGUMENT; otherwise as rd_preprocess_bwd_views. */
#define RD_K5_SH_ONLY 1u
#define RD_K5_GEOMETRY_ONLY 2u
#define RD_K5_SET_SH 4u
rd_status rd_preprocess_bwd_views_ex(rd_view* const* views, int32_t n_views, const rd_gaussians* g,
                                     const rd_grads* grads, uint32_t flags, rd_stream stream);

/* NEXT-2: normal consistency (reading S22) on rendered maps (device, fp32,
 * the layouts of rd_render_fwd): ñ = the finite-difference normal of the median depth map
 * (back-project the pixel and its right / lower neighbours with the camera intrinsics,
 * ñ = normalize((P_r − P) × (P_d − P)) oriented so ñ·P < 0, 0 where a depth is 0 or the
 * neighbour is outside the image), consistency[H][W] = Σ_i ω_i (1 − n_iᵀñ) = alpha − normal·ñ
 * (0 where ñ is 0), depth_normal[3][H][W] = ñ. Either output may be NULL. Only fx, fy, cx, cy,
 * width, height of `cam` are used. */
rd_status rd_normal_consistency(const rd_camera* cam, const float* depth, const float* alpha, const float* normal,
                                float* consistency, float* depth_normal, rd_stream stream);
/* Backward of Σ_p dL_dconsistency[p]·consistency[p] into the map cotangents, ACCUMULATED
 * (+=): dL_ddepth[H][W] (through ñ; neighbours by atomics), dL_dalpha[H][W],
 * dL_dnormal[3][H][W]; any may be NULL. Pass the results to rd_blend_bwd / rd_render_bwd. */
rd_status rd_normal_consistency_bwd(const rd_camera* cam, const float* depth, const float* normal,
                                    const float* dL_dconsistency, float* dL_ddepth, float* dL_dalpha,
                                    float* dL_dnormal, rd_stream stream);

/* NEXT-4: TSDF fusion of rendered median depth maps (reading S24). The volume
 * is a [Z][Y][X] grid of fp32 tsdf and weight (DEVICE, caller-owned, initialise weight = 0);
 * voxel (i, j, k) has its centre at origin + (i+½, j+½, k+½)·voxel_size. Each view updates
 * every voxel that is in front of the camera (z_c > znear), projects into the image and
 * finds a depth sample 0 < D ≤ max_depth with sdf = D − z_c > −truncation:
 * tsdf ← (w·tsdf + clamp(sdf/truncation, −1, 1))/(w + 1), w ← w + 1. Views are applied in
 * order; up to 32 views per kernel launch are fused (one read and one write of the volume per
 * 32 views). depths: DEVICE [n_views][H][W] (0 = hole), all cameras the same width/height;
 * cams: HOST array of n_views cameras. rd_marching_cubes extracts the mesh afterwards. */
typedef struct rd_tsdf {
  float origin[3];
  float voxel_size;
  int32_t dims[3];  /* X, Y, Z */
  float truncation; /* e.g. 4 voxel_size */
  float max_depth;  /* samples farther than this are ignored */
  float* tsdf;      /* [Z][Y][X] */
  float* weight;    /* [Z][Y][X] */
} rd_tsdf;
rd_status rd_tsdf_integrate(const rd_tsdf* volume, const float* depths, const rd_camera* cams, int32_t n_views,
                            rd_stream stream);

/* NEXT-4: marching cubes on the fused volume ("with the Marching Cube algorithm",
 * reading S25). Cells join 2×2×2 voxel centres; a cell with a corner of weight 0 is skipped;
 * corner c (x = c & 1, y = c >> 1 & 1, z = c >> 2 & 1) is inside when tsdf < iso. Each cell's
 * triangles come from the face-walking table of reading S25 (watertight, normals pointing from
 * inside to outside, ≤ 5 per cell); a vertex on the edge a→b is
 * p_a + (iso − v_a)/(v_b − v_a)·(p_b − p_a), in fp32. The output is a triangle soup in cell
 * order (x fastest, then y, z), triangles in table order: triangles = DEVICE f32
 * [capacity][3 vertices][xyz], caller-owned. *n_triangles (HOST) receives the count; the
 * triangles are written only when triangles != NULL and capacity ≥ the count (call once with
 * NULL to size the buffer, or pass a capacity guess and repeat only if it was short).
 * Synchronises `stream` once (to read the count back); its temporaries (8 B per cell + the
 * scan's) are a per-host-thread, grow-only cache kept across calls. Only volume->{origin,
 * voxel_size, dims, tsdf, weight} are read. */
rd_status rd_marching_cubes(const rd_tsdf* volume, float iso, float* triangles, int64_t capacity,
                            int64_t* n_triangles, rd_stream stream);

/* Profiling: when enabled, every kernel launch of this view is bracketed by CUDA events on
 * its stream and K3/K4 count the pairs they evaluate (a few atomics per warp). Enabling
 * or disabling resets the accumulators. rd_get_timings synchronises on the recorded
 * events, sums their durations into *out, and resets if `reset` is non-zero. */
rd_status rd_set_profiling(rd_view* view, int32_t enabled);
rd_status rd_get_timings(rd_view* view, rd_timings* out, int32_t reset);

/* Statistics of the last calls (host). */
rd_status rd_view_stats(const rd_view* view, rd_stats* out);

/* Debug copies (device → caller device buffers, async on `stream`), for bit-exact tests:
 *  rd_debug_binning: keys u64[M], ids u32[M] (sorted), ranges u32[2*T] ([first, last)).
 *  rd_debug_preprocess: records f32[n][16] (u_hi, v_hi, g11, g21, g22, log2 o, r, g, b, nx,
 *    ny, nz, z_c, p0, p1, uv_lo) with [[g11, g21], [0, g22]] the Cholesky factor U of
 *    (log2 e / 2)·[[a,b],[b,c]] (UᵀU), [[a,b],[b,c]] the conic of the dilated 2-D
 *    covariance, and uv_lo the bits of two fp16 remainders: u_c = u_hi + u_lo,
 *    v_c = v_hi + v_lo; rects u32[n][2] (x0 | y0 << 16, x1 | y1 << 16; tiles,
 *    half-open), tiles_touched u32[n]. Any pointer may be NULL. Valid for visible Gaussians.
 *  rd_debug_pixel_state: T_final f32[H*W], n_contrib i32[H*W], median_pos i32[H*W].
 *  rd_debug_grads2d: after rd_blend_bwd / rd_render_bwd, the per-Gaussian sums K4
 *    accumulated, as f32[n][16] (valid for visible Gaussians): Σ dA·dx, Σ dA·dy, Σ dA·dx²,
 *    Σ dA·dx·dy, Σ dA·dy² (accumulated in fp64), Σ dA, Σ w·g_C (3), Σ w·g_N (3), and over
 *    the pixels whose median splat it is Σ g_D, Σ g_D·dx, Σ g_D·dy; then 0. Here
 *    dA = α_raw·∂L/∂α, (dx, dy) = centre − pixel, w = α·T. */
rd_status rd_debug_binning(const rd_view* view, uint64_t* keys, uint32_t* ids, uint32_t* ranges, rd_stream stream);
rd_status rd_debug_preprocess(const rd_view* view, float* records, uint32_t* rects, uint32_t* tiles_touched,
                              rd_stream stream);
rd_status rd_debug_pixel_state(const rd_view* view, float* T_final, int32_t* n_contrib, int32_t* median_pos,
                               rd_stream stream);
rd_status rd_debug_grads2d(const rd_view* view, float* grads2d, rd_stream stream);

/* Thread-local message of the last error ("" if none). */
const char* rd_last_error(void);

/* Library version / build string. */
const char* rd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RADE_H_ */
