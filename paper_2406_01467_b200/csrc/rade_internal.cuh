// rade_internal.cuh — device-side types and math shared by the sm_100a kernels of the
// RaDe-GS rasterizer (K1 preprocess, K2 binning, K3 blend fwd, K4 blend bwd, K5
// preprocess bwd). Nothing here is shared with oracle/ (which is test infrastructure).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#ifdef RD_CHECKS
#include <cstdio>
#endif

namespace rade {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Camera as the kernels see it (by value in kernel parameters).
struct DevCam {
  float fx, fy, cx, cy;
  int W, H;
  float R[9];   // world -> camera, row-major
  float t[3];
  float znear;
  float campos[3];  // -R^T t (camera centre in world space), for SH view directions
  // guard band (reading S6b, rd_options.guard_band = g > 0): float(−g W − cx), float((1+g) W − cx),
  // same for v; guard = 0: off
  int guard;
  float gu0, gu1, gv0, gv1;
};

struct DevOpt {
  int tile;
  float alpha_min, alpha_max, T_min, median_T, dilation;
  float bg[3];
  int sh_degree;  // active degree
  float ln_alpha_min;
  float log2_alpha_min;
};

struct DevGauss {
  int64_t n;
  int sh_coeffs;
  const float* __restrict__ means;
  const float* __restrict__ scales;
  const float* __restrict__ rot;
  const float* __restrict__ opac;
  const float* __restrict__ sh;
  const float* __restrict__ filter3d;  // NULL, or the 3D filter size per Gaussian (reading S23)
};

struct DevGrads {
  float* __restrict__ means;
  float* __restrict__ scales;
  float* __restrict__ rot;
  float* __restrict__ opac;
  float* __restrict__ sh;
  float* __restrict__ means2d;  // optional [n][2]: dL/d(u_c, v_c)
};

// Per-visible-Gaussian record written by K1 and gathered by K3/K4 (64 B, 4 x float4):
//   r0 = (u_hi, v_hi, g11, g21)   r1 = (g22, log2 o, R, G)   r2 = (B, nx, ny, nz)
//   r3 = (z_c, p0, p1, half2(u_lo, v_lo))
// where UᵀU = (log2 e / 2)·[[a, b], [b, c]], U = [[g11, g21], [0, g22]], is the Cholesky
// factor of the conic of the dilated 2-D covariance, so that
//   G = exp(−½ΔᵀCΔ) = 2^−((g11 dx + g21 dy)² + (g22 dy)²),  (dx, dy) = (u_c − u, v_c − v)
// (readings S1, S4, S5). A sum of two squares has no cancellation: the
// expanded a·dx² + 2b·dx·dy + c·dy² of a long thin splat is a difference of terms ~10⁵
// times larger than the result, whose fp32 rounding would move α by percents. The centre
// is a float + half pair, u_c = u_hi + u_lo: an fp32 pixel coordinate alone carries up to
// 3e-5 px of rounding at u ~ 600, which moves α of a 1-px splat by ~6e-5 relative.
struct __align__(16) Record {
  float4 r0, r1, r2, r3;
};

// Per-Gaussian backward sums, accumulated by K4's atomics over (pixel, splat) pairs and
// read by K5 (80 B row; zeroed by K1 for every visible Gaussian). dA = α_raw·∂L/∂α,
// (dx, dy) = centre − pixel, w = α T, g_* the pixel cotangents:
//   m[0..4] = Σ dA·dx, Σ dA·dy, Σ dA·dx², Σ dA·dx·dy, Σ dA·dy²   (fp64: for screen-sized
//             splats these are sums of ~10⁶ terms of size ~10⁶ whose result is orders of
//             magnitude smaller; fp32 atomics would leave ~1e-6 relative noise, which the
//             chain rule through the conic amplifies ~10⁴-fold)
//   f[0] = Σ dA, f[1..3] = Σ w·g_C, f[4..6] = Σ w·g_N,
//   f[7..9] = Σ g_D, Σ g_D·dx, Σ g_D·dy over the pixels whose median splat this is.
struct __align__(16) G2D {
  double m[5];
  float f[10];
};
static_assert(sizeof(G2D) == 80, "G2D row");
// K5b runs in fp64 for splats whose tile rect covers more pixels than this (their conic
// gradient is the small difference of large terms); in fp32 otherwise.
constexpr uint32_t kBigPixels = 64 * 256;
__device__ __forceinline__ bool is_big(uint32_t tiles_touched, int tile) {
  return tiles_touched * (uint32_t)(tile * tile) > kBigPixels;
}

// 16-byte global → shared copy without a register round trip (cp.async / LDGSTS, L2-only).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Shared-memory loads through a precomputed 32-bit shared address (keeps the address
// arithmetic out of the inner loops; ptxas otherwise re-derives the shared window base).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));  // opaque: not rematerialised in loops
  return r;
}
__device__ __forceinline__ float4 lds128(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(unsigned a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The per-pair α evaluation shared bit-for-bit by K3 and K4 (explicit roundings so the
// two kernels take identical skip / stop decisions). With lo = log2(o) stored in the record,
//   e = lo − (g11 dx + g21 dy)² − (g22 dy)²,   α_raw = o·exp(−½ΔᵀCΔ) = 2^e,
// so the α ≥ α_min test is e ≥ log2(α_min) — taken BEFORE the exp2, which rejected pairs
// never evaluate — and α = min(α_max, 2^e) (readings S1, S8).
struct PairAlpha {
  float dx, dy, e;
  bool pass;
};
// (u_lo, v_lo) of a record's r3.w
__device__ __forceinline__ float2 uv_lo(float w) { return __half22float2(*reinterpret_cast<const __half2*>(&w)); }
// dx = (u_hi − px) + u_lo: the first difference is exact or carries |dx|-relative rounding
// only, so Δ is accurate to ~1e-7·|Δ| + the half rounding of u_lo (< 3e-8 px).
// A thread's pixels share their column: the column terms dx and g11·dx come from
// pair_column once per splat, pair_power adds the row terms per pixel.
struct PairColumn {
  float dx, g11dx;
};
__device__ __forceinline__ PairColumn pair_column(const float4& r0, float2 ulo, float px) {
  PairColumn c;
  c.dx = __fadd_rn(__fsub_rn(r0.x, px), ulo.x);
  c.g11dx = __fmul_rn(r0.z, c.dx);
  return c;
}
__device__ __forceinline__ PairAlpha pair_power(const float4& r0, float g22, float lo, float2 ulo,
                                                const PairColumn& col, float py, float log2_alpha_min) {
  PairAlpha pa;
  pa.dx = col.dx;
  pa.dy = __fadd_rn(__fsub_rn(r0.y, py), ulo.y);
  const float t1 = __fmaf_rn(r0.w, pa.dy, col.g11dx);  // g11 dx + g21 dy
  const float t2 = __fmul_rn(g22, pa.dy);
  const float pw = __fmaf_rn(t1, t1, __fmul_rn(t2, t2));
  pa.e = __fsub_rn(lo, pw);
  pa.pass = pa.e >= log2_alpha_min;
  return pa;
}

// Depth distortion (reading S21) plumbing: K3 writes the L_d map (dist, may be NULL) and the
// per-pixel state d0 (first blended depth) and D1 = Σω(d − d0) when d0 != NULL; K4 adds the
// L_d gradient when dL_ddist != NULL (then d0/D1 must hold K3's values).
// Debug build (-DRD_CHECKS, `python -m paper_2406_01467_b200.build --checks` → librade_checks.so,
// selected with RADE_LIB): device-side bounds assertions on the index math of the binning
// passes, K1's list appends and K3/K4's staging, blend-mask words and record gathers — a
// failed check prints its condition and traps (the launch fails with an error). compute-
// sanitizer is not available on the GPU pool, so this build plus the bit-exact / rerun
// determinism tests stand in for memcheck / racecheck.
#ifdef RD_CHECKS
#define RD_CHECK(cond)                                                                                         \
  do {                                                                                                         \
    if (!(cond)) {                                                                                             \
      printf("RD_CHECK failed %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                                \
      __trap();                                                                                                \
    }                                                                                                          \
  } while (0)
#else
#define RD_CHECK(cond) \
  do {                 \
  } while (0)
#endif
// Capacities the RD_CHECKS build checks K3/K4's indices against (unused otherwise).
struct DevBounds {
  int64_t n;           // Gaussians (records)
  int64_t m;           // duplicates (sorted ids)
  int64_t mask_words;  // blend-mask words
  int64_t n_tiles;
};

struct DistIO {
  float* dist;
  float* d0;
  float* D1;
  const float* dL_ddist;
};

// ------------------------------------------------------------------ launchers (host)
// Profiling counters (nullable): [0] pairs evaluated by K3, [1] pairs blended by K3,
// [2] pairs evaluated by K4, [3] visible Gaussians (K1), [4] Gaussians visible in at least
// one view of a batched K5 (rd_preprocess_bwd_views), [5 + 64 r + b] K1's culls by reason r
// (invalid input, near plane, guard band, opacity < alpha_min, degenerate, off screen),
// spread over 64 slots b so the atomics of 23 k warps do not all hit one address.
typedef unsigned long long Counter;
constexpr int kIssuedCounter = 5;  // K3: warp steps × 64 pixels
constexpr int kCullCounter0 = 6;
constexpr int kCullSlots = 64;  // each reason's count spread over 64 addresses (block index mod 64)
constexpr int kNumCounters = kCullCounter0 + 6 * kCullSlots;

__device__ __forceinline__ void warp_count(Counter* ctr, unsigned v) {
  // all 32 lanes must call this (converged)
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, (Counter)v);
}

// K1 also writes the depth-sort input dkey[i] = float_bits(z_c) in id order (0xFFFFFFFF if
// the Gaussian touches no tile), zeroes the G2D row of every visible Gaussian, appends the
// visible ids to vis (count[0]) and the big ones (is_big) to big (count[1]); count is zeroed
// beforehand.
void launch_preprocess_fwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, int tiles_x, Record* rec,
                           uint2* rect, uint32_t* tiles_touched, uint32_t* dkey, uint32_t* count,
                           uint32_t* vis, uint32_t* big, G2D* g2d, Counter* counters, cudaStream_t s);
// K5 = K5a (SH; over the n_vis visible ids of K1's list) then K5b (geometry: fp32 in id
// order for the visible Gaussians that are not is_big, fp64 over the big list).
// K1 over a round of views (rd_preprocess_views): per view its camera and output arrays
struct K1Out {
  DevCam cam;
  Record* rec;
  uint2* rect;
  uint32_t* touched;
  uint32_t* dkey;
  uint32_t* count;
  uint32_t* vis;
  uint32_t* big;
  G2D* g2d;
  Counter* counters;
};
struct K1Views {
  int nv;
  K1Out v[8];
};
void launch_preprocess_fwd_views(const DevGauss& g, const DevOpt& opt, const K1Views& kv, cudaStream_t s);
// K5 parts: the SH colour (+ view-direction) part and the geometry part (K5b64 + K5b); both
// add into the gradients with reductions, so they may run in any order
constexpr int kK5Sh = 1, kK5Geometry = 2, kK5All = 3;
// with kK5Sh: SET the SH gradient rows instead of adding (every row written, 0 for Gaussians
// visible in none of the views; only by the batched views kernel, rows of 4k floats)
constexpr int kK5ShSet = 4;
void launch_preprocess_bwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, const uint32_t* tiles_touched,
                           const uint32_t* vis, int64_t n_vis, const uint32_t* big, int64_t n_big, const G2D* g2d,
                           DevGrads grads, cudaStream_t s, int parts = kK5All);
// K5 for nv ≤ kMaxBatchViews views of the same Gaussians at once (rd_preprocess_bwd_views):
// per-view cameras, tiles_touched, G2D rows, visible and big lists; gradients += the sum over
// the views (the SH part fused over the views, the geometry part per view).
constexpr int kMaxBatchViews = 8;
void launch_preprocess_bwd_views(const DevGauss& g, const DevOpt& opt, int nv, const DevCam* cams,
                                 const uint32_t* const* touched, const G2D* const* g2d, const uint32_t* const* vis,
                                 const int64_t* n_vis, const uint32_t* const* big, const int64_t* n_big,
                                 DevGrads grads, Counter* counters, cudaStream_t s, int parts = kK5All);
// debug: G2D rows → f32 [n][16] (m[0..4], f[0..9], 0)
void launch_g2d_to_f32(const G2D* g2d, int64_t n, float* out, cudaStream_t s);
// K2 (binning.cu). Sorts return the CUB DoubleBuffer selector (1: result in the *1 buffers).
// K2 (binning.cu): hand-written onesweep radix passes with decoupled look-back. BinSort is the
// view's look-back state: status words (zeroed when allocated, epoch-tagged after that) and
// the host-side epoch counter.
struct BinSort {
  unsigned long long* status;
  uint32_t epoch;
};
size_t bin_status_words(int64_t n_items);
size_t bin_bstart_words(int64_t m);
int bin_max_tiles_per_axis();
int bin_bases_words();
// bincnt layout (u32): [0] visible, [1] big (K1), [2] M (K2h) (zeroed before K1), [3] K2h's
// done-counter (zeroed before K1, reset by K2h), [4, 4 + 1024) the four depth digit
// histograms, then diff_x[tiles_x + 1], diff_y[tiles_y + 1] (zeroed before K2h), then the
// digit bases of every pass (bin_bases_words(), written by K2h)
constexpr int kBinCntHist = 4;
constexpr int kBinCntDiff = 4 + 1024;
// K2h: also adds M to cnt[2] and writes cnt[0..2] to host_counts (mapped pinned memory)
void launch_bin_hist(int64_t n, const uint32_t* dkey, const uint2* rect, int tiles_x, int tiles_y, uint32_t* cnt,
                     uint32_t* bases, uint32_t* host_counts, cudaStream_t s);
void launch_depth_pass(int p, const uint32_t* dkey_id_order, int64_t n, const uint32_t* n_vis_dev,
                       const uint32_t* bases, uint32_t* const kb[2], uint32_t* const vb[2], BinSort& bs,
                       cudaStream_t s);
void launch_scan(const uint32_t* sorted_ids, const uint2* rect, uint2* rect_s, uint32_t* offsets, int64_t n_max,
                 const uint32_t* n_dev, uint32_t* bstart, int64_t m, BinSort& bs, cudaStream_t s);
int tile_sort_passes(int tiles_x, int tiles_y);
// exclusive scan of n u32 (look-back state bs: scan_status_words(n) words, zeroed when allocated)
size_t scan_status_words(int64_t n);
void launch_scan_excl_u32(const uint32_t* in, uint32_t* out, int64_t n, BinSort& bs, cudaStream_t s);
void launch_tile_pass(int p, int64_t m, int64_t n_gauss, const uint32_t* offsets, const uint32_t* sorted_ids,
                      const uint2* rect, const uint32_t* bstart, int tiles_x, int tiles_y, const uint32_t* bases,
                      uint32_t* const kb[2], uint32_t* const vb[2], BinSort& bs, cudaStream_t s);
void launch_ranges(const uint32_t* keys, int64_t m, int n_tiles, uint2* ranges, cudaStream_t s);
// NEXT-2 (regularize.cu): L_n = A − Nᵀñ per pixel and ñ (either may be NULL); backward adds
// into the map cotangents gD (atomics), gA, gN (any may be NULL).
void launch_normal_consistency(float fx, float fy, float cx, float cy, int W, int H, const float* depth,
                               const float* alpha, const float* normal, float* Ln, float* nt, cudaStream_t s);
void launch_normal_consistency_bwd(float fx, float fy, float cx, float cy, int W, int H, const float* depth,
                                   const float* normal, const float* gL, float* gD, float* gA, float* gN,
                                   cudaStream_t s);
// NEXT-4 (tsdf.cu): fuse n_views ≤ tsdf_views_per_launch() depth maps [n_views][H][W]; cam_rows
// = n_views × 17 floats (R[9], t[3], fx, fy, cx, cy, znear); dims = X, Y, Z; tsdf/weight [Z][Y][X].
int tsdf_views_per_launch();
void launch_tsdf_integrate(const float* cam_rows, int n_views, const float* depths, int W, int H, const float origin[3],
                           float voxel, float trunc, float max_depth, const int dims[3], float* tsdf, float* weight,
                           cudaStream_t s);
// NEXT-4 (mcubes.cu): count, scan, emit; synchronises s once. cudaErrorInvalidValue when the
// volume has ≥ 2^31 cells. triangles: f32 [capacity][3][3], written iff capacity ≥ count.
cudaError_t launch_marching_cubes(const float origin[3], float voxel, const int dims[3], const float* tsdf,
                                  const float* weight, float iso, float* triangles, int64_t capacity,
                                  int64_t* n_triangles, cudaStream_t s);
// debug: 64-bit keys (tile << 32 | float_bits(z_c)) of the sorted list
void launch_keys64(const uint32_t* tiles, const uint32_t* ids, const Record* rec, int64_t m, uint64_t* out,
                   cudaStream_t s);
// order: tiles_x·tiles_y u32, the K3/K4 launch order written by launch_render_fwd (read by the
// backward of the same forward).
// K3/K4 blend mask (tile 8): ≥ blend_mask_words(M, n_tiles) u32, written by K3, read by K4.
inline size_t blend_mask_words(int64_t m, int n_tiles) { return (size_t)(m / 32) + (size_t)n_tiles + 8; }
void launch_render_fwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, float* color, float* depth, float* normal,
                       float* alpha, float* T_final, int32_t* n_contrib, int32_t* median_pos, const DistIO& dio,
                       uint32_t* bmask, uint32_t* order, Counter* counters, const DevBounds& bd, cudaStream_t s);
void launch_render_bwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, const float* T_final, const int32_t* n_contrib,
                       const int32_t* median_pos, const float* dL_dcolor, const float* dL_ddepth,
                       const float* dL_dnormal, const float* dL_dalpha, const DistIO& dio,
                       const uint32_t* bmask, const uint32_t* order, G2D* g2d, Counter* counters,
                       const DevBounds& bd, cudaStream_t s);

}  // namespace rade
