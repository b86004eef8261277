// rade_internal.cuh — device-side types and math shared by the sm_100a kernels of the
// RaDe-GS rasterizer (K1 preprocess, K2 binning, K3 blend fwd, K4 blend bwd, K5
// preprocess bwd). Nothing here is shared with oracle/ (which is test infrastructure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
};

struct DevGrads {
  float* __restrict__ means;
  float* __restrict__ scales;
  float* __restrict__ rot;
  float* __restrict__ opac;
  float* __restrict__ sh;
};

// Per-visible-Gaussian record written by K1 and gathered by K3/K4 (64 B, 4 x float4):
//   r0 = (u_c, v_c, A2, B2)   r1 = (C2, log2 o, R, G)   r2 = (B, nx, ny, nz)   r3 = (z_c, p0, p1, 1/o)
// where (A2, B2, C2) = log2(e) * (-a/2, -b, -c/2) for the conic [[a, b], [b, c]] of the
// dilated 2-D covariance, so that G = exp2(A2 dx^2 + B2 dx dy + C2 dy^2) with
// (dx, dy) = (u_c - u, v_c - v) (readings S1, S4, S5).
struct __align__(16) Record {
  float4 r0, r1, r2, r3;
};

// 2-D gradient accumulator per Gaussian (64 B):
//   du, dv, dA2, dB2, dC2, dopacity, dR, dG, dB, dnx, dny, dnz, dz, dp0, dp1, unused
constexpr int kG2D = 16;

// 16-byte global → shared copy without a register round trip (cp.async / LDGSTS, L2-only).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
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
//   e = A2 dx² + B2 dx dy + C2 dy² + lo,   α_raw = o·exp(−½ΔᵀCΔ) = 2^e,
// so the α ≥ α_min test is e ≥ log2(α_min) — taken BEFORE the exp2, which rejected pairs
// never evaluate — and α = min(α_max, 2^e) (readings S1, S8).
struct PairAlpha {
  float dx, dy, e;
  bool pass;
};
__device__ __forceinline__ PairAlpha pair_power(const float4& r0, float C2, float lo, float px, float py,
                                                float log2_alpha_min) {
  PairAlpha pa;
  pa.dx = __fsub_rn(r0.x, px);
  pa.dy = __fsub_rn(r0.y, py);
  const float inner = __fmaf_rn(r0.z, pa.dx, __fmul_rn(r0.w, pa.dy));                    // A2 dx + B2 dy
  const float pw = __fmaf_rn(pa.dx, inner, __fmul_rn(__fmul_rn(C2, pa.dy), pa.dy));     // + C2 dy²
  pa.e = __fadd_rn(pw, lo);
  pa.pass = pa.e >= log2_alpha_min;
  return pa;
}

// ------------------------------------------------------------------ launchers (host)
// Profiling counters (nullable): [0] pairs evaluated by K3, [1] pairs blended by K3,
// [2] pairs evaluated by K4, [3] visible Gaussians (K1).
typedef unsigned long long Counter;
constexpr int kNumCounters = 4;

__device__ __forceinline__ void warp_count(Counter* ctr, unsigned v) {
  // all 32 lanes must call this (converged)
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, (Counter)v);
}

// K1 also writes the depth-sort input: dkey[i] = float_bits(z_c) (0xFFFFFFFF if the
// Gaussian touches no tile) and didx[i] = i, and appends the visible ids to vis
// (*n_visible, zeroed beforehand).
void launch_preprocess_fwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, int tiles_x, Record* rec,
                           uint2* rect, uint32_t* tiles_touched, uint32_t* dkey, uint32_t* didx, uint32_t* n_visible,
                           uint32_t* vis, Counter* counters, cudaStream_t s);
// K5 = K5a (SH; over the n_vis visible ids of K1's list) then K5b (geometry, id order).
void launch_preprocess_bwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, const uint32_t* tiles_touched,
                           const uint32_t* vis, int64_t n_vis, const float* g2d, DevGrads grads, cudaStream_t s);
// K2 (binning.cu). Sorts return the CUB DoubleBuffer selector (1: result in the *1 buffers).
size_t binning_temp_bytes(int64_t n, int64_t m, int tile_bits);
int launch_depth_sort(uint32_t* dkey0, uint32_t* dkey1, uint32_t* idx0, uint32_t* idx1, int64_t n, void* temp,
                      size_t temp_bytes, cudaStream_t s);
void launch_scan(const uint32_t* sorted_ids, const uint32_t* tiles_touched, uint32_t* offsets, int64_t n, void* temp,
                 size_t temp_bytes, cudaStream_t s);
void launch_duplicate(int64_t n, int64_t m, const uint32_t* offsets, const uint32_t* sorted_ids, const uint2* rect,
                      int tiles_x, uint32_t* tile_keys, uint32_t* vals, cudaStream_t s);
int launch_tile_sort(uint32_t* keys0, uint32_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t m, int tile_bits,
                     void* temp, size_t temp_bytes, cudaStream_t s);
void launch_ranges(const uint32_t* keys, int64_t m, int n_tiles, uint2* ranges, cudaStream_t s);
// debug: 64-bit keys (tile << 32 | float_bits(z_c)) of the sorted list
void launch_keys64(const uint32_t* tiles, const uint32_t* ids, const Record* rec, int64_t m, uint64_t* out,
                   cudaStream_t s);
void launch_render_fwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, float* color, float* depth, float* normal,
                       float* alpha, float* T_final, int32_t* n_contrib, int32_t* median_pos, Counter* counters,
                       cudaStream_t s);
void launch_render_bwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, const float* T_final, const int32_t* n_contrib,
                       const int32_t* median_pos, const float* dL_dcolor, const float* dL_ddepth,
                       const float* dL_dnormal, const float* dL_dalpha, float* g2d, Counter* counters,
                       cudaStream_t s);

}  // namespace rade
