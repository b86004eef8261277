// regularize.cu — NEXT-2 of the RaDe-GS hot path, sm_100a: the normal-consistency term
// on the rendered maps, and its backward into the map cotangents that
// rd_blend_bwd then takes. Image-space, one thread per pixel, memory-bound (≈ 36 B/px in,
// 16 B/px out forward).
//
// Reading S22: ñ from finite differences of the median depth map — back-project
// the pixel centre and its right and lower neighbours, P = D·r, r = ((x+½−cx)/fx,
// (y+½−cy)/fy, 1); m = (P_right − P) × (P_down − P); ñ = s·m/‖m‖ with s = ±1 so that
// ñ·P < 0; undefined (ñ = 0, L_n = 0) where any of the three depths is 0 (no median depth)
// or the neighbour is outside the image. L_n = Σ_i ω_i (1 − n_iᵀñ) = A − Nᵀñ per pixel,
// A the alpha map, N the normal map.
#include "rade_internal.cuh"

namespace rade {
namespace {

struct Intr {
  float fx, fy, cx, cy;
  int W, H;
};

__device__ __forceinline__ float3 ray(const Intr& c, int x, int y) {
  return make_float3(((float)x + 0.5f - c.cx) / c.fx, ((float)y + 0.5f - c.cy) / c.fy, 1.f);
}
__device__ __forceinline__ float3 f3sub(float3 a, float3 b) { return make_float3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 f3scale(float3 a, float s) { return make_float3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float f3dot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 f3cross(float3 a, float3 b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// The stencil of pixel (x, y): false if ñ is undefined there.
struct Stencil {
  float3 P, a, b, n;  // P, P_right − P, P_down − P, ñ
  float s, inv_len;   // orientation sign, 1/‖m‖
};
__device__ __forceinline__ bool stencil(const Intr& c, const float* __restrict__ depth, int x, int y, Stencil& st) {
  if (x + 1 >= c.W || y + 1 >= c.H) return false;
  const int p = y * c.W + x;
  const float d = depth[p], dr = depth[p + 1], dd = depth[p + c.W];
  if (d == 0.f || dr == 0.f || dd == 0.f) return false;
  st.P = f3scale(ray(c, x, y), d);
  st.a = f3sub(f3scale(ray(c, x + 1, y), dr), st.P);
  st.b = f3sub(f3scale(ray(c, x, y + 1), dd), st.P);
  const float3 m = f3cross(st.a, st.b);
  const float len = sqrtf(f3dot(m, m));
  if (!(len > 0.f)) return false;
  st.inv_len = 1.f / len;
  st.s = f3dot(m, st.P) > 0.f ? -1.f : 1.f;
  st.n = f3scale(m, st.s * st.inv_len);
  return true;
}

__global__ void __launch_bounds__(256) k_normal_consistency(Intr c, const float* __restrict__ depth,
                                                            const float* __restrict__ alpha,
                                                            const float* __restrict__ normal, float* __restrict__ Ln,
                                                            float* __restrict__ nt) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= c.W || y >= c.H) return;
  const int p = y * c.W + x, HW = c.W * c.H;
  Stencil st;
  const bool ok = stencil(c, depth, x, y, st);
  const float3 n = ok ? st.n : make_float3(0.f, 0.f, 0.f);
  if (Ln) {
    const float3 N = make_float3(normal[p], normal[HW + p], normal[2 * HW + p]);
    Ln[p] = ok ? alpha[p] - f3dot(N, n) : 0.f;
  }
  if (nt) {
    nt[p] = n.x;
    nt[HW + p] = n.y;
    nt[2 * HW + p] = n.z;
  }
}

// Backward of Σ_p g_p L_n(p): dL/dA_p += g_p, dL/dN_p += −g_p ñ_p, and through ñ = s m/‖m‖,
// m = a × b, a = P_r − P, b = P_d − P, P = D r into the three depths of the stencil
// (the neighbours' by atomics: a pixel's depth feeds three stencils).
__global__ void __launch_bounds__(256) k_normal_consistency_bwd(Intr c, const float* __restrict__ depth,
                                                                const float* __restrict__ normal,
                                                                const float* __restrict__ gL, float* __restrict__ gD,
                                                                float* __restrict__ gA, float* __restrict__ gN) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= c.W || y >= c.H) return;
  const int p = y * c.W + x, HW = c.W * c.H;
  Stencil st;
  if (!stencil(c, depth, x, y, st)) return;
  const float g = gL[p];
  if (g == 0.f) return;
  if (gA) gA[p] += g;
  const float3 N = make_float3(normal[p], normal[HW + p], normal[2 * HW + p]);
  if (gN) {
    gN[p] -= g * st.n.x;
    gN[HW + p] -= g * st.n.y;
    gN[2 * HW + p] -= g * st.n.z;
  }
  if (!gD) return;
  const float3 gn = f3scale(N, -g);                                           // dL/dñ
  const float3 gm = f3scale(f3sub(gn, f3scale(st.n, f3dot(st.n, gn))), st.s * st.inv_len);  // dL/dm
  const float3 ga = f3cross(st.b, gm), gb = f3cross(gm, st.a);                // m = a × b
  atomicAdd(gD + p, -f3dot(make_float3(ga.x + gb.x, ga.y + gb.y, ga.z + gb.z), ray(c, x, y)));  // P
  atomicAdd(gD + p + 1, f3dot(ga, ray(c, x + 1, y)));    // P_right
  atomicAdd(gD + p + c.W, f3dot(gb, ray(c, x, y + 1)));  // P_down
}

}  // namespace

void launch_normal_consistency(float fx, float fy, float cx, float cy, int W, int H, const float* depth,
                               const float* alpha, const float* normal, float* Ln, float* nt, cudaStream_t s) {
  if (W == 0 || H == 0) return;
  const dim3 grid((W + 31) / 32, (H + 7) / 8);
  k_normal_consistency<<<grid, 256, 0, s>>>(Intr{fx, fy, cx, cy, W, H}, depth, alpha, normal, Ln, nt);
}

void launch_normal_consistency_bwd(float fx, float fy, float cx, float cy, int W, int H, const float* depth,
                                   const float* normal, const float* gL, float* gD, float* gA, float* gN,
                                   cudaStream_t s) {
  if (W == 0 || H == 0) return;
  const dim3 grid((W + 31) / 32, (H + 7) / 8);
  k_normal_consistency_bwd<<<grid, 256, 0, s>>>(Intr{fx, fy, cx, cy, W, H}, depth, normal, gL, gD, gA, gN);
}

}  // namespace rade
