// render.cu — stage 3 (K3, blend forward) and the first half of stage 4 (K4, blend
// backward) of the RaDe-GS rasterizer, sm_100a.
//
// One CTA per TILE×TILE tile, one thread per pixel (sampled at (i+½, j+½), reading S4).
// Each CTA walks its tile's depth-sorted list (ranges from K2) in batches of TILE² splats
// staged in shared memory (one coalesced 64-B record gather per thread), the whole block
// leaving as soon as every pixel is saturated (__syncthreads_count).
//
// Per (pixel, splat), front to back (Eq.3; readings S1, S8, S9, S10):
//   α = min(α_max, o·exp(−½ Δᵀ conic Δ)), Δ = (u_c − u, v_c − v)  (skip if α < α_min)
//   T′ = T(1 − α); stop before blending if T′ < T_min
//   w = α T; C += w c; N += w n
//   first splat with T > median_T ≥ T′: D = z_c + p·Δ        (Eq.4)
// Epilogue: C += T·bg, A = 1 − T; per pixel state (T_final, n_contrib, median_pos) for K4.
//
// K4 replays each pixel's list backwards from n_contrib, reconstructing T_i = T_{i+1}/(1−α_i)
// and suffix sums of colour and normal, and produces the 15 per-splat 2-D gradients, which
// are warp-reduced with shuffles before one set of L2 atomics per (warp, splat).
#include "rade_internal.cuh"

namespace rade {
namespace {

template <int TILE>
__global__ void __launch_bounds__(TILE* TILE) k_render_fwd(DevCam cam, DevOpt opt, int tiles_x,
                                                            const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ ids,
                                                            const Record* __restrict__ rec, float* __restrict__ color,
                                                            float* __restrict__ depth, float* __restrict__ normal,
                                                            float* __restrict__ alpha_out, float* __restrict__ T_final,
                                                            int32_t* __restrict__ n_contrib,
                                                            int32_t* __restrict__ median_pos,
                                                            Counter* __restrict__ counters) {
  constexpr int BLOCK = TILE * TILE;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * TILE + (int)(threadIdx.x % TILE), py = ty * TILE + (int)(threadIdx.x / TILE);
  const bool inside = px < cam.W && py < cam.H;
  const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
  const uint2 range = ranges[tile];
  const int total = (int)(range.y - range.x);

  __shared__ float4 s0[BLOCK], s1[BLOCK], s2[BLOCK];
  __shared__ uint32_t sid[BLOCK];

  float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, N0 = 0.f, N1 = 0.f, N2 = 0.f, D = 0.f;
  int last = 0, med = -1;
  unsigned n_eval = 0, n_blend = 0;
  bool done = !inside;
  for (int base = 0; base < total; base += BLOCK) {
    if (__syncthreads_count(done) == BLOCK) break;
    const int k = base + (int)threadIdx.x;
    if (k < total) {
      const uint32_t id = ids[range.x + k];
      const Record* r = rec + id;
      sid[threadIdx.x] = id;
      s0[threadIdx.x] = r->r0;
      s1[threadIdx.x] = r->r1;
      s2[threadIdx.x] = r->r2;
    }
    __syncthreads();
    const int cnt = min(BLOCK, total - base);
    for (int j = 0; j < cnt && !done; ++j) {
      const float4 a0 = s0[j], a1 = s1[j];
      const PairAlpha pa = eval_alpha(a0, a1.x, a1.y, fpx, fpy, opt.alpha_max);
      ++n_eval;
      if (pa.alpha < opt.alpha_min) continue;
      const float Tn = __fmul_rn(T, __fsub_rn(1.f, pa.alpha));
      if (Tn < opt.T_min) {
        done = true;
        break;
      }
      const float4 a2 = s2[j];
      const float w = __fmul_rn(pa.alpha, T);
      C0 = __fmaf_rn(w, a1.z, C0);
      C1 = __fmaf_rn(w, a1.w, C1);
      C2 = __fmaf_rn(w, a2.x, C2);
      N0 = __fmaf_rn(w, a2.y, N0);
      N1 = __fmaf_rn(w, a2.z, N1);
      N2 = __fmaf_rn(w, a2.w, N2);
      if (T > opt.median_T && Tn <= opt.median_T) {
        const float4 a3 = rec[sid[j]].r3;  // (z_c, p0, p1): once per pixel
        D = __fmaf_rn(a3.y, pa.dx, __fmaf_rn(a3.z, pa.dy, a3.x));
        med = base + j;
      }
      T = Tn;
      last = base + j + 1;
      ++n_blend;
    }
  }
  if (counters) {
    warp_count(counters + 0, n_eval);
    warp_count(counters + 1, n_blend);
  }
  if (!inside) return;
  const int HW = cam.W * cam.H;
  const int pix = py * cam.W + px;
  if (color) {
    color[pix] = __fmaf_rn(T, opt.bg[0], C0);
    color[HW + pix] = __fmaf_rn(T, opt.bg[1], C1);
    color[2 * HW + pix] = __fmaf_rn(T, opt.bg[2], C2);
  }
  if (normal) {
    normal[pix] = N0;
    normal[HW + pix] = N1;
    normal[2 * HW + pix] = N2;
  }
  if (depth) depth[pix] = D;
  if (alpha_out) alpha_out[pix] = 1.f - T;
  T_final[pix] = T;
  n_contrib[pix] = last;
  median_pos[pix] = med;
}

// Reduce-scatter of v[0..15] across the warp (16 shuffles instead of 75 for a plain
// all-reduce of 15 values): level off=16,8,4,2 halves the set of values a lane keeps (the
// half selected by that lane bit) and adds the partner's copy of it; a final xor-1 exchange
// completes the sum. Returns Σ_lanes v[lane >> 1] (lanes l and l^1 hold the same value).
__device__ __forceinline__ float reduce_scatter16(float (&v)[16], int lane) {
#pragma unroll
  for (int half = 8, off = 16; half >= 1; half >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < half; ++k) {
      const float send = up ? v[k] : v[k + half];
      const float keep = up ? v[k + half] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// K4. Per pixel, reverse replay of its blended splats. With the per-pixel scalar
//   D_i = Σ_{j>i} w_j (c_j·g_C + n_j·g_N)   (suffix sum, w_j = α_j T_j)
// the α gradient of Eq.3's colour and of the normal map is
//   ∂L/∂α_i = T_i (c_i·g_C + n_i·g_N) − D_i / (1 − α_i) + T_final/(1 − α_i) (g_A − bg·g_C),
// (3DGS-style derivation collapsed to one scalar: gC, gN are per-pixel constants). The 15
// per-splat values (du, dv, dA2, dB2, dC2, do, dRGB, dN, and at the pixel's median splat
// dz, dp of Eq.4) are warp-reduced and added with one L2 atomic per value per warp.
template <int TILE>
__global__ void __launch_bounds__(TILE* TILE) k_render_bwd(
    DevCam cam, DevOpt opt, int tiles_x, const uint2* __restrict__ ranges, const uint32_t* __restrict__ ids,
    const Record* __restrict__ rec, const float* __restrict__ T_final, const int32_t* __restrict__ n_contrib,
    const int32_t* __restrict__ median_pos, const float* __restrict__ dL_dcolor, const float* __restrict__ dL_ddepth,
    const float* __restrict__ dL_dnormal, const float* __restrict__ dL_dalpha, float* __restrict__ g2d,
    Counter* __restrict__ counters) {
  constexpr int BLOCK = TILE * TILE;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * TILE + (int)(threadIdx.x % TILE), py = ty * TILE + (int)(threadIdx.x / TILE);
  const bool inside = px < cam.W && py < cam.H;
  const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
  const uint2 range = ranges[tile];
  const int HW = cam.W * cam.H;
  const int pix = py * cam.W + px;
  const int lane = (int)(threadIdx.x & 31);

  __shared__ float4 s0[BLOCK], s1[BLOCK], s2[BLOCK];
  __shared__ float2 s3[BLOCK];  // (p0, p1) for the median-depth gradient
  __shared__ uint32_t sid[BLOCK];
  __shared__ int s_maxlast;

  int last = 0, med = -1;
  float T = 1.f;
  float gC0 = 0.f, gC1 = 0.f, gC2 = 0.f, gN0 = 0.f, gN1 = 0.f, gN2 = 0.f, gD = 0.f, gA = 0.f;
  if (inside) {
    last = n_contrib[pix];
    med = median_pos[pix];
    T = T_final[pix];
    if (dL_dcolor) { gC0 = dL_dcolor[pix]; gC1 = dL_dcolor[HW + pix]; gC2 = dL_dcolor[2 * HW + pix]; }
    if (dL_dnormal) { gN0 = dL_dnormal[pix]; gN1 = dL_dnormal[HW + pix]; gN2 = dL_dnormal[2 * HW + pix]; }
    if (dL_ddepth) gD = dL_ddepth[pix];
    if (dL_dalpha) gA = dL_dalpha[pix];
  }
  if (counters) warp_count(counters + 2, (unsigned)last);
  if (threadIdx.x == 0) s_maxlast = 0;
  __syncthreads();
  if (last > 0) atomicMax(&s_maxlast, last);
  __syncthreads();
  const int maxlast = s_maxlast;

  const float TFa = T * (gA - (opt.bg[0] * gC0 + opt.bg[1] * gC1 + opt.bg[2] * gC2));
  float Dsuf = 0.f;

  for (int end = maxlast; end > 0; end -= BLOCK) {
    const int start = max(0, end - BLOCK);
    const int cnt = end - start;
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      const uint32_t id = ids[range.x + start + threadIdx.x];
      const Record* r = rec + id;
      sid[threadIdx.x] = id;
      s0[threadIdx.x] = r->r0;
      s1[threadIdx.x] = r->r1;
      s2[threadIdx.x] = r->r2;
      const float4 r3 = r->r3;
      s3[threadIdx.x] = make_float2(r3.y, r3.z);
    }
    __syncthreads();
    for (int j = cnt - 1; j >= 0; --j) {
      const int pos = start + j;
      const float4 a0 = s0[j], a1 = s1[j];
      float g[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) g[k] = 0.f;
      bool active = pos < last;
      if (active) {
        const PairAlpha pa = eval_alpha(a0, a1.x, a1.y, fpx, fpy, opt.alpha_max);
        if (pa.alpha < opt.alpha_min) {
          active = false;
        } else {
          const float4 a2 = s2[j];
          const float rinv = __fdividef(1.f, 1.f - pa.alpha);  // α ≤ α_max < 1
          T = T * rinv;  // T_i = T_{i+1} / (1 − α_i)
          const float w = pa.alpha * T;
          const float dot = a1.z * gC0 + a1.w * gC1 + a2.x * gC2 + a2.y * gN0 + a2.z * gN1 + a2.w * gN2;
          const float dL_dal = T * dot - rinv * (Dsuf - TFa);
          Dsuf = fmaf(w, dot, Dsuf);
          g[6] = w * gC0; g[7] = w * gC1; g[8] = w * gC2;
          g[9] = w * gN0; g[10] = w * gN1; g[11] = w * gN2;
          if (pa.a_raw <= opt.alpha_max) {  // α not clamped (S8)
            g[5] = pa.G * dL_dal;
            const float dpw = a1.y * g[5] * kLn2;  // dL/d(power in log2 units)
            const float hx = dpw * pa.dx, hy = dpw * pa.dy;
            g[0] = 2.f * a0.z * hx + a0.w * hy;
            g[1] = a0.w * hx + 2.f * a1.x * hy;
            g[2] = hx * pa.dx;
            g[3] = hx * pa.dy;
            g[4] = hy * pa.dy;
          }
          if (pos == med) {  // median depth D = z_c + p·Δ (Eq.4)
            const float2 p = s3[j];
            g[0] += gD * p.x;
            g[1] += gD * p.y;
            g[12] = gD;
            g[13] = gD * pa.dx;
            g[14] = gD * pa.dy;
          }
        }
      }
      const unsigned act = __ballot_sync(0xffffffffu, active);
      if (act) {
        float* dst = g2d + (size_t)sid[j] * kG2D;
        if (__popc(act) == 1) {  // one contributing pixel in this warp: no reduction needed
          if (active) {
#pragma unroll
            for (int k = 0; k < 15; ++k) atomicAdd(dst + k, g[k]);
          }
        } else {
          const float v = reduce_scatter16(g, lane);
          const int k = lane >> 1;
          if ((lane & 1) == 0 && k < 15) atomicAdd(dst + k, v);
        }
      }
    }
  }
}

}  // namespace

void launch_render_fwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, float* color, float* depth, float* normal, float* alpha,
                       float* T_final, int32_t* n_contrib, int32_t* median_pos, Counter* counters, cudaStream_t s) {
  const unsigned grid = (unsigned)(tiles_x * tiles_y);
  if (opt.tile == 16)
    k_render_fwd<16><<<grid, 256, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, color, depth, normal, alpha, T_final,
                                          n_contrib, median_pos, counters);
  else
    k_render_fwd<8><<<grid, 64, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, color, depth, normal, alpha, T_final,
                                        n_contrib, median_pos, counters);
}

void launch_render_bwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, const float* T_final, const int32_t* n_contrib,
                       const int32_t* median_pos, const float* dL_dcolor, const float* dL_ddepth,
                       const float* dL_dnormal, const float* dL_dalpha, float* g2d, Counter* counters,
                       cudaStream_t s) {
  const unsigned grid = (unsigned)(tiles_x * tiles_y);
  if (opt.tile == 16)
    k_render_bwd<16><<<grid, 256, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, T_final, n_contrib, median_pos,
                                          dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, g2d, counters);
  else
    k_render_bwd<8><<<grid, 64, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, T_final, n_contrib, median_pos,
                                        dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, g2d, counters);
}

}  // namespace rade
