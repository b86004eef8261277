// render.cu — stage 3 (K3, blend forward) and the first half of stage 4 (K4, blend
// backward) of the RaDe-GS rasterizer, sm_100a.
//
// One CTA per TILE×TILE tile, TILE²/2 threads, each owning two pixels of the same column;
// each warp owns an 8×8 pixel quadrant (lane l: column l % 8, rows l / 8 and l / 8 + 4), so
// at the default 8×8 tiles a CTA is one warp (pixels sampled at (i+½, j+½), reading S4).
// Each CTA walks its tile's depth-sorted list (ranges from K2) in batches of TILE² splats
// staged in shared memory (one coalesced 64-B record gather per splat); every shared-memory
// broadcast, loop step and — in K4 — every warp reduction then serves two pixels per thread.
// The block leaves as soon as every pixel is saturated (__syncthreads_count). The CTAs are
// launched longest tile list first (k_tile_order, computed before K3 and reused by K4).
//
// Per (pixel, splat), front to back (Eq.3; readings S1, S8, S9, S10):
//   α = min(α_max, o·exp(−½ Δᵀ conic Δ)), Δ = (u_c − u, v_c − v)  (skip if α < α_min)
//   T′ = T(1 − α); stop before blending if T′ < T_min
//   w = α T; C += w c; N += w n
//   first splat with T > median_T ≥ T′: D = z_c + p·Δ        (Eq.4)
// Epilogue: C += T·bg, A = 1 − T; per pixel state (T_final, n_contrib, median_pos) for K4.
//
// K4 replays each pixel's list backwards from n_contrib, reconstructing T_i = T_{i+1}/(1−α_i)
// and one scalar suffix sum, and produces the 12 per-splat sums of the 2-D gradients, which
// are summed over the thread's two pixels and then warp-reduced (through shared memory)
// before one L2 atomic per value per (warp, splat). At 8×8 tiles K3 leaves a per-tile bit
// mask of the list positions some pixel blends; K4 stages and visits only those.
#include "rade_internal.cuh"

namespace rade {
namespace {

// Splats staged per batch: TILE² (one per pixel), capped at 256 for 32×32 tiles so the
// staged records, warp lists and reduction rows fit the 48-KB static shared memory.
__host__ __device__ constexpr int batch_of(int tile) { return tile * tile < 256 ? tile * tile : 256; }

struct PixF {  // forward state of one pixel
  float px, py;
  float T, C0, C1, C2, N0, N1, N2, D;
  float d0, D1, D2;  // depth distortion (S21): Σω(d − d0), Σω(d − d0)², d0 = first blended depth
  int last, med;
  unsigned n_eval, n_blend;
};
// Pins a loop-invariant value in a register (ptxas otherwise rematerialises it every
// iteration, e.g. (float)px + 0.5 or a constant-bank load).
__device__ __forceinline__ float opaque(float x) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Blackwell packed FP32 (FFMA2 / FADD2 / FMUL2): a thread's two pixels — rows A and B of one
// column — as the lo / hi halves of a 64-bit register pair, so their per-pair arithmetic is one
// instruction per operation instead of two (each half is rounded exactly as the scalar IEEE op:
// the decisions stay bit-identical to the scalar code and to K4). A scalar operand of a packed
// op is broadcast by ptxas (`R.F32` operand), so bc() costs nothing.
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2 bc(float x) { return pk(x, x); }
__device__ __forceinline__ float lo_of(f2 v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float hi_of(f2 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ float2 lds64f(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

// A saturated (or outside) pixel is marked by py = +inf: pair_power then yields e = −inf or
// NaN, whose α test fails, so the blend loop needs no separate "done" test per pair.
__device__ __forceinline__ bool pix_done(const PixF& s) { return s.py == __int_as_float(0x7f800000); }

__device__ __forceinline__ void pixf_init(PixF& s, float px, float py, bool inside) {
  s.px = px;
  s.py = py;
  s.T = 1.f;
  s.C0 = s.C1 = s.C2 = s.N0 = s.N1 = s.N2 = s.D = 0.f;
  s.d0 = s.D1 = s.D2 = 0.f;
  s.last = 0;
  s.med = -1;
  s.n_eval = s.n_blend = 0;
  if (!inside) s.py = __int_as_float(0x7f800000);
}

// The blend part of one (pixel, splat) step of Eq.3 (pair_power established α ≥ α_min, S8)
// with the median-depth selection of reading S9, and with DIST the depth-distortion sums of
// reading S21 (centred on the first blended depth d0, so L_d = 2(A·D2 − D1²) loses no digits
// to cancellation: it is shift invariant). a3 = the record's r3 (z_c, p0, p1, ·) when DIST,
// else read from shared memory (a3addr) only at the median splat.
template <bool PROF, bool DIST>
__device__ __forceinline__ void fwd_blend(PixF& s, const PairAlpha& pa, const float4& a1, const float4& a2,
                                          const float4& a3in, unsigned a3addr, int pos, const DevOpt& opt) {
  const float alpha = fminf(opt.alpha_max, ex2_approx(pa.e));
  const float Tn = __fmul_rn(s.T, __fsub_rn(1.f, alpha));
  if (Tn < opt.T_min) {  // stop before blending this splat (S8)
    s.py = __int_as_float(0x7f800000);  // done
    return;
  }
  const float w = __fmul_rn(alpha, s.T);
  s.C0 = __fmaf_rn(w, a1.z, s.C0);
  s.C1 = __fmaf_rn(w, a1.w, s.C1);
  s.C2 = __fmaf_rn(w, a2.x, s.C2);
  s.N0 = __fmaf_rn(w, a2.y, s.N0);
  s.N1 = __fmaf_rn(w, a2.z, s.N1);
  s.N2 = __fmaf_rn(w, a2.w, s.N2);
  if (s.T > opt.median_T && Tn <= opt.median_T) {
    const float4 a3 = DIST ? a3in : lds128(a3addr);  // (z_c, p0, p1, ·)
    s.D = __fmaf_rn(a3.y, pa.dx, __fmaf_rn(a3.z, pa.dy, a3.x));
    s.med = pos;
  }
  if (DIST) {  // d of Eq.15 for this splat (the median channel's depth)
    const float d = __fmaf_rn(a3in.y, pa.dx, __fmaf_rn(a3in.z, pa.dy, a3in.x));
    if (s.last == 0) s.d0 = d;
    const float e = d - s.d0;
    s.D1 = fmaf(w, e, s.D1);
    s.D2 = fmaf(w * e, e, s.D2);
  }
  s.T = Tn;
  s.last = pos + 1;
  if (PROF) ++s.n_blend;
}

template <bool DIST>
__device__ __forceinline__ void fwd_store(const PixF& s, bool inside, int pix, int HW, const DevOpt& opt,
                                          float* __restrict__ color, float* __restrict__ depth,
                                          float* __restrict__ normal, float* __restrict__ alpha_out,
                                          float* __restrict__ T_final, int32_t* __restrict__ n_contrib,
                                          int32_t* __restrict__ median_pos, const DistIO& dio) {
  if (!inside) return;
  if (DIST) {  // L_d = Σ_ij ω_i ω_j (d_i − d_j)² = 2(A·D2 − D1²), A = Σω = 1 − T
    const float A = 1.f - s.T;
    if (dio.dist) dio.dist[pix] = fmaxf(2.f * fmaf(A, s.D2, -s.D1 * s.D1), 0.f);
    dio.d0[pix] = s.d0;
    dio.D1[pix] = s.D1;
  }
  if (color) {
    color[pix] = __fmaf_rn(s.T, opt.bg[0], s.C0);
    color[HW + pix] = __fmaf_rn(s.T, opt.bg[1], s.C1);
    color[2 * HW + pix] = __fmaf_rn(s.T, opt.bg[2], s.C2);
  }
  if (normal) {
    normal[pix] = s.N0;
    normal[HW + pix] = s.N1;
    normal[2 * HW + pix] = s.N2;
  }
  if (depth) depth[pix] = s.D;
  if (alpha_out) alpha_out[pix] = 1.f - s.T;
  T_final[pix] = s.T;
  n_contrib[pix] = s.last;
  median_pos[pix] = s.med;
}

// Can the splat reach α ≥ α_min at a pixel centre of [x0, x1] × [y0, y1]? It does where
// q(Δ) = t1² + t2² ≤ K = log2 o − log2 α_min (t1 = g11 dx + g21 dy, t2 = g22 dy, Δ = centre −
// pixel), so the exact test is min over the Δ-box of the convex q ≤ K. Its unconstrained
// minimiser is Δ = 0; if that lies outside the box the minimum lies on a face whose side
// excludes 0 (at most one per axis), where q is a 1-D quadratic minimised in closed form
// and clamped to the face. Accepting with a 1e-5 relative margin keeps the test
// conservative against pair_power's fp32 roundings (it never drops a pair pair_power
// would accept).
__device__ __forceinline__ bool splat_reaches(const float4& r0, const float4& r1, float2 c, float x0, float x1,
                                              float y0, float y1, float log2_alpha_min) {
  const float K = r1.y - log2_alpha_min;
  if (!(K > 0.f)) return false;
  const float g11 = r0.z, g21 = r0.w, g22 = r1.x;
  const float dxa = c.x - x1, dxb = c.x - x0, dya = c.y - y1, dyb = c.y - y0;  // Δ-box
  const bool in_x = dxa <= 0.f && dxb >= 0.f, in_y = dya <= 0.f && dyb >= 0.f;
  if (in_x && in_y) return true;
  float qmin = 3.4e38f;
  if (!in_x) {  // face dx = cx, dy ∈ [dya, dyb]
    const float cx = dxa > 0.f ? dxa : dxb;
    const float a = fmaf(g21, g21, g22 * g22);
    const float dy = fminf(fmaxf(-g11 * g21 * cx / a, dya), dyb);
    const float t1 = fmaf(g11, cx, g21 * dy), t2 = g22 * dy;
    qmin = fminf(qmin, fmaf(t1, t1, t2 * t2));
  }
  if (!in_y) {  // face dy = cy, dx ∈ [dxa, dxb]
    const float cy = dya > 0.f ? dya : dyb;
    const float dx = fminf(fmaxf(-g21 * cy / g11, dxa), dxb);
    const float t1 = fmaf(g11, dx, g21 * cy), t2 = g22 * cy;
    qmin = fminf(qmin, fmaf(t1, t1, t2 * t2));
  }
  return qmin <= K * 1.00001f + 1e-5f;
}

// Per-warp filter of a staged batch: the indices k < cnt (in order) of the splats that can
// reach the warp's pixel rectangle, written to wl; returns their number. Lane-parallel (32
// splats per pass), so a warp then steps only through splats that touch its pixels.
__device__ __forceinline__ int warp_filter(const float4* s0, const float4* s1, const float4* s3, int cnt, int lane,
                                           float x0, float x1, float y0, float y1, float log2_alpha_min,
                                           uint16_t* wl) {
  int nsel = 0;
  for (int k0 = 0; k0 < cnt; k0 += 32) {
    const int k = k0 + lane;
    bool ok = false;
    if (k < cnt) {
      const float4 r0 = s0[k], r1 = s1[k];
      const float2 lo = uv_lo(s3[k].w);
      ok = splat_reaches(r0, r1, make_float2(r0.x + lo.x, r0.y + lo.y), x0, x1, y0, y1, log2_alpha_min);
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (ok) wl[nsel + __popc(m & ((1u << lane) - 1u))] = (uint16_t)k;
    nsel += __popc(m);
  }
  __syncwarp();
  return nsel;
}

// Blend mask (TILE 8, K3 → K4): bit p of tile t says that some pixel of the tile passes the α
// test at list position p while still blending (K4's active set is a subset of it: a pixel is
// active at p iff p < n_contrib and α ≥ α_min, decided bit-identically by both kernels). Tile
// t's words start at (range.x >> 5) + t, which is past the previous tile's last word
// ((y >> 5) − (x >> 5) ≥ ⌊(y − x)/32⌋), so K3 writes whole words with plain stores, two per
// staged batch of 64: word(p) = (range.x >> 5) + t + p / 32, bit p % 32. Batches past K3's
// early exit are never read (K4 stops at max n_contrib ≤ K3's last position + 1).
__device__ __forceinline__ unsigned blend_mask_word(unsigned rx, int pos, int tile) {
  return (rx >> 5) + (unsigned)tile + ((unsigned)pos >> 5);
}

// Launch order of the tiles for K3/K4: longest lists first (log2 buckets), so the heavy tiles
// — clustered where the scene is — do not start last and leave a tail. One block; the order
// within a bucket is arbitrary (a tile's outputs do not depend on when it runs).
#ifndef RD_ORDER_SUB
#define RD_ORDER_SUB 2  // buckets of 2^-SUB octave of list length (the SUB bits below the leading one)
#endif
constexpr int kNB = 32 << RD_ORDER_SUB;  // buckets (bucket 0 = the longest lists)
__device__ __forceinline__ int tile_bucket(uint32_t len) {
  const int lg = len ? 31 - __clz((int)len) : -1;  // floor(log2 len)
  const int sub = lg >= RD_ORDER_SUB ? (int)((len >> (lg - RD_ORDER_SUB)) & ((1u << RD_ORDER_SUB) - 1u))
                                     : (lg > 0 ? (int)((len << (RD_ORDER_SUB - lg)) & ((1u << RD_ORDER_SUB) - 1u)) : 0);
  return (kNB - 1) - min(kNB - 1, ((lg + 1) << RD_ORDER_SUB) + sub);
}
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int n_tiles,
                                                     uint32_t* __restrict__ order) {
  __shared__ uint32_t cnt[kNB], off[kNB];
  if (threadIdx.x < kNB) cnt[threadIdx.x] = 0u;
  const unsigned lane = threadIdx.x & 31u, below = (1u << lane) - 1u;
  // thread t owns tiles t, t + 1024, ...: their buckets are computed once, up to kPer of them
  // with all range loads in flight together (one block: the kernel is a chain of dependent
  // rounds, so the loads must not be one round trip per round)
  constexpr int kPer = 16;  // 16 × 1024 tiles (C3 at 8×8: 15 965; more: further chunks)
  const int rounds = (n_tiles + (int)blockDim.x - 1) / (int)blockDim.x;
  __syncthreads();
  for (int r0 = 0; r0 < rounds; r0 += kPer) {
    uint2 rg[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = (r0 + k) * (int)blockDim.x + (int)threadIdx.x;
      rg[k] = (r0 + k < rounds && t < n_tiles) ? ranges[t] : make_uint2(0u, 0u);
    }
    // most tiles share a few buckets: one shared atomic per (warp, bucket) group (__match_any)
    // instead of one per tile, which would serialise thousands of updates of one address
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = (r0 + k) * (int)blockDim.x + (int)threadIdx.x;
      if (r0 + k >= rounds) break;  // block-uniform
      const int b = t < n_tiles ? tile_bucket(rg[k].y - rg[k].x) : kNB;  // longer → smaller
#ifndef RD_ORDER_ATOMIC
#define RD_ORDER_ATOMIC 1  // one plain shared atomic per tile (0: __match_any grouping; with 128 buckets
                           // the contention is low and the plain atomics are cheaper)
#endif
      if (RD_ORDER_ATOMIC) {
        if (b < kNB) atomicAdd(&cnt[b], 1u);
        continue;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      if (b < kNB && (peers & below) == 0u) atomicAdd(&cnt[b], (unsigned)__popc(peers));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0u;
    for (int b = 0; b < kNB; ++b) {
      off[b] = a;
      a += cnt[b];
    }
  }
  __syncthreads();
  for (int r0 = 0; r0 < rounds; r0 += kPer) {
    uint2 rg[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = (r0 + k) * (int)blockDim.x + (int)threadIdx.x;
      rg[k] = (r0 + k < rounds && t < n_tiles) ? ranges[t] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int t = (r0 + k) * (int)blockDim.x + (int)threadIdx.x;
      if (r0 + k >= rounds) break;
      const int b = t < n_tiles ? tile_bucket(rg[k].y - rg[k].x) : kNB;
      if (RD_ORDER_ATOMIC) {
        if (b < kNB) order[atomicAdd(&off[b], 1u)] = (uint32_t)t;
        continue;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0u;
      if (b < kNB && (int)lane == leader) base = atomicAdd(&off[b], (unsigned)__popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (b < kNB) order[base + (uint32_t)__popc(peers & below)] = (uint32_t)t;
    }
  }
}

// K3: one CTA per TILE×TILE tile, TILE²/2 threads; warp w owns the 8×8 quadrant w of the
// tile (lane l: column l % 8, rows l / 8 and l / 8 + 4). Per staged batch each warp first
// filters the batch down to the splats that reach its quadrant, then blends those.
template <int TILE, bool PROF, bool DIST>
__global__ void __launch_bounds__(TILE* TILE / 2) k_render_fwd(DevCam cam, DevOpt opt, int tiles_x,
                                                                const uint2* __restrict__ ranges,
                                                                const uint32_t* __restrict__ ids,
                                                                const Record* __restrict__ rec,
                                                                float* __restrict__ color, float* __restrict__ depth,
                                                                float* __restrict__ normal,
                                                                float* __restrict__ alpha_out,
                                                                float* __restrict__ T_final,
                                                                int32_t* __restrict__ n_contrib,
                                                                int32_t* __restrict__ median_pos,
                                                                DistIO dio, uint32_t* __restrict__ bmask,
                                                                const uint32_t* __restrict__ order,
                                                                Counter* __restrict__ counters, DevBounds bd) {
  constexpr int NT = TILE * TILE / 2;  // threads
  constexpr int NW = NT / 32;          // warps = 8×8 quadrants
  constexpr int BATCH = batch_of(TILE);  // splats staged per round
#ifndef RD_K3_FILTER8
#define RD_K3_FILTER8 0
#endif
  constexpr bool kFilter = TILE > 8 || RD_K3_FILTER8;
  constexpr bool kMask = TILE == 8;    // one warp per tile: it records the blend mask for K4
  const int tile = (int)order[blockIdx.x];
  RD_CHECK(tile >= 0 && tile < bd.n_tiles);
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  const int qx = tx * TILE + (warp % (TILE / 8)) * 8, qy = ty * TILE + (warp / (TILE / 8)) * 8;
  const int px = qx + lane % 8, pyA = qy + lane / 8, pyB = pyA + 4;
  const bool inA = px < cam.W && pyA < cam.H, inB = px < cam.W && pyB < cam.H;
  const float fx0 = (float)qx + 0.5f, fy0 = (float)qy + 0.5f;  // pixel-centre rectangle of the quadrant
  const uint2 range = ranges[tile];
  const int total = (int)(range.y - range.x);
  RD_CHECK(range.x <= range.y && (int64_t)range.y <= bd.m);

  __shared__ float4 sbuf[4][BATCH];  // record quarters r0..r3 of the batch
  __shared__ uint16_t wlist[kFilter ? NW : 1][kFilter ? BATCH : 1];
  float4* s0 = sbuf[0];
  float4* s1 = sbuf[1];
  float4* s2 = sbuf[2];
  float4* s3 = sbuf[3];

  PixF A, B;
  pixf_init(A, (float)px + 0.5f, (float)pyA + 0.5f, inA);
  pixf_init(B, (float)px + 0.5f, (float)pyB + 0.5f, inB);
#ifndef RD_K3_PACKED
#define RD_K3_PACKED 1
#endif
  constexpr bool kPacked = RD_K3_PACKED != 0;
  const float kInf = __int_as_float(0x7f800000);
  // packed state (rows A | B): −py (−inf once the pixel is done), T, colour, normal, and with
  // DIST the distortion sums; the scalar PixF keeps px, D, last, med and the counters
  f2 NPY = pk(-A.py, -B.py), T2 = bc(1.f), C0 = bc(0.f), C1 = C0, C2 = C0, N0 = C0, N1 = C0, N2 = C0;
  f2 DD0 = C0, DD1 = C0, DD2 = C0;
  unsigned steps = 0;  // PROF: this warp's splat steps (E_issued)
  auto done_A = [&]() { return kPacked ? lo_of(NPY) == -kInf : pix_done(A); };
  auto done_B = [&]() { return kPacked ? hi_of(NPY) == -kInf : pix_done(B); };
  for (int base = 0; base < total; base += BATCH) {
    if (__syncthreads_count(done_A() && done_B()) == NT) break;
#pragma unroll
    for (int h = 0; h < (BATCH + NT - 1) / NT; ++h) {
      const int t = (int)threadIdx.x + h * NT;
      const int k = base + t;
      if (t < BATCH && k < total) {
        RD_CHECK((int64_t)ids[range.x + k] < bd.n);
        const Record* r = rec + ids[range.x + k];
        s0[t] = r->r0;
        s1[t] = r->r1;
        s2[t] = r->r2;
        s3[t] = r->r3;
      }
    }
    __syncthreads();
    if (__all_sync(0xffffffffu, done_A() && done_B())) continue;  // this warp is saturated
    const int cnt = min(BATCH, total - base);
    // 8×8 tiles: the binning rect is already tight, filtering costs more than it saves
    const int nsel = kFilter ? warp_filter(s0, s1, s3, cnt, lane, fx0, fx0 + 7.f, fy0, fy0 + 7.f,
                                           opt.log2_alpha_min, wlist[warp])
                             : cnt;
    const unsigned a_s0 = smem_addr(s0);  // s0..s3 are contiguous
    const float cpx = opaque(A.px);
    const float la_min = __shfl_sync(0xffffffffu, opt.log2_alpha_min, 0);  // a register, not a per-step LDC
    unsigned mine = 0u;  // kMask: bit 0 / 1 = this batch's step lane / lane + 32 was blended
    for (int i = 0; i < nsel; ++i) {  // the warp stays converged: uniform exits and skips only
      if (PROF) ++steps;
      const int j = kFilter ? (int)wlist[warp][i] : i;
      const unsigned a = a_s0 + 16u * j;
      const float4 a0 = lds128(a), a1 = lds128(a + 16u * BATCH);
      const float2 ulo = uv_lo(__uint_as_float(lds32(a + 48u * BATCH + 12u)));  // r3.w
      const PairColumn col = pair_column(a0, ulo, cpx);  // A and B share the column
      if constexpr (kPacked) {
        // pair_power for both rows at once: dy = (v_hi − py) + v_lo, t1 = g21 dy + g11 dx,
        // t2 = g22 dy, e = log2 o − (t1² + t2²) — the same IEEE ops, per half
        const f2 DY = add2(add2(bc(a0.y), NPY), bc(ulo.y));
        const f2 T1 = fma2(bc(a0.w), DY, bc(col.g11dx));
        const f2 T2s = mul2(bc(a1.x), DY);
        const f2 E = fma2(fma2(T1, T1, mul2(T2s, T2s)), bc(-1.f), bc(a1.y));
        const float eA = lo_of(E), eB = hi_of(E);
        if (PROF) {
          A.n_eval += done_A() ? 0u : 1u;
          B.n_eval += done_B() ? 0u : 1u;
        }
        const bool okA = eA >= la_min, okB = eB >= la_min;  // α ≥ α_min (S8); false when done
        if (!__any_sync(0xffffffffu, okA || okB)) continue;  // no pixel of the warp blends it
        if (kMask && (j & 31) == lane) mine |= 1u + (unsigned)(j >> 5);
        const float4 a2 = lds128(a + 32u * BATCH);
        // both rows branch-free: an inactive row gets α = 0 (T, colour, normal unchanged exactly)
        const float alA = okA ? fminf(opt.alpha_max, ex2_approx(eA)) : 0.f;
        const float alB = okB ? fminf(opt.alpha_max, ex2_approx(eB)) : 0.f;
        const f2 TN = mul2(T2, fma2(pk(alA, alB), bc(-1.f), bc(1.f)));  // T·(1 − α)
        const float TnA = lo_of(TN), TnB = hi_of(TN), TA = lo_of(T2), TB = hi_of(T2);
        const bool stA = okA && TnA < opt.T_min, stB = okB && TnB < opt.T_min;  // stop before it (S8)
        const bool bA = okA && !stA, bB = okB && !stB;
        const f2 W = mul2(pk(bA ? alA : 0.f, bB ? alB : 0.f), T2);  // w = α T
        C0 = fma2(W, bc(a1.z), C0);
        C1 = fma2(W, bc(a1.w), C1);
        C2 = fma2(W, bc(a2.x), C2);
        N0 = fma2(W, bc(a2.y), N0);
        N1 = fma2(W, bc(a2.z), N1);
        N2 = fma2(W, bc(a2.w), N2);
        const int pos = base + j;
        const bool mA = bA && TA > opt.median_T && TnA <= opt.median_T;  // the median splat (S9)
        const bool mB = bB && TB > opt.median_T && TnB <= opt.median_T;
#ifndef RD_K3_MEDBR
// 0: the median-depth candidates of every blending step computed branch-free (one basic block:
// ptxas then keeps the packed accumulators in place instead of copying them on the back edge;
// −20% instructions on the blending path, K3 0.263 → 0.2555 ms); 1: behind a warp vote
#define RD_K3_MEDBR 0
#endif
        if (DIST || !RD_K3_MEDBR || __any_sync(0xffffffffu, mA || mB)) {
          const float4 a3 = lds128(a + 48u * BATCH);  // (z_c, p0, p1, ·)
          const float dA = __fmaf_rn(a3.y, col.dx, __fmaf_rn(a3.z, lo_of(DY), a3.x));
          const float dB = __fmaf_rn(a3.y, col.dx, __fmaf_rn(a3.z, hi_of(DY), a3.x));
          if (mA) { A.D = dA; A.med = pos; }
          if (mB) { B.D = dB; B.med = pos; }
          if (DIST) {  // Σω(d − d0), Σω(d − d0)², d0 = the first blended depth (S21)
            DD0 = pk(bA && A.last == 0 ? dA : lo_of(DD0), bB && B.last == 0 ? dB : hi_of(DD0));
            const f2 Ed = pk(bA ? dA - lo_of(DD0) : 0.f, bB ? dB - hi_of(DD0) : 0.f);
            DD1 = fma2(W, Ed, DD1);
            DD2 = fma2(mul2(W, Ed), Ed, DD2);
          }
        }
        T2 = pk(bA ? TnA : TA, bB ? TnB : TB);
        NPY = pk(stA ? -kInf : lo_of(NPY), stB ? -kInf : hi_of(NPY));
        if (bA) A.last = pos + 1;
        if (bB) B.last = pos + 1;
        if (PROF) {
          A.n_blend += bA ? 1u : 0u;
          B.n_blend += bB ? 1u : 0u;
        }
        // a pixel can only saturate in a step that blends: test for the whole warp only then
        if (__all_sync(0xffffffffu, done_A() && done_B())) break;
        continue;
      }
      const PairAlpha pA = pair_power(a0, a1.x, a1.y, ulo, col, A.py, la_min);
      const PairAlpha pB = pair_power(a0, a1.x, a1.y, ulo, col, B.py, la_min);
      if (PROF) {
        A.n_eval += pix_done(A) ? 0u : 1u;
        B.n_eval += pix_done(B) ? 0u : 1u;
      }
      const bool okA = pA.pass, okB = pB.pass;  // α ≥ α_min (S8); false for saturated pixels
      if (!__any_sync(0xffffffffu, okA || okB)) continue;  // no pixel of the warp blends it
      if (kMask && (j & 31) == lane) mine |= 1u + (unsigned)(j >> 5);  // some pixel blends (or stops at) base + j
      const float4 a2 = lds128(a + 32u * BATCH);
      const float4 a3 = DIST ? lds128(a + 48u * BATCH) : a2;
      if (okA) fwd_blend<PROF, DIST>(A, pA, a1, a2, a3, a + 48u * BATCH, base + j, opt);
      if (okB) fwd_blend<PROF, DIST>(B, pB, a1, a2, a3, a + 48u * BATCH, base + j, opt);
      // a pixel can only saturate in a step that blends: test for the whole warp only then
      if (__all_sync(0xffffffffu, pix_done(A) && pix_done(B))) break;
    }
    if (kMask) {  // the batch's words (positions past the last step: zero bits); a word past
      const unsigned lo = __ballot_sync(0xffffffffu, mine & 1u);  // the list's end may be the
      const unsigned hi = __ballot_sync(0xffffffffu, mine & 2u);  // next tile's first
      if (lane == 0) {
        RD_CHECK((int64_t)blend_mask_word(range.x, base, tile) + (base + 32 < total ? 1 : 0) < bd.mask_words);
        uint32_t* w = bmask + blend_mask_word(range.x, base, tile);
        w[0] = lo;
        if (base + 32 < total) w[1] = hi;
      }
    }
  }
  if (PROF) {
    warp_count(counters + 0, A.n_eval + B.n_eval);
    warp_count(counters + 1, A.n_blend + B.n_blend);
    if (lane == 0 && steps) atomicAdd(counters + kIssuedCounter, (Counter)steps * 64u);  // 64 pixels per warp
  }
  if constexpr (kPacked) {  // back to the per-pixel records for the store
    A.T = lo_of(T2); B.T = hi_of(T2);
    A.C0 = lo_of(C0); B.C0 = hi_of(C0); A.C1 = lo_of(C1); B.C1 = hi_of(C1); A.C2 = lo_of(C2); B.C2 = hi_of(C2);
    A.N0 = lo_of(N0); B.N0 = hi_of(N0); A.N1 = lo_of(N1); B.N1 = hi_of(N1); A.N2 = lo_of(N2); B.N2 = hi_of(N2);
    A.d0 = lo_of(DD0); B.d0 = hi_of(DD0); A.D1 = lo_of(DD1); B.D1 = hi_of(DD1); A.D2 = lo_of(DD2); B.D2 = hi_of(DD2);
  }
  const int HW = cam.W * cam.H;
  fwd_store<DIST>(A, inA, pyA * cam.W + px, HW, opt, color, depth, normal, alpha_out, T_final, n_contrib,
                  median_pos, dio);
  fwd_store<DIST>(B, inB, pyB * cam.W + px, HW, opt, color, depth, normal, alpha_out, T_final, n_contrib,
                  median_pos, dio);
}

// Warp sum of v[0..NV) through shared memory (NV ≤ 16; red = this warp's [16][36] floats):
// every lane stores its NV values in column `lane` of row k, lane pair (2k, 2k+1) then reads
// row k's two halves as four float4 each, and one xor-1 shuffle completes the sum. Lanes 2k
// and 2k+1 return Σ_lanes v[k]; ≈ NV + 22 instructions against ≈ 5·NV for a shuffle butterfly.
// K4: when at most this many lanes hold contributions for a splat, each adds its own sums with
// atomics instead of the warp reduction (round 1: 1 → 5 K4 −2.5%, 8+: L2 contention; re-tuned
// after the packed reduction made the reduction cheaper: 5 → 4 K4 0.379 → 0.377 ms, 6 slower)
#ifndef RD_K4_DIRECT
#define RD_K4_DIRECT 4
#endif
constexpr int kDirectLanes = RD_K4_DIRECT;
#ifndef RD_REDUCE_PACKED
#define RD_REDUCE_PACKED 1
#endif
constexpr int kRedPitch = 36;  // floats per row: 16-B aligned rows, conflict-free column stores
template <int NV>
__device__ __forceinline__ float smem_reduce(const float (&v)[NV], unsigned red, int lane) {
#pragma unroll
  for (int k = 0; k < NV; ++k)
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(red + 4u * (unsigned)(k * kRedPitch + lane)), "f"(v[k]) : "memory");
  __syncwarp();
  const int k = lane >> 1, q = lane & 1;
  float s = 0.f;
  if (k < NV) {
    const unsigned a = red + 4u * (unsigned)(k * kRedPitch + 16 * q);
    const float4 x0 = lds128(a), x1 = lds128(a + 16u), x2 = lds128(a + 32u), x3 = lds128(a + 48u);
#if RD_REDUCE_PACKED
    // the 16 values as 8 register pairs summed with packed adds: 7 FADD2 + 1 FADD instead of 15
    const f2 t0 = add2(pk(x0.x, x0.y), pk(x0.z, x0.w)), t1 = add2(pk(x1.x, x1.y), pk(x1.z, x1.w));
    const f2 t2 = add2(pk(x2.x, x2.y), pk(x2.z, x2.w)), t3 = add2(pk(x3.x, x3.y), pk(x3.z, x3.w));
    const f2 t = add2(add2(t0, t1), add2(t2, t3));
    s = lo_of(t) + hi_of(t);
#else
    s = ((x0.x + x0.y) + (x0.z + x0.w)) + ((x1.x + x1.y) + (x1.z + x1.w)) +
        (((x2.x + x2.y) + (x2.z + x2.w)) + ((x3.x + x3.y) + (x3.z + x3.w)));
#endif
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  __syncwarp();  // the rows are rewritten by the next splat
  return s;
}

struct PixB {  // backward state of one pixel
  float px, py;
  float T, TFa, Dsuf;
  float gC0, gC1, gC2, gN0, gN1, gN2, gD;
  float gL, d0, D1, A;  // depth distortion (S21): 4·dL/dL_d, K3's d0 and D1, A = Σω
  int last, med;
};

__device__ __forceinline__ void pixb_init(PixB& s, float px, float py, bool inside, int pix, int HW,
                                          const DevOpt& opt, const float* __restrict__ T_final,
                                          const int32_t* __restrict__ n_contrib,
                                          const int32_t* __restrict__ median_pos,
                                          const float* __restrict__ dL_dcolor, const float* __restrict__ dL_ddepth,
                                          const float* __restrict__ dL_dnormal, const float* __restrict__ dL_dalpha,
                                          const DistIO& dio) {
  s.px = px;
  s.py = py;
  s.T = 1.f;
  s.last = 0;
  s.med = -1;
  s.gC0 = s.gC1 = s.gC2 = s.gN0 = s.gN1 = s.gN2 = s.gD = 0.f;
  s.gL = s.d0 = s.D1 = s.A = 0.f;
  float gA = 0.f;
  if (inside) {
    s.last = n_contrib[pix];
    s.med = median_pos[pix];
    s.T = T_final[pix];
    if (dL_dcolor) { s.gC0 = dL_dcolor[pix]; s.gC1 = dL_dcolor[HW + pix]; s.gC2 = dL_dcolor[2 * HW + pix]; }
    if (dL_dnormal) { s.gN0 = dL_dnormal[pix]; s.gN1 = dL_dnormal[HW + pix]; s.gN2 = dL_dnormal[2 * HW + pix]; }
    if (dL_ddepth) s.gD = dL_ddepth[pix];
    if (s.gD == 0.f) s.med = -1;  // no median-depth gradient from this pixel: never a hit
    if (dL_dalpha) gA = dL_dalpha[pix];
    if (dio.dL_ddist) {
      s.gL = 4.f * dio.dL_ddist[pix];
      s.d0 = dio.d0[pix];
      s.D1 = dio.D1[pix];
      s.A = 1.f - s.T;
    }
  }
  // ∂L/∂α_i gets T_final/(1 − α_i)·(g_A − bg·g_C) from A = 1 − T_final and C += T_final·bg
  s.TFa = s.T * (gA - (opt.bg[0] * s.gC0 + opt.bg[1] * s.gC1 + opt.bg[2] * s.gC2));
  s.Dsuf = 0.f;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One (pixel, splat) step of K4: adds this pixel's contribution to the 12 per-splat sums
//   g0 = Σ dA·dx, g1 = Σ dA·dy, g2 = Σ dA·dx², g3 = Σ dA·dx·dy, g4 = Σ dA·dy², g5 = Σ dA,
//   g6..8 = Σ w·g_C, g9..11 = Σ w·g_N        (dA = α_raw·∂L/∂α)
// from which the 2-D gradients follow per splat after the warp reduction (k_render_bwd).
// With the per-pixel scalar D_i = Σ_{j>i} w_j (c_j·g_C + n_j·g_N) (suffix sum, w_j = α_j T_j)
// the α gradient of Eq.3's colour and of the normal map is
//   ∂L/∂α_i = T_i (c_i·g_C + n_i·g_N) − D_i / (1 − α_i) + T_final/(1 − α_i) (g_A − bg·g_C)
// (the 3DGS derivation collapsed to one scalar, since g_C, g_N are per-pixel constants).
// Branch-free: an inactive pair (past the pixel's list, or α < α_min) contributes exact
// zeros (α masked to 0 ⇒ rinv = rcp(1) = 1, w = 0, dA = 0).
template <bool DIST, int NG, bool FIRST>
__device__ __forceinline__ void bwd_accum(PixB& s, float (&g)[NG], const PairAlpha& pa, bool act, const float4& a1,
                                          const float4& a2, const float4& a3, const DevOpt& opt) {
  const float a_raw = ex2_approx(pa.e);                  // o·exp(−½ΔᵀCΔ)
  const float al = act ? fminf(opt.alpha_max, a_raw) : 0.f;
  const float rinv = rcp_approx(1.f - al);               // α ≤ α_max < 1; exact 1 when masked
  s.T = s.T * rinv;                                      // T_i = T_{i+1} / (1 − α_i)
  const float w = al * s.T;
  const float dot = a1.z * s.gC0 + a1.w * s.gC1 + a2.x * s.gC2 + a2.y * s.gN0 + a2.z * s.gN1 + a2.w * s.gN2;
  const float dL_dal = act && a_raw <= opt.alpha_max ? s.T * dot - rinv * (s.Dsuf - s.TFa) : 0.f;  // clamp (S8)
  s.Dsuf = fmaf(w, dot, s.Dsuf);
  const float dA = a_raw * dL_dal;
  const float hx = dA * pa.dx, hy = dA * pa.dy;
  // FIRST: the first pixel row of the step writes the sums instead of adding to zeros
  auto add = [&](int k, float v) { g[k] = FIRST ? v : g[k] + v; };
  auto fma_ = [&](int k, float a, float b) { g[k] = FIRST ? a * b : fmaf(a, b, g[k]); };
  add(0, hx);
  add(1, hy);
  fma_(2, hx, pa.dx);
  fma_(3, hx, pa.dy);
  fma_(4, hy, pa.dy);
  add(5, dA);
  fma_(6, w, s.gC0);
  fma_(7, w, s.gC1);
  fma_(8, w, s.gC2);
  fma_(9, w, s.gN0);
  fma_(10, w, s.gN1);
  fma_(11, w, s.gN2);
  if constexpr (DIST) {  // ∂L_d/∂d = 4 ω (A (d − d0) − D1), ω detached (S21); into the Eq.15 sums
    const float d = __fmaf_rn(a3.y, pa.dx, __fmaf_rn(a3.z, pa.dy, a3.x));
    const float gd = s.gL * w * fmaf(s.A, d - s.d0, -s.D1);
    add(12, gd);
    fma_(13, gd, pa.dx);
    fma_(14, gd, pa.dy);
  }
}


// K4 with Blackwell packed FP32 (PPT = 2): the thread's two pixels — rows A and B of one column —
// as the halves of 64-bit register pairs (see k_render_fwd). Per step the α evaluation is the
// same IEEE ops per half as pair_power (decisions bit-identical to K3), and the per-splat sums
// use that the two pixels share dx: of the six moment sums only Σ dA, Σ dA·dy, Σ dA·dy² need
// both rows; Σ dA·dx = dx Σ dA, Σ dA·dx² = dx² Σ dA, Σ dA·dx·dy = dx Σ dA·dy (likewise for
// the distortion sums).
#ifndef RD_K4_PACKED
#define RD_K4_PACKED 1
#endif
struct PixB2 {  // backward state of the thread's two pixels (lo = row A, hi = row B)
  f2 NPY, T, TFa, Dsuf, gC0, gC1, gC2, gN0, gN1, gN2;
  f2 gL, d0, D1, A;  // depth distortion (S21)
};
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { return fma2(b, bc(-1.f), a); }

template <bool DIST, int NG>
__device__ __forceinline__ void bwd_accum2(PixB2& s, float (&g)[NG], f2 DY, float dx, float eA, float eB, bool actA,
                                           bool actB, const float4& a1, const float4& a2, const float4& a3,
                                           const DevOpt& opt) {
  const float rA = ex2_approx(eA), rB = ex2_approx(eB);  // α_raw = o·exp(−½ΔᵀCΔ)
  const f2 AL = pk(actA ? fminf(opt.alpha_max, rA) : 0.f, actB ? fminf(opt.alpha_max, rB) : 0.f);
  const f2 OMA = fma2(AL, bc(-1.f), bc(1.f));  // 1 − α (exact 1 when masked)
  const f2 RINV = pk(rcp_approx(lo_of(OMA)), rcp_approx(hi_of(OMA)));
  s.T = mul2(s.T, RINV);  // T_i = T_{i+1} / (1 − α_i)
  const f2 W = mul2(AL, s.T);
  f2 DOT = mul2(bc(a1.z), s.gC0);
  DOT = fma2(bc(a1.w), s.gC1, DOT);
  DOT = fma2(bc(a2.x), s.gC2, DOT);
  DOT = fma2(bc(a2.y), s.gN0, DOT);
  DOT = fma2(bc(a2.z), s.gN1, DOT);
  DOT = fma2(bc(a2.w), s.gN2, DOT);
  // ∂L/∂α = T·dot − (D_suf − T_final·(g_A − bg·g_C))/(1 − α)
  const f2 X = fma2(s.T, DOT, mul2(RINV, sub2(s.TFa, s.Dsuf)));
  s.Dsuf = fma2(W, DOT, s.Dsuf);
  const float dlA = actA && rA <= opt.alpha_max ? lo_of(X) : 0.f;  // clamped α: no gradient (S8)
  const float dlB = actB && rB <= opt.alpha_max ? hi_of(X) : 0.f;
  const f2 DA = mul2(pk(rA, rB), pk(dlA, dlB));  // dA = α_raw·∂L/∂α
  const f2 PY = mul2(DA, DY), PYY = mul2(PY, DY);
  const float S0 = lo_of(DA) + hi_of(DA), S1 = lo_of(PY) + hi_of(PY);
  g[5] = S0;
  g[0] = dx * S0;
  g[2] = dx * g[0];
  g[1] = S1;
  g[3] = dx * S1;
  g[4] = lo_of(PYY) + hi_of(PYY);
  const f2 C0 = mul2(W, s.gC0), C1 = mul2(W, s.gC1), C2 = mul2(W, s.gC2);
  const f2 N0 = mul2(W, s.gN0), N1 = mul2(W, s.gN1), N2 = mul2(W, s.gN2);
  g[6] = lo_of(C0) + hi_of(C0);
  g[7] = lo_of(C1) + hi_of(C1);
  g[8] = lo_of(C2) + hi_of(C2);
  g[9] = lo_of(N0) + hi_of(N0);
  g[10] = lo_of(N1) + hi_of(N1);
  g[11] = lo_of(N2) + hi_of(N2);
  if constexpr (DIST) {  // ∂L_d/∂d = 4 ω (A (d − d0) − D1), ω detached (S21); d of Eq.15 per row
    const f2 D = fma2(bc(a3.y), bc(dx), fma2(bc(a3.z), DY, bc(a3.x)));
    const f2 GD = mul2(mul2(s.gL, W), fma2(s.A, sub2(D, s.d0), mul2(s.D1, bc(-1.f))));
    const f2 GDY = mul2(GD, DY);
    const float S3 = lo_of(GD) + hi_of(GD);
    g[12] = S3;
    g[13] = dx * S3;
    g[14] = lo_of(GDY) + hi_of(GDY);
  }
}

// Median-depth sums Σ g_D, Σ g_D·dx, Σ g_D·dy (G2D f[7..9]) for D = z_c + p·Δ (Eq.4,
// PAPER:443-450): one pixel per splat at most, so added directly (no warp reduction).
__device__ __forceinline__ void bwd_median(const PixB& s, G2D* row, const PairAlpha& pa) {
  atomicAdd(&row->f[7], s.gD);
  atomicAdd(&row->f[8], s.gD * pa.dx);
  atomicAdd(&row->f[9], s.gD * pa.dy);
}

// Sum k of one splat into its G2D row (k < 5: fp64 moments, see rade_internal.cuh).
__device__ __forceinline__ void g2d_add(G2D* row, int k, float v) {
  if (k < 5)
    atomicAdd(&row->m[k], (double)v);
  else
    atomicAdd(&row->f[k - 5], v);
}

// K4: one CTA per tile, TILE²/PPT threads, PPT pixels per thread. Warp w owns an 8-wide,
// 4·PPT-tall pixel rectangle of the tile (lane l: column l % 8, rows l / 8 + 4k, k < PPT).
// The list is walked backwards from the tile's largest n_contrib in batches of TILE² list
// positions. At 8×8 tiles (kMask) only the positions K3's blend mask marks are staged
// (compacted, with their 32-bit positions); at 16×16 each warp filters the staged batch down
// to the splats that can reach its rectangle (warp_filter). Per splat the warp evaluates α
// for its pixels, skips the splat if none uses it (ballot), otherwise accumulates the 12
// sums (15 with L_d) over the thread's PPT pixels, adds the median-depth terms of the pixels
// whose median splat it is (warp-uniform hit test), and either lets up to kDirectLanes
// contributing lanes add their sums with atomics or reduces the sums across the warp
// (smem_reduce) and issues one L2 atomic per value.
#ifndef RD_K4_MINB
// ≤ 73 registers at 8×8 tiles (70 used, no spills): K4 alone is 1.5% slower than at 77, but
// its CTAs leave room for the other views' kernels, and the step runs 0.7% faster
#define RD_K4_MINB 28
#endif
template <int TILE, int PPT, bool DIST>
__global__ void __launch_bounds__(TILE* TILE / PPT, (TILE == 8 ? RD_K4_MINB : 1)) k_render_bwd(
    DevCam cam, DevOpt opt, int tiles_x, const uint2* __restrict__ ranges, const uint32_t* __restrict__ ids,
    const Record* __restrict__ rec, const float* __restrict__ T_final, const int32_t* __restrict__ n_contrib,
    const int32_t* __restrict__ median_pos, const float* __restrict__ dL_dcolor, const float* __restrict__ dL_ddepth,
    const float* __restrict__ dL_dnormal, const float* __restrict__ dL_dalpha, DistIO dio,
    const uint32_t* __restrict__ bmask, const uint32_t* __restrict__ order, G2D* __restrict__ g2d,
    Counter* __restrict__ counters, DevBounds bd) {
  constexpr int NT = TILE * TILE / PPT;
  constexpr int NW = NT / 32;
  constexpr int BATCH = batch_of(TILE);
  constexpr int SH = 4 * PPT;  // each warp: an 8-wide, SH-tall pixel rectangle
  constexpr bool kFilter = TILE > 8;
  constexpr bool kMask = TILE == 8;  // one warp per tile: K3's blend mask selects the splats
  constexpr int NV = DIST ? 15 : 12;  // per-splat sums (G2D order; + Σ gd, Σ gd·dx, Σ gd·dy)
  static_assert(NT % 32 == 0 && TILE % SH == 0, "whole warps tiling the tile");
  static_assert(!kMask || NW == 1, "the blend mask is per tile = per warp");
  const int tile = (int)order[blockIdx.x];
  RD_CHECK(tile >= 0 && tile < bd.n_tiles);
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  const int qx = tx * TILE + (warp % (TILE / 8)) * 8, qy = ty * TILE + (warp / (TILE / 8)) * SH;
  const int px = qx + lane % 8;
  const int py0 = qy + lane / 8;  // pixel k at row py0 + 4k
  const float fx0 = (float)qx + 0.5f, fy0 = (float)qy + 0.5f;
  const uint2 range = ranges[tile];
  const int HW = cam.W * cam.H;
  RD_CHECK(range.x <= range.y && (int64_t)range.y <= bd.m);

  __shared__ float4 sbuf[4][BATCH];  // record quarters r0..r3 of the batch
#ifndef RD_K4_ULO
#define RD_K4_ULO 1
#endif
  // the centre's fp16 remainder (r3.w) as floats, converted once per staged splat (K4 stages
  // only the splats the blend mask selects, so the conversion is cheaper than per step)
  __shared__ float2 sulo[RD_K4_ULO ? BATCH : 1];
  __shared__ uint32_t sid[BATCH];
  __shared__ uint16_t wlist[kFilter ? NW : 1][kFilter ? BATCH : 1];  // per warp: batch slots (kFilter)
  __shared__ int spos[kMask ? BATCH : 1];                            // list position per slot (kMask)
  __shared__ __align__(16) float sred[NW][16 * kRedPitch];
  __shared__ int s_maxlast;

  PixB s[PPT];
  int mylast = 0;
  unsigned evals = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int py = py0 + 4 * k;
    const bool in = px < cam.W && py < cam.H;
    pixb_init(s[k], (float)px + 0.5f, (float)py + 0.5f, in, py * cam.W + px, HW, opt, T_final, n_contrib, median_pos,
              dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha, dio);
    mylast = max(mylast, s[k].last);
    evals += (unsigned)s[k].last;
  }
  if (counters) warp_count(counters + 2, evals);
  if (threadIdx.x == 0) s_maxlast = 0;
  __syncthreads();
  if (mylast > 0) atomicMax(&s_maxlast, mylast);
  __syncthreads();
  const int maxlast = s_maxlast;
  RD_CHECK(maxlast <= (int)(range.y - range.x));
  const unsigned a_red = smem_addr(sred[warp]);
  constexpr bool kPk = PPT == 2 && RD_K4_PACKED != 0;
  const float la_min = __shfl_sync(0xffffffffu, opt.log2_alpha_min, 0);  // a register, not a per-step LDC
  PixB2 P2;  // kPk: the two pixels' state as packed pairs (s[k] keeps last, med, gD, px)
  if constexpr (kPk) {
    const PixB& A = s[0];
    const PixB& B = s[PPT - 1];
    P2.NPY = pk(-A.py, -B.py);
    P2.T = pk(A.T, B.T);
    P2.TFa = pk(A.TFa, B.TFa);
    P2.Dsuf = pk(0.f, 0.f);
    P2.gC0 = pk(A.gC0, B.gC0); P2.gC1 = pk(A.gC1, B.gC1); P2.gC2 = pk(A.gC2, B.gC2);
    P2.gN0 = pk(A.gN0, B.gN0); P2.gN1 = pk(A.gN1, B.gN1); P2.gN2 = pk(A.gN2, B.gN2);
    P2.gL = pk(A.gL, B.gL); P2.d0 = pk(A.d0, B.d0); P2.D1 = pk(A.D1, B.D1); P2.A = pk(A.A, B.A);
  }

  for (int end = maxlast; end > 0; end -= BATCH) {
    const int start = max(0, end - BATCH);
    const int cnt = end - start;
    int nsel = cnt;
    unsigned long long bm = 0ull;
    if (kMask) {  // the batch's 64 mask bits (relative positions 0..cnt-1)
      const unsigned sh = (unsigned)start & 31u;
      RD_CHECK((int64_t)blend_mask_word(range.x, start, tile) + ((unsigned)start % 32u + (unsigned)cnt > 64u ? 2 : 1) <
               bd.mask_words);
      const uint32_t* w = bmask + blend_mask_word(range.x, start, tile);
      const unsigned long long lo = (unsigned long long)w[0] | ((unsigned long long)w[1] << 32);
      bm = lo >> sh;
      if (sh + (unsigned)cnt > 64u) bm |= (unsigned long long)w[2] << (64u - sh);
      if (cnt < 64) bm &= (1ull << cnt) - 1ull;
      nsel = __popcll(bm);
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < (BATCH + NT - 1) / NT; ++h) {
      const int t = (int)threadIdx.x + h * NT;
      if (t >= BATCH) break;
      if (kMask) {  // stage only the splats some pixel of the tile blends, in list order
        if ((bm >> t) & 1ull) {
          const int slot = __popcll(bm & ((1ull << t) - 1ull));
          const uint32_t id = ids[range.x + start + t];
          RD_CHECK(slot < BATCH && (int64_t)id < bd.n);
          const Record* r = rec + id;
          sid[slot] = id;
          spos[slot] = start + t;
          sbuf[0][slot] = r->r0;
          sbuf[1][slot] = r->r1;
          sbuf[2][slot] = r->r2;
          const float4 q3 = r->r3;
          sbuf[3][slot] = q3;
          if (RD_K4_ULO) sulo[slot] = uv_lo(q3.w);
        }
      } else if (t < cnt) {
        const uint32_t id = ids[range.x + start + t];
        RD_CHECK((int64_t)id < bd.n);
        const Record* r = rec + id;
        sid[t] = id;
        sbuf[0][t] = r->r0;
        sbuf[1][t] = r->r1;
        sbuf[2][t] = r->r2;
        const float4 q3 = r->r3;
        sbuf[3][t] = q3;
        if (RD_K4_ULO) sulo[t] = uv_lo(q3.w);
      }
    }
    __syncthreads();
    if (!__any_sync(0xffffffffu, start < mylast)) continue;  // the whole warp is past its pixels' lists
    if (kFilter)
      nsel = warp_filter(sbuf[0], sbuf[1], sbuf[3], cnt, lane, fx0, fx0 + 7.f, fy0, fy0 + (float)(SH - 1),
                         opt.log2_alpha_min, wlist[warp]);
    const unsigned a_s0 = smem_addr(sbuf[0]), a_id = smem_addr(sid), a_pos = smem_addr(spos);
    const unsigned a_ulo = smem_addr(sulo);
    for (int i = nsel - 1; i >= 0; --i) {
      // slot j of the staged batch, at list position pos
      int j, pos;
      if (kMask) {
        j = i;
        pos = (int)lds32(a_pos + 4u * (unsigned)i);
      } else if (kFilter) {
        j = (int)wlist[warp][i];
        pos = start + j;
      } else {
        j = i;
        pos = start + j;
      }
      // the whole warp is past its pixels' lists (never at 8×8 tiles: the warp is the tile, and
      // the walk starts at the tile's largest n_contrib)
      if (!kMask && !__any_sync(0xffffffffu, pos < mylast)) continue;
      const unsigned a = a_s0 + 16u * j;
      const float4 a0 = lds128(a), a1 = lds128(a + 16u * BATCH);
      const float2 ulo = RD_K4_ULO ? lds64f(a_ulo + 8u * j) : uv_lo(__uint_as_float(lds32(a + 48u * BATCH + 12u)));
      const PairColumn col = pair_column(a0, ulo, s[0].px);  // the thread's pixels share the column
      if constexpr (kPk) {
        // pair_power for both rows at once (the same IEEE ops per half)
        const f2 DY = add2(add2(bc(a0.y), P2.NPY), bc(ulo.y));
        const f2 T1 = fma2(bc(a0.w), DY, bc(col.g11dx));
        const f2 T2s = mul2(bc(a1.x), DY);
        const f2 E = fma2(fma2(T1, T1, mul2(T2s, T2s)), bc(-1.f), bc(a1.y));
        const float eA = lo_of(E), eB = hi_of(E);
        const bool actA = pos < s[0].last && eA >= la_min, actB = pos < s[1].last && eB >= la_min;
        const bool any = actA || actB;
        const unsigned am = __ballot_sync(0xffffffffu, any);
        if (am == 0u) continue;  // warp-uniform: no pixel of this warp uses the splat
        const float4 a2 = lds128(a + 32u * BATCH);
        const float4 a3 = DIST ? lds128(a + 48u * BATCH) : a2;
        constexpr int NG = DIST ? 16 : 12;
        float g[NG];
        bwd_accum2<DIST, NG>(P2, g, DY, col.dx, eA, eB, actA, actB, a1, a2, a3, opt);
        G2D* dst = g2d + lds32(a_id + 4u * j);
        const bool hA = actA && pos == s[0].med, hB = actB && pos == s[1].med;  // median splat (med = -1 if g_D = 0)
        if (__any_sync(0xffffffffu, hA || hB)) {
          if (hA) bwd_median(s[0], dst, PairAlpha{col.dx, lo_of(DY), eA, true});
          if (hB) bwd_median(s[1], dst, PairAlpha{col.dx, hi_of(DY), eB, true});
        }
        if (__popc(am) <= kDirectLanes) {  // few contributing threads: their own atomics, no reduction
          if (any) {
#pragma unroll
            for (int k = 0; k < NV; ++k) g2d_add(dst, k, g[k]);
          }
        } else {
          float gv[NV];
#pragma unroll
          for (int k = 0; k < NV; ++k) gv[k] = g[k];
          const float v = smem_reduce<NV>(gv, a_red, lane);
          const int k = lane >> 1;
          if ((lane & 1) == 0 && k < NV) g2d_add(dst, k, v);
        }
        continue;
      }
      PairAlpha pa[PPT];
      bool act[PPT];
      bool any = false;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        pa[k] = pair_power(a0, a1.x, a1.y, ulo, col, s[k].py, opt.log2_alpha_min);
        act[k] = pos < s[k].last && pa[k].pass;
        any = any || act[k];
      }
      const unsigned am = __ballot_sync(0xffffffffu, any);
      if (am == 0u) continue;  // warp-uniform: no pixel of this warp uses the splat
      const float4 a2 = lds128(a + 32u * BATCH);
      const float4 a3 = DIST ? lds128(a + 48u * BATCH) : a2;  // (z_c, p0, p1, ·) for d of Eq.15
      constexpr int NG = DIST ? 16 : 12;
      float g[NG];
      // a pixel row no lane uses contributes exact zeros: skip it (the first row writes g)
      if (__any_sync(0xffffffffu, act[0])) {
        bwd_accum<DIST, NG, true>(s[0], g, pa[0], act[0], a1, a2, a3, opt);
      } else {
#pragma unroll
        for (int k = 0; k < NG; ++k) g[k] = 0.f;
      }
#pragma unroll
      for (int k = 1; k < PPT; ++k)
        if (__any_sync(0xffffffffu, act[k])) bwd_accum<DIST, NG, false>(s[k], g, pa[k], act[k], a1, a2, a3, opt);
      G2D* dst = g2d + lds32(a_id + 4u * j);
      bool hit[PPT], any_hit = false;  // the splat is this pixel's median one (med = -1 if g_D = 0)
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        hit[k] = act[k] && pos == s[k].med;
        any_hit = any_hit || hit[k];
      }
      if (__any_sync(0xffffffffu, any_hit)) {  // warp-uniform: most steps have no median hit
#pragma unroll
        for (int k = 0; k < PPT; ++k)
          if (hit[k]) bwd_median(s[k], dst, pa[k]);
      }
      if (__popc(am) <= kDirectLanes) {  // few contributing threads: their own atomics, no reduction
        if (any) {
#pragma unroll
          for (int k = 0; k < NV; ++k) g2d_add(dst, k, g[k]);
        }
      } else {
        float gv[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) gv[k] = g[k];
        const float v = smem_reduce<NV>(gv, a_red, lane);
        const int k = lane >> 1;
        if ((lane & 1) == 0 && k < NV) g2d_add(dst, k, v);  // DIST: 12..14 → f[7..9] (Eq.15 sums)
      }
    }
  }
}

}  // namespace

void launch_render_fwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, float* color, float* depth, float* normal, float* alpha,
                       float* T_final, int32_t* n_contrib, int32_t* median_pos, const DistIO& dio,
                       uint32_t* bmask, uint32_t* order, Counter* counters, const DevBounds& bd, cudaStream_t s) {
  const unsigned grid = (unsigned)(tiles_x * tiles_y);
  k_tile_order<<<1, 1024, 0, s>>>(ranges, (int)grid, order);
#define RD_K3(T, P, D)                                                                                            \
  k_render_fwd<T, P, D><<<grid, T * T / 2, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, color, depth, normal,   \
                                                   alpha, T_final, n_contrib, median_pos, dio, bmask, order, counters, bd)
#define RD_K3T(T)                                     \
  if (dio.d0) {                                       \
    if (counters) RD_K3(T, true, true); else RD_K3(T, false, true);   \
  } else {                                            \
    if (counters) RD_K3(T, true, false); else RD_K3(T, false, false); \
  }
  if (opt.tile == 32) {
    RD_K3T(32)
  } else if (opt.tile == 16) {
    RD_K3T(16)
  } else {
    RD_K3T(8)
  }
#undef RD_K3T
#undef RD_K3
}

void launch_render_bwd(const DevCam& cam, const DevOpt& opt, int tiles_x, int tiles_y, const uint2* ranges,
                       const uint32_t* ids, const Record* rec, const float* T_final, const int32_t* n_contrib,
                       const int32_t* median_pos, const float* dL_dcolor, const float* dL_ddepth,
                       const float* dL_dnormal, const float* dL_dalpha, const DistIO& dio,
                       const uint32_t* bmask, const uint32_t* order, G2D* g2d, Counter* counters,
                       const DevBounds& bd, cudaStream_t s) {
  const unsigned grid = (unsigned)(tiles_x * tiles_y);
#define RD_K4(T, PPT, D)                                                                                       \
  k_render_bwd<T, PPT, D><<<grid, T * T / PPT, 0, s>>>(cam, opt, tiles_x, ranges, ids, rec, T_final, n_contrib, \
                                                       median_pos, dL_dcolor, dL_ddepth, dL_dnormal, dL_dalpha,  \
                                                       dio, bmask, order, g2d, counters, bd)
  if (opt.tile == 32) {  // 4 pixels per thread: 8 warps of 8×16 pixels (the reduction rows fit)
    if (dio.dL_ddist) RD_K4(32, 4, true); else RD_K4(32, 4, false);
  } else if (opt.tile == 16) {
    if (dio.dL_ddist) RD_K4(16, 2, true); else RD_K4(16, 2, false);
  } else {
    if (dio.dL_ddist) RD_K4(8, 2, true); else RD_K4(8, 2, false);
  }
#undef RD_K4
}

}  // namespace rade
