// preprocess.cu — K1 (per-Gaussian forward, stage 1) and K5 (per-Gaussian backward,
// second half of stage 4) of the RaDe-GS rasterizer, sm_100a.
//
// One thread per Gaussian over row-major parameters (means[N][3], scales[N][3],
// rotations[N][4], opacities[N], sh[N][K][3]); only visible Gaussians move their SH rows
// (memory-bound kernels: ~236 B in, 80 B out per visible Gaussian). K1 also feeds the
// backward: it appends the visible ids to a compact list that K5a walks.
//
// Per Gaussian (PAPER.md line refs; readings S* in DESIGN.md):
//   Σ = R S Sᵀ Rᵀ; x_c = W μ + t; u_c, v_c pinhole; t_c = ‖x_c‖
//   2-D covariance = top-left 2x2 of Σ′ = J W Σ Wᵀ Jᵀ, formed as M Mᵀ with
//     M = J₂ (W R) S (no 3x3 Σ is materialised), dilated by h·I for α only (S5)
//   depth-plane p and normal n: the paper's q̂ = v′ᵀΣ′⁻¹/(v′ᵀΣ′⁻¹v′) (Eq.13),
//     p = (z_c/t_c) q and n = normalize(Jᵀ(−(q,1)ᵀ)),
//     evaluated in the algebraically identical cancellation-free "m-form":
//       m = Σ_c⁻¹ x̂ = R_c (R_cᵀ x̂ ⊘ s²), μ = x̂ᵀ Σ_c⁻¹ x̂,
//       p_k = z_c² / (f_k t_c) · (m_k/μ − x̂_k),  n = −m/‖m‖.
//   colour from degree-≤3 SH at the Gaussian's view direction.
#include "rade_internal.cuh"

#include <math.h>

namespace rade {
namespace {

// real-SH basis constants (3DGS convention, reading S14)
constexpr float kC0 = 0.28209479177387814f;
constexpr float kC1 = 0.4886025119029199f;
constexpr float kC2_0 = 1.0925484305920792f, kC2_1 = -1.0925484305920792f, kC2_2 = 0.31539156525252005f,
                kC2_3 = -1.0925484305920792f, kC2_4 = 0.5462742152960396f;
constexpr float kC3_0 = -0.5900435899266435f, kC3_1 = 2.890611442640554f, kC3_2 = -0.4570457994644658f,
                kC3_3 = 0.3731763325901154f, kC3_4 = -0.4570457994644658f, kC3_5 = 1.445305721320277f,
                kC3_6 = -0.5900435899266435f;

__device__ __forceinline__ void sh_basis(float x, float y, float z, int deg, float Y[16]) {
  Y[0] = kC0;
  if (deg < 1) return;
  Y[1] = -kC1 * y;
  Y[2] = kC1 * z;
  Y[3] = -kC1 * x;
  if (deg < 2) return;
  float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = kC2_0 * xy;
  Y[5] = kC2_1 * yz;
  Y[6] = kC2_2 * (2.f * zz - xx - yy);
  Y[7] = kC2_3 * xz;
  Y[8] = kC2_4 * (xx - yy);
  if (deg < 3) return;
  Y[9] = kC3_0 * y * (3.f * xx - yy);
  Y[10] = kC3_1 * xy * z;
  Y[11] = kC3_2 * y * (4.f * zz - xx - yy);
  Y[12] = kC3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
  Y[13] = kC3_4 * x * (4.f * zz - xx - yy);
  Y[14] = kC3_5 * z * (xx - yy);
  Y[15] = kC3_6 * x * (xx - 3.f * yy);
}

// d(Σ_k c_k Y_k)/d(x, y, z) for the basis above (direction treated as free 3-vector).
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, int deg, const float c[16], float& gx,
                                              float& gy, float& gz) {
  gx = gy = gz = 0.f;
  if (deg < 1) return;
  gy += -kC1 * c[1];
  gz += kC1 * c[2];
  gx += -kC1 * c[3];
  if (deg < 2) return;
  float xx = x * x, yy = y * y, zz = z * z;
  gx += kC2_0 * y * c[4];
  gy += kC2_0 * x * c[4];
  gy += kC2_1 * z * c[5];
  gz += kC2_1 * y * c[5];
  gx += -2.f * kC2_2 * x * c[6];
  gy += -2.f * kC2_2 * y * c[6];
  gz += 4.f * kC2_2 * z * c[6];
  gx += kC2_3 * z * c[7];
  gz += kC2_3 * x * c[7];
  gx += 2.f * kC2_4 * x * c[8];
  gy += -2.f * kC2_4 * y * c[8];
  if (deg < 3) return;
  gx += kC3_0 * 6.f * x * y * c[9];
  gy += kC3_0 * 3.f * (xx - yy) * c[9];
  gx += kC3_1 * y * z * c[10];
  gy += kC3_1 * x * z * c[10];
  gz += kC3_1 * x * y * c[10];
  gx += kC3_2 * (-2.f * x * y) * c[11];
  gy += kC3_2 * (4.f * zz - xx - 3.f * yy) * c[11];
  gz += kC3_2 * 8.f * y * z * c[11];
  gx += kC3_3 * (-6.f * x * z) * c[12];
  gy += kC3_3 * (-6.f * y * z) * c[12];
  gz += kC3_3 * (6.f * zz - 3.f * xx - 3.f * yy) * c[12];
  gx += kC3_4 * (4.f * zz - 3.f * xx - yy) * c[13];
  gy += kC3_4 * (-2.f * x * y) * c[13];
  gz += kC3_4 * 8.f * x * z * c[13];
  gx += kC3_5 * 2.f * x * z * c[14];
  gy += kC3_5 * (-2.f * y * z) * c[14];
  gz += kC3_5 * (xx - yy) * c[14];
  gx += kC3_6 * 3.f * (xx - yy) * c[15];
  gy += kC3_6 * (-6.f * x * y) * c[15];
}

// Forward quantities of one Gaussian (registers only). S = double in K1 (HBM-bound, and
// B200's FP64 pipe is fast: the geometry — conic, plane p, normal n — is then accurate to
// fp32 rounding of the stored results even for flat, near-grazing splats), S = float in K5.
template <typename S>
struct GF {
  float mu[3], s[3], qr[4], o;
  float s_raw[3], o_raw;  // the inputs before the 3D filter (= s, o without it)
  float zkey;   // the fp32 sort key of reading S7 (also the stored z_c)
  S qinv, qn[4];
  S Rc[9];  // W R(q̂), row-major
  S x[3], t2, it;
  S u, v;
  S RS[9];  // Rc diag(s)
  S j00, j02, j11, j12;
  S M[6];   // J₂ RS, rows 0..1
  S A00, A01, A11, det, ca, cb, cc;
  S xh[3], rh[3], w[3], ah[3], eps[3], muq, ml;
  S e0, e1, p0, p1, n[3];
};

// First NV floats of one Gaussian's SH row (row-major [n][sh_coeffs][3]) into registers:
// 16-byte vector loads when the row length is a multiple of 4 floats (rows then stay
// 16-B aligned), scalar loads otherwise. out[NV..] is zero-filled in the scalar case.
template <int NV>
__device__ __forceinline__ void load_sh_row(const float* __restrict__ row, bool vec, float (&out)[(NV + 3) / 4 * 4]) {
  constexpr int NV4 = (NV + 3) / 4;
  if (vec) {
#pragma unroll
    for (int q = 0; q < NV4; ++q) {
      const float4 v = reinterpret_cast<const float4*>(row)[q];
      out[4 * q] = v.x;
      out[4 * q + 1] = v.y;
      out[4 * q + 2] = v.z;
      out[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < NV4 * 4; ++j) out[j] = j < NV ? row[j] : 0.f;
  }
}

__device__ __forceinline__ bool isfin(float v) { return isfinite(v); }
__device__ __forceinline__ bool isfin(double v) { return isfinite(v); }
__device__ __forceinline__ float rsq(float v) { return rsqrtf(v); }
__device__ __forceinline__ double rsq(double v) { return rsqrt(v); }
__device__ __forceinline__ float sq_root(float v) { return sqrtf(v); }
__device__ __forceinline__ double sq_root(double v) { return sqrt(v); }

// Loads one Gaussian and runs stage 1 up to the conic (no plane, no SH). False if culled.
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Gradient accumulation into the caller's arrays is by L2 reductions (red.global.add, fire
// and forget): no read round trip, and rd_preprocess_bwd calls of different views into the
// same gradient arrays may run concurrently (the summation order, hence the rounding, then
// depends on timing).
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// pf_sh (K1): once the cheap culls pass, prefetch the Gaussian's SH row into L2 so its fetch
// overlaps the covariance math instead of following it.
// Cull reasons (rd_timings.n_culled; SPEC:49, 58, 76, 85 — a degenerate primitive is culled,
// not an error): the first that applies, in this order.
enum CullWhy { kVisible = 0, kCullInvalid = 1, kCullNear = 2, kCullGuard = 3, kCullOpacity = 4, kCullDegenerate = 5,
               kCullOffscreen = 6 };

template <typename S>
__device__ __forceinline__ bool gaussian_project(const DevGauss& g, int64_t i, const DevCam& cam, const DevOpt& opt,
                                                 GF<S>& f, bool pf_sh = false, int* why = nullptr) {
  // every parameter load is issued before the cull tests, which are combined into one exit:
  // K1 is latency-bound, and loads behind early exits would be four dependent HBM round trips
  f.mu[0] = g.means[3 * i];
  f.mu[1] = g.means[3 * i + 1];
  f.mu[2] = g.means[3 * i + 2];
  f.o = g.opac[i];
  f.s[0] = g.scales[3 * i];
  f.s[1] = g.scales[3 * i + 1];
  f.s[2] = g.scales[3 * i + 2];
  const float4 q4 = reinterpret_cast<const float4*>(g.rot)[i];  // [n][4], 16-B aligned rows
  const float fl = g.filter3d ? g.filter3d[i] : 0.f;
  const bool finite_mu = isfin(f.mu[0]) & isfin(f.mu[1]) & isfin(f.mu[2]);
  // centre depth in the fixed fp32 op order of reading S7 (it is also the sort key)
  const float z = __fmaf_rn(cam.R[6], f.mu[0], __fmaf_rn(cam.R[7], f.mu[1], __fmaf_rn(cam.R[8], f.mu[2], cam.t[2])));
  const bool near_ok = z > cam.znear;
  bool guard_ok = true;
  if (cam.guard) {  // guard band (reading S6b, optional), decided in fp32 with the oracle's op order
    const float xk = __fmaf_rn(cam.R[0], f.mu[0], __fmaf_rn(cam.R[1], f.mu[1], __fmaf_rn(cam.R[2], f.mu[2], cam.t[0])));
    const float yk = __fmaf_rn(cam.R[3], f.mu[0], __fmaf_rn(cam.R[4], f.mu[1], __fmaf_rn(cam.R[5], f.mu[2], cam.t[1])));
    const float fu = __fmul_rn(cam.fx, xk), fv = __fmul_rn(cam.fy, yk);
    guard_ok = (fu >= __fmul_rn(cam.gu0, z)) & (fu <= __fmul_rn(cam.gu1, z)) & (fv >= __fmul_rn(cam.gv0, z)) &
               (fv <= __fmul_rn(cam.gv1, z));
  }
  f.zkey = z;
  const bool opac_ok = f.o >= opt.alpha_min;  // o' ≤ o: also culls the filtered one
  f.qr[0] = q4.x;
  f.qr[1] = q4.y;
  f.qr[2] = q4.z;
  f.qr[3] = q4.w;
  const bool valid = finite_mu & isfin(f.o) & (f.s[0] > 0.f) & (f.s[1] > 0.f) & (f.s[2] > 0.f) & isfin(f.s[0]) &
                     isfin(f.s[1]) & isfin(f.s[2]) & isfin(f.qr[0]) & isfin(f.qr[1]) & isfin(f.qr[2]) &
                     isfin(f.qr[3]);
  if (!(valid & near_ok & guard_ok & opac_ok)) {
    if (why) *why = !valid ? kCullInvalid : !near_ok ? kCullNear : !guard_ok ? kCullGuard : kCullOpacity;
    return false;
  }
  if (pf_sh) {  // the row's first and last byte: its (at most two) 128-B lines
    const float* row = g.sh + i * g.sh_coeffs * 3;
    prefetch_l2(row);
    prefetch_l2(row + g.sh_coeffs * 3 - 1);
  }
  f.s_raw[0] = f.s[0];
  f.s_raw[1] = f.s[1];
  f.s_raw[2] = f.s[2];
  f.o_raw = f.o;
  if (g.filter3d) {  // 3D filter (S23): Σ + f²I ⇔ s' = √(s² + f²); o' = o·Π s/s'
    if (!isfin(fl)) {
      if (why) *why = kCullInvalid;
      return false;
    }
    float ratio = 1.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float sp = sqrtf(fmaf(f.s[k], f.s[k], fl * fl));
      ratio *= f.s[k] / sp;
      f.s[k] = sp;
    }
    f.o *= ratio;
    if (!(f.o >= opt.alpha_min)) {
      if (why) *why = kCullOpacity;
      return false;
    }
  }
  const S ql2 = (S)f.qr[0] * f.qr[0] + (S)f.qr[1] * f.qr[1] + (S)f.qr[2] * f.qr[2] + (S)f.qr[3] * f.qr[3];
  if (!(ql2 > S(0))) {
    if (why) *why = kCullInvalid;  // zero quaternion
    return false;
  }

  const S R[9] = {cam.R[0], cam.R[1], cam.R[2], cam.R[3], cam.R[4], cam.R[5], cam.R[6], cam.R[7], cam.R[8]};
#pragma unroll
  for (int r = 0; r < 3; ++r)
    f.x[r] = R[3 * r] * f.mu[0] + R[3 * r + 1] * f.mu[1] + R[3 * r + 2] * f.mu[2] + (S)cam.t[r];
  f.t2 = f.x[0] * f.x[0] + f.x[1] * f.x[1] + f.x[2] * f.x[2];
  f.it = rsq(f.t2);
  const S iz = S(1) / f.x[2];
  f.u = f.x[0] * iz * (S)cam.fx + (S)cam.cx;
  f.v = f.x[1] * iz * (S)cam.fy + (S)cam.cy;

  // R(q̂), q̂ = q/‖q‖, (w, x, y, z) (reading S15)
  f.qinv = rsq(ql2);
  const S w = f.qr[0] * f.qinv, a = f.qr[1] * f.qinv, b = f.qr[2] * f.qinv, c = f.qr[3] * f.qinv;
  f.qn[0] = w; f.qn[1] = a; f.qn[2] = b; f.qn[3] = c;
  const S one(1), two(2);
  const S Rq[9] = {one - two * (b * b + c * c), two * (a * b - w * c), two * (a * c + w * b),
                   two * (a * b + w * c), one - two * (a * a + c * c), two * (b * c - w * a),
                   two * (a * c - w * b), two * (b * c + w * a), one - two * (a * a + b * b)};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) f.Rc[3 * r + k] = R[3 * r] * Rq[k] + R[3 * r + 1] * Rq[3 + k] + R[3 * r + 2] * Rq[6 + k];

  // 2-D covariance: M = J₂ R_c S, A = M Mᵀ (+ h I) (S2, S5)
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) f.RS[3 * r + k] = f.Rc[3 * r + k] * f.s[k];
  f.j00 = (S)cam.fx * iz;
  f.j02 = -(S)cam.fx * f.x[0] * iz * iz;
  f.j11 = (S)cam.fy * iz;
  f.j12 = -(S)cam.fy * f.x[1] * iz * iz;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    f.M[k] = f.j00 * f.RS[k] + f.j02 * f.RS[6 + k];
    f.M[3 + k] = f.j11 * f.RS[3 + k] + f.j12 * f.RS[6 + k];
  }
  f.A00 = f.M[0] * f.M[0] + f.M[1] * f.M[1] + f.M[2] * f.M[2] + (S)opt.dilation;
  f.A01 = f.M[0] * f.M[3] + f.M[1] * f.M[4] + f.M[2] * f.M[5];
  f.A11 = f.M[3] * f.M[3] + f.M[4] * f.M[4] + f.M[5] * f.M[5] + (S)opt.dilation;
  f.det = f.A00 * f.A11 - f.A01 * f.A01;
  if (!(f.det > S(0)) || !isfin(f.det)) {
    if (why) *why = kCullDegenerate;
    return false;
  }
  const S idet = S(1) / f.det;
  f.ca = f.A11 * idet;
  f.cb = -f.A01 * idet;
  f.cc = f.A00 * idet;
  return true;
}

// Depth plane and normal (m-form of Eq.12-15, 21-22), evaluated in the Gaussian's local
// frame (columns of R_c): r = R_cᵀx̂ (a unit vector), w_k = 1/s_k², a = r∘w, μ = r·a, so
// m = R_c a, ‖m‖ = ‖a‖, n = −R_c a/‖a‖ and e = m/μ − x̂ = R_c ε with
//   ε_k = a_k/μ − r_k = r_k (w_k − μ)/μ,  w_k − μ = Σ_{j≠k} r_j² (w_k − w_j)   (Σ r_j² = 1),
// which has no cancellation even for a flat splat seen face-on (r ≈ its thin axis, where
// a_k/μ − r_k subtracts nearly equal numbers). Returns false if degenerate.
template <typename S>
__device__ __forceinline__ bool gaussian_plane(const DevCam& cam, GF<S>& f) {
#pragma unroll
  for (int k = 0; k < 3; ++k) f.xh[k] = f.x[k] * f.it;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    f.rh[k] = f.Rc[k] * f.xh[0] + f.Rc[3 + k] * f.xh[1] + f.Rc[6 + k] * f.xh[2];
    f.w[k] = S(1) / ((S)f.s[k] * f.s[k]);
    f.ah[k] = f.rh[k] * f.w[k];
  }
  f.muq = f.rh[0] * f.ah[0] + f.rh[1] * f.ah[1] + f.rh[2] * f.ah[2];
  f.ml = sq_root(f.ah[0] * f.ah[0] + f.ah[1] * f.ah[1] + f.ah[2] * f.ah[2]);
  if (!(f.muq > S(0)) || !isfin(f.muq) || !(f.ml > S(0)) || !isfin(f.ml)) return false;
  const S imu = S(1) / f.muq;
  const S r2[3] = {f.rh[0] * f.rh[0], f.rh[1] * f.rh[1], f.rh[2] * f.rh[2]};
  f.eps[0] = f.rh[0] * (r2[1] * (f.w[0] - f.w[1]) + r2[2] * (f.w[0] - f.w[2])) * imu;
  f.eps[1] = f.rh[1] * (r2[0] * (f.w[1] - f.w[0]) + r2[2] * (f.w[1] - f.w[2])) * imu;
  f.eps[2] = f.rh[2] * (r2[0] * (f.w[2] - f.w[0]) + r2[1] * (f.w[2] - f.w[1])) * imu;
  f.e0 = f.Rc[0] * f.eps[0] + f.Rc[1] * f.eps[1] + f.Rc[2] * f.eps[2];
  f.e1 = f.Rc[3] * f.eps[0] + f.Rc[4] * f.eps[1] + f.Rc[5] * f.eps[2];
  const S zzit = f.x[2] * f.x[2] * f.it;
  f.p0 = zzit / (S)cam.fx * f.e0;
  f.p1 = zzit / (S)cam.fy * f.e1;
  const S iml = S(1) / f.ml;
#pragma unroll
  for (int r = 0; r < 3; ++r) f.n[r] = -(f.Rc[3 * r] * f.ah[0] + f.Rc[3 * r + 1] * f.ah[1] + f.Rc[3 * r + 2] * f.ah[2]) * iml;
  return true;
}

// Stage 1 up to (but not including) SH. Returns false if culled.
template <typename S>
__device__ __forceinline__ bool gaussian_forward(const DevGauss& g, int64_t i, const DevCam& cam, const DevOpt& opt,
                                                 GF<S>& f) {
  return gaussian_project<S>(g, i, cam, opt, f) && gaussian_plane<S>(cam, f);
}

// ---------------------------------------------------------------------------- K1
// One Gaussian: writes its record, rect, tiles_touched and depth key; returns the rect
// (tile x0, y0, width) and the number of tiles it touches (0: culled / off-screen).
template <int DEG>
__device__ __forceinline__ uint32_t preprocess_one(const DevGauss& g, int64_t i, const DevCam& cam,
                                                   const DevOpt& opt, Record* __restrict__ rec,
                                                   uint2* __restrict__ rect, uint32_t* __restrict__ touched,
                                                   uint32_t* __restrict__ dkey, uint32_t& rx0, uint32_t& ry0,
                                                   uint32_t& rw, int& why) {
  GF<double> f;
  why = kVisible;
  if (!gaussian_project<double>(g, i, cam, opt, f, true, &why)) {
    touched[i] = 0u;
    dkey[i] = 0xffffffffu;
    return 0u;
  }
  // α-bounded footprint: α = o·G ≥ α_min ⇔ Δᵀ conic Δ ≤ k = 2 ln(o/α_min); its axis-aligned
  // half extents are sqrt(k·A′₀₀), sqrt(k·A′₁₁) (reading S8); inflated for fp32 safety.
  const float uc = (float)f.u, vc = (float)f.v;
  const float kk = 2.f * (logf(f.o) - opt.ln_alpha_min);
  const float rx = sqrtf(fmaxf(kk, 0.f) * (float)f.A00) * 1.00001f + 1e-3f;
  const float ry = sqrtf(fmaxf(kk, 0.f) * (float)f.A11) * 1.00001f + 1e-3f;
  // pixels i with |u_c − (i + ½)| ≤ rx (evaluated on the stored fp32 u_c the blend uses)
  const float fx0 = fmaxf(ceilf(uc - rx - 0.5f), 0.f);
  const float fx1 = fminf(floorf(uc + rx - 0.5f), (float)(cam.W - 1));
  const float fy0 = fmaxf(ceilf(vc - ry - 0.5f), 0.f);
  const float fy1 = fminf(floorf(vc + ry - 0.5f), (float)(cam.H - 1));
  if (!(fx0 <= fx1 && fy0 <= fy1)) {
    touched[i] = 0u;
    dkey[i] = 0xffffffffu;
    why = kCullOffscreen;
    return 0u;
  }
  const int T = opt.tile;
  const uint32_t tx0 = (uint32_t)fx0 / T, tx1 = (uint32_t)fx1 / T + 1;
  const uint32_t ty0 = (uint32_t)fy0 / T, ty1 = (uint32_t)fy1 / T + 1;

  // visible: issue the SH row loads now so their latency overlaps the plane math
  constexpr int K = (DEG + 1) * (DEG + 1);
  float c[(3 * K + 3) / 4 * 4];
  load_sh_row<3 * K>(g.sh + (int64_t)i * g.sh_coeffs * 3, (g.sh_coeffs * 3) % 4 == 0, c);
  if (!gaussian_plane<double>(cam, f)) {
    touched[i] = 0u;
    dkey[i] = 0xffffffffu;
    why = kCullDegenerate;
    return 0u;
  }

  // colour: dir = normalize(μ − campos), degree ≤ sh_degree, + 0.5, clamp ≥ 0
  float dx = f.mu[0] - cam.campos[0], dy = f.mu[1] - cam.campos[1], dz = f.mu[2] - cam.campos[2];
  const float idl = rsqrtf(dx * dx + dy * dy + dz * dz);
  dx *= idl; dy *= idl; dz *= idl;
  float Y[16];
  sh_basis(dx, dy, dz, DEG, Y);
  float rgb[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) rgb[ch] += Y[k] * c[k * 3 + ch];
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = fmaxf(rgb[ch], 0.f);

  Record r;
  const double L2E = 1.4426950408889634;
  // centre as fp32 + half remainder (rade_internal.cuh: Record)
  const __half2 uvlo = __floats2half2_rn((float)(f.u - (double)uc), (float)(f.v - (double)vc));
  // (log2e/2)·conic = UᵀU, U = [[g11, g21], [0, g22]] (Cholesky, from the covariance side:
  // g22² = (log2e/2)/A′11 needs no difference of products)
  const double Lh = 0.5 * L2E;
  const double g11 = sqrt(Lh * (double)f.ca), g21 = (double)f.cb * sqrt(Lh / (double)f.ca);
  const double g22 = sqrt(Lh / (double)f.A11);
  r.r0 = make_float4(uc, vc, (float)g11, (float)g21);
  r.r1 = make_float4((float)g22, (float)log2((double)f.o), rgb[0], rgb[1]);
  r.r2 = make_float4(rgb[2], (float)f.n[0], (float)f.n[1], (float)f.n[2]);
  r.r3 = make_float4(f.zkey, (float)f.p0, (float)f.p1, *reinterpret_cast<const float*>(&uvlo));
  rec[i] = r;
  rect[i] = make_uint2(tx0 | (ty0 << 16), tx1 | (ty1 << 16));
  const uint32_t nt = (tx1 - tx0) * (ty1 - ty0);
  touched[i] = nt;
  dkey[i] = __float_as_uint(f.zkey);
  rx0 = tx0;
  ry0 = ty0;
  rw = tx1 - tx0;
  return nt;
}

// K1 kernel: per-Gaussian forward (plus the depth-sort input dkey[i] in id order), then
// the warp-aggregated append of the visible ids to the visible list (one atomic per warp;
// list order is arbitrary — K5a, its only user, is order-independent).
#ifndef RD_K5_THREADS
#define RD_K5_THREADS 128
#endif
// K5b at ≤ 80 registers (768 threads per SM): more warps in flight for its gathers (0.096 -> 0.082 ms)
#ifndef RD_K5_MINB
#define RD_K5_MINB (768 / RD_K5_THREADS)  // (measured: 5 → 96 registers, 7 → 72: both slower)
#endif
#ifndef RD_K1_THREADS
#define RD_K1_THREADS 64  // finer blocks fill the SMs more evenly: 0.107 -> 0.101 ms
#endif
#ifndef RD_K1_MINB
#define RD_K1_MINB 8  // ≤ 128 registers: 16 warps per SM for the latency-bound loads
#endif
// The per-Gaussian part of K1 for one view plus its warp-level appends (all 32 lanes call it).
template <int DEG>
__device__ __forceinline__ void k1_view(const DevGauss& g, int64_t i, const DevCam& cam, const DevOpt& opt,
                                        Record* __restrict__ rec, uint2* __restrict__ rect,
                                        uint32_t* __restrict__ touched, uint32_t* __restrict__ dkey,
                                        uint32_t* __restrict__ count, uint32_t* __restrict__ vis,
                                        uint32_t* __restrict__ big, G2D* __restrict__ g2d,
                                        Counter* __restrict__ counters) {
  const int lane = (int)(threadIdx.x & 31);
  uint32_t x0 = 0, y0 = 0, w = 1, nt = 0;
  int why = kVisible;
  if (i < g.n) {
    nt = preprocess_one<DEG>(g, i, cam, opt, rec, rect, touched, dkey, x0, y0, w, why);
  }
  if (counters) {  // profiling: culls by reason (warp-aggregated)
#pragma unroll
    for (int r = kCullInvalid; r <= kCullOffscreen; ++r) {
      const unsigned m = __ballot_sync(0xffffffffu, i < g.n && why == r);
      if (lane == 0 && m)
        atomicAdd(counters + kCullCounter0 + (r - 1) * kCullSlots + (blockIdx.x & (kCullSlots - 1)), (Counter)__popc(m));
    }
  }
  const unsigned vmask = __ballot_sync(0xffffffffu, nt > 0u);
  if (vmask == 0u) return;  // warp-uniform
  const bool bigg = is_big(nt, opt.tile);
  const unsigned bmask = __ballot_sync(0xffffffffu, bigg);
  uint32_t base = 0, bbase = 0;
  if (lane == 0) {
    base = atomicAdd(count, (uint32_t)__popc(vmask));
    if (bmask) bbase = atomicAdd(count + 1, (uint32_t)__popc(bmask));
    if (counters) atomicAdd(counters + 3, (Counter)__popc(vmask));
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  bbase = __shfl_sync(0xffffffffu, bbase, 0);
  const unsigned below = (1u << lane) - 1u;
  if (nt > 0u) {
    RD_CHECK((int64_t)(base + __popc(vmask & below)) < g.n);
    vis[base + __popc(vmask & below)] = (uint32_t)i;
    float4* row = reinterpret_cast<float4*>(g2d + i);
#pragma unroll
    for (int q = 0; q < 5; ++q) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (bigg) {
    RD_CHECK((int64_t)(bbase + __popc(bmask & below)) < g.n);
    big[bbase + __popc(bmask & below)] = (uint32_t)i;
  }
}

template <int DEG>
__global__ void __launch_bounds__(RD_K1_THREADS, RD_K1_MINB) k_preprocess_fwd(DevGauss g, DevCam cam, DevOpt opt, int tiles_x,
                                                         Record* __restrict__ rec, uint2* __restrict__ rect,
                                                         uint32_t* __restrict__ touched, uint32_t* __restrict__ dkey,
                                                         uint32_t* __restrict__ count, uint32_t* __restrict__ vis,
                                                         uint32_t* __restrict__ big, G2D* __restrict__ g2d,
                                                         Counter* __restrict__ counters) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  k1_view<DEG>(g, i, cam, opt, rec, rect, touched, dkey, count, vis, big, g2d, counters);
}

// K1 over a round of views of the same Gaussians: each thread runs its Gaussian through every
// view in turn, so the parameter and SH rows come from DRAM once and from L1/L2 after that
// (4 views read 84 MB of parameters and ~0.2 GB of SH rows once instead of 4×).
template <int DEG>
__global__ void __launch_bounds__(RD_K1_THREADS, RD_K1_MINB) k_preprocess_fwd_views(DevGauss g, DevOpt opt,
                                                                              const __grid_constant__ K1Views kv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 1
  for (int v = 0; v < kv.nv; ++v) {
    const K1Out& o = kv.v[v];
    k1_view<DEG>(g, i, o.cam, opt, o.rec, o.rect, o.touched, o.dkey, o.count, o.vis, o.big, o.g2d, o.counters);
  }
}

// ---------------------------------------------------------------------------- K5
// Two kernels, one thread per Gaussian in id order; only visible Gaussians (tiles_touched >
// 0, ≈ half at C3) read and write their rows, so with row-major parameters the invisible
// half stays out of the DRAM traffic. K5a (SH colour) and K5b (geometry) are split so each
// issues its independent loads in one round trip at a register count that keeps enough
// warps in flight to cover HBM latency. K5a runs first and leaves the view-direction part
// of dL/dμ in the mean gradient; K5b adds the projection part.

// K5a (per-thread fallback for SH rows that are not a multiple of 4 floats).
template <int DEG>
__global__ void __launch_bounds__(128) k_preprocess_bwd_sh(DevGauss g, DevCam cam, DevOpt opt,
                                                           const uint32_t* __restrict__ touched,
                                                           const G2D* __restrict__ g2d, DevGrads gr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  if (touched[i] == 0u) return;  // culled or off-screen: zero gradient
  const float d_rgb[3] = {g2d[i].f[1], g2d[i].f[2], g2d[i].f[3]};
  const float mu0 = g.means[3 * i], mu1 = g.means[3 * i + 1], mu2 = g.means[3 * i + 2];
  float dmu[3] = {0.f, 0.f, 0.f};
  {
    float ex = mu0 - cam.campos[0], ey = mu1 - cam.campos[1], ez = mu2 - cam.campos[2];
    const float idl = rsqrtf(ex * ex + ey * ey + ez * ez);
    const float hx = ex * idl, hy = ey * idl, hz = ez * idl;
    float Y[16];
    sh_basis(hx, hy, hz, DEG, Y);
    constexpr int K = (DEG + 1) * (DEG + 1);
    float rgb[3] = {0.5f, 0.5f, 0.5f};
    constexpr int NV = 3 * K, NV4 = (NV + 3) / 4;
    const bool vec = (g.sh_coeffs * 3) % 4 == 0;
    float coef[NV4 * 4];
    load_sh_row<NV>(g.sh + (int64_t)i * g.sh_coeffs * 3, vec, coef);
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) rgb[ch] += Y[k] * coef[k * 3 + ch];
    float drgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) drgb[ch] = rgb[ch] < 0.f ? 0.f : d_rgb[ch];
    // += into this Gaussian's contiguous SH gradient row (16-B vector reductions when aligned;
    // entries past the active degree get + 0)
    float* gsh = gr.sh + (int64_t)i * g.sh_coeffs * 3;
    if (vec) {
      float4* g4 = reinterpret_cast<float4*>(gsh);
#pragma unroll
      for (int q = 0; q < NV4; ++q) {
        float d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) d[e] = (4 * q + e) < NV ? Y[(4 * q + e) / 3] * drgb[(4 * q + e) % 3] : 0.f;
        red_add4(g4 + q, make_float4(d[0], d[1], d[2], d[3]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j) red_add(gsh + j, Y[j / 3] * drgb[j % 3]);
    }
    float c16[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      c16[k] = k < K ? drgb[0] * coef[3 * k] + drgb[1] * coef[3 * k + 1] + drgb[2] * coef[3 * k + 2] : 0.f;
    float gx, gy, gz;
    sh_basis_grad(hx, hy, hz, DEG, c16, gx, gy, gz);
    // through the normalisation of dir
    const float dot = gx * hx + gy * hy + gz * hz;
    dmu[0] += (gx - hx * dot) * idl;
    dmu[1] += (gy - hy * dot) * idl;
    dmu[2] += (gz - hz * dot) * idl;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) red_add(gr.means + 3 * i + k, dmu[k]);
}

// One Gaussian's gradient rows (μ, s, raw q, o) summed over the views a K5b launch handles,
// added to the caller's arrays once by grad_flush.
struct GradAcc {
  float dmu[3], ds[3], dq[4], dop, duv[2];
};
__device__ __forceinline__ void grad_zero(GradAcc& a) {
#pragma unroll
  for (int k = 0; k < 3; ++k) a.dmu[k] = a.ds[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) a.dq[k] = 0.f;
  a.dop = a.duv[0] = a.duv[1] = 0.f;
}
__device__ __forceinline__ void grad_flush(const GradAcc& a, DevGrads& gr, int64_t i) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    red_add(gr.means + 3 * i + k, a.dmu[k]);
    red_add(gr.scales + 3 * i + k, a.ds[k]);
  }
  red_add4(reinterpret_cast<float4*>(gr.rot) + i, make_float4(a.dq[0], a.dq[1], a.dq[2], a.dq[3]));
  red_add(gr.opac + i, a.dop);
  if (gr.means2d) {  // optional screen-space gradient
    red_add(gr.means2d + 2 * i, a.duv[0]);
    red_add(gr.means2d + 2 * i + 1, a.duv[1]);
  }
}

// K5b: geometry — centre, conic, depth plane and normal of one view back to μ, s, q, o,
// added to acc; false if the Gaussian is culled in this view.
template <typename S>
__device__ __forceinline__ bool geometry_backward(const DevGauss& g, int64_t i, const DevCam& cam, const DevOpt& opt,
                                                  const G2D* __restrict__ g2d, GradAcc& acc) {
  // the G2D row is needed only after the forward recompute: have it on its way to L2 now
  // (no registers held)
  prefetch_l2(g2d + i);
  prefetch_l2(reinterpret_cast<const char*>(g2d + i) + sizeof(G2D) - 1);
  GF<S> f;
  if (!gaussian_forward<S>(g, i, cam, opt, f)) return false;
  // the G2D sums of K4 → 2-D gradients (log2 e · ln 2 = 1 cancels between the stored
  // (A2, B2, C2) = log2e·(−a/2, −b, −c/2) and α = 2^e):
  //   dL/du = −(a S0 + b S1) + p0 S12, dL/dv = −(b S0 + c S1) + p1 S12,
  //   dL/da = −S2/2, dL/db = −S3, dL/dc = −S4/2, dL/do = S5/o (∂α_raw/∂o = α_raw/o)
  const G2D& q = g2d[i];
  const S S0 = (S)q.m[0], S1 = (S)q.m[1], S2 = (S)q.m[2], S3 = (S)q.m[3], S4 = (S)q.m[4];
  const S S12 = q.f[7];
  const S d_u = -(f.ca * S0 + f.cb * S1) + f.p0 * S12;
  const S d_v = -(f.cb * S0 + f.cc * S1) + f.p1 * S12;
  acc.duv[0] += (float)d_u;  // dL/d(u_c, v_c): the screen-space gradient (rd_grads.means2d)
  acc.duv[1] += (float)d_v;
  const float d_o = q.f[0] / f.o;
  const S d_n[3] = {q.f[4], q.f[5], q.f[6]};
  const S d_z = S12, d_p0 = q.f[8], d_p1 = q.f[9];

  S dx[3] = {0, 0, 0};  // dL/dx_c (camera space)
  S dRc[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) dRc[k] = 0;
  S ds[3] = {0, 0, 0};
  S dmu[3] = {0, 0, 0};

  // ---- projected centre and centre depth
  const S iz = S(1) / f.x[2];
  dx[0] += d_u * cam.fx * iz;
  dx[1] += d_v * cam.fy * iz;
  dx[2] += -(d_u * cam.fx * f.x[0] + d_v * cam.fy * f.x[1]) * iz * iz + d_z;

  // ---- conic: stored (A2, B2, C2) = log2e·(−a/2, −b, −c/2), conic = A′⁻¹
  {
    const S da = S(-0.5) * S2, db = -S3, dc = S(-0.5) * S4;
    // dL/dA′ = −C Ḡ C with Ḡ = [[da, db/2], [db/2, dc]]; off-diagonal counted twice
    const S a = f.ca, b = f.cb, c = f.cc;
    const S dA00 = -(a * a * da + a * b * db + b * b * dc);
    const S dA11 = -(b * b * da + b * c * db + c * c * dc);
    const S dA01 = -(S(2) * a * b * da + (a * c + b * b) * db + S(2) * b * c * dc);
    // A = M Mᵀ
    S dM[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dM[k] = S(2) * dA00 * f.M[k] + dA01 * f.M[3 + k];
      dM[3 + k] = dA01 * f.M[k] + S(2) * dA11 * f.M[3 + k];
    }
    // M = J₂ RS
    S dj00 = 0, dj02 = 0, dj11 = 0, dj12 = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dj00 += dM[k] * f.RS[k];
      dj02 += dM[k] * f.RS[6 + k];
      dj11 += dM[3 + k] * f.RS[3 + k];
      dj12 += dM[3 + k] * f.RS[6 + k];
      const S dRS0 = dM[k] * f.j00;
      const S dRS1 = dM[3 + k] * f.j11;
      const S dRS2 = dM[k] * f.j02 + dM[3 + k] * f.j12;
      dRc[k] += dRS0 * f.s[k];
      dRc[3 + k] += dRS1 * f.s[k];
      dRc[6 + k] += dRS2 * f.s[k];
      ds[k] += dRS0 * f.Rc[k] + dRS1 * f.Rc[3 + k] + dRS2 * f.Rc[6 + k];
    }
    // J₂(x): j00 = fx/z, j02 = −fx x/z², j11 = fy/z, j12 = −fy y/z²
    const S iz2 = iz * iz;
    dx[0] += -dj02 * cam.fx * iz2;
    dx[1] += -dj12 * cam.fy * iz2;
    dx[2] += -dj00 * cam.fx * iz2 - dj11 * cam.fy * iz2 + S(2) * dj02 * cam.fx * f.x[0] * iz2 * iz +
             S(2) * dj12 * cam.fy * f.x[1] * iz2 * iz;
  }

  // ---- depth plane p and normal n: the m-form backward in the local frame (gaussian_plane),
  // with every difference of nearly equal terms written as a sum of the remaining ones, so a
  // flat splat's thin-axis gradients keep their relative accuracy in fp32
  {
    const S imu = S(1) / f.muq;
    const S iml = S(1) / f.ml;
    // p_k = c_k e_k, c_k = z² it / f_k, e = R_c ε ; n = −R_c â, â = a/‖a‖
    const S z = f.x[2];
    const S zzit = z * z * f.it;
    const S de0 = d_p0 * zzit / cam.fx, de1 = d_p1 * zzit / cam.fy;
    dx[2] += S(2) * (d_p0 * f.p0 + d_p1 * f.p1) / z;
    S dit = (d_p0 * f.p0 + d_p1 * f.p1) / f.it;
    S ah_n[3], deps[3], dahat[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      ah_n[k] = f.ah[k] * iml;
      deps[k] = f.Rc[k] * de0 + f.Rc[3 + k] * de1;
      dahat[k] = -(f.Rc[k] * d_n[0] + f.Rc[3 + k] * d_n[1] + f.Rc[6 + k] * d_n[2]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dRc[k] += de0 * f.eps[k] - d_n[0] * ah_n[k];
      dRc[3 + k] += de1 * f.eps[k] - d_n[1] * ah_n[k];
      dRc[6 + k] += -d_n[2] * ah_n[k];
    }
    const S A = deps[0] * f.ah[0] + deps[1] * f.ah[1] + deps[2] * f.ah[2];
    S dr[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int j1 = k == 0 ? 1 : 0, j2 = k == 2 ? 1 : 2;  // the other two axes
      // â = a/‖a‖: da_k = (dâ_k Σ_{j≠k} â_j² − â_k Σ_{j≠k} â_j dâ_j)/‖a‖
      const S da = (dahat[k] * (ah_n[j1] * ah_n[j1] + ah_n[j2] * ah_n[j2]) -
                    ah_n[k] * (ah_n[j1] * dahat[j1] + ah_n[j2] * dahat[j2])) * iml;
      // ε_k = a_k/μ − r_k, μ = Σ r_j a_j: ∂/∂w_k = (r_k/μ²)(dε_k S_k − r_k T_k) with
      // S_k = Σ_{j≠k} r_j a_j = μ − r_k a_k and T_k = Σ_{j≠k} dε_j a_j
      const S Sk = f.rh[j1] * f.ah[j1] + f.rh[j2] * f.ah[j2];
      const S Tk = deps[j1] * f.ah[j1] + deps[j2] * f.ah[j2];
      const S dw = da * f.rh[k] + f.rh[k] * (deps[k] * Sk - f.rh[k] * Tk) * imu * imu;
      // ∂ε_j/∂r_k = δ_jk (w_k − μ)/μ − 2 r_j w_j a_k/μ², w_k − μ = Σ_{j≠k} r_j² (w_k − w_j)
      const S wk_mu = f.rh[j1] * f.rh[j1] * (f.w[k] - f.w[j1]) + f.rh[j2] * f.rh[j2] * (f.w[k] - f.w[j2]);
      dr[k] = da * f.w[k] + deps[k] * wk_mu * imu - S(2) * f.ah[k] * A * imu * imu;
      ds[k] += -S(2) * dw * f.w[k] / f.s[k];  // w_k = s_k⁻²
    }
    // r = R_cᵀ x̂
    S dxh[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      dxh[r] = f.Rc[3 * r] * dr[0] + f.Rc[3 * r + 1] * dr[1] + f.Rc[3 * r + 2] * dr[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) dRc[3 * r + k] += f.xh[r] * dr[k];
    }
    // x̂ = x·it, it = t2^{-1/2}
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      dx[r] += dxh[r] * f.it;
      dit += dxh[r] * f.x[r];
    }
    const S dt2 = S(-0.5) * dit * f.it * f.it * f.it;
#pragma unroll
    for (int r = 0; r < 3; ++r) dx[r] += S(2) * f.x[r] * dt2;
  }

  // ---- x_c = W μ + t ; R_c = W R_q
#pragma unroll
  for (int k = 0; k < 3; ++k) dmu[k] += cam.R[k] * dx[0] + cam.R[3 + k] * dx[1] + cam.R[6 + k] * dx[2];
  S dRq[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) dRq[3 * r + k] = cam.R[r] * dRc[k] + cam.R[3 + r] * dRc[3 + k] + cam.R[6 + r] * dRc[6 + k];
  // R(q̂) → q̂ → raw q
  const S w = f.qn[0], a = f.qn[1], b = f.qn[2], c = f.qn[3];
  S dqn[4];
  dqn[0] = S(2) * (-c * dRq[1] + b * dRq[2] + c * dRq[3] - a * dRq[5] - b * dRq[6] + a * dRq[7]);
  dqn[1] = S(2) * (b * dRq[1] + c * dRq[2] + b * dRq[3] - S(2) * a * dRq[4] - w * dRq[5] + c * dRq[6] + w * dRq[7] -
                  S(2) * a * dRq[8]);
  dqn[2] = S(2) * (-S(2) * b * dRq[0] + a * dRq[1] + w * dRq[2] + a * dRq[3] + c * dRq[5] - w * dRq[6] + c * dRq[7] -
                  S(2) * b * dRq[8]);
  dqn[3] = S(2) * (-S(2) * c * dRq[0] - w * dRq[1] + a * dRq[2] + w * dRq[3] - S(2) * c * dRq[4] + b * dRq[5] +
                  a * dRq[6] + b * dRq[7]);
  const S qd = dqn[0] * w + dqn[1] * a + dqn[2] * b + dqn[3] * c;

  float d_o_raw = d_o;
  if (g.filter3d) {  // through s' = √(s² + f²), o' = o·Π s/s' back to the raw s, o (S23)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      ds[k] = ds[k] * (S)(f.s_raw[k] / f.s[k]) +
              (S)d_o * (S)f.o * ((S)1 / (S)f.s_raw[k] - (S)f.s_raw[k] / ((S)f.s[k] * (S)f.s[k]));
    d_o_raw = d_o * (f.o / f.o_raw);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    acc.dmu[k] += (float)dmu[k];
    acc.ds[k] += (float)ds[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) acc.dq[k] += (float)((dqn[k] - f.qn[k] * qd) * f.qinv);
  // α = min(α_max, o·G): d_o already excludes the clamp (K4)
  acc.dop += d_o_raw;
  return true;
}

// K5b, fp32, one thread per entry of the visible list (the ones that are not is_big)
// tiles (the others are K5b64's).
__global__ void __launch_bounds__(RD_K5_THREADS, RD_K5_MINB) k_preprocess_bwd(DevGauss g, DevCam cam, DevOpt opt,
                                                        const uint32_t* __restrict__ touched,
                                                        const uint32_t* __restrict__ vis, int64_t n_vis,
                                                        const G2D* __restrict__ g2d, DevGrads gr) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_vis) {
    const uint32_t i = vis[p];  // over K1's visible list: every thread has work
#ifndef RD_K5B_EARLY
#define RD_K5B_EARLY 1
#endif
    if (RD_K5B_EARLY) {
      // tiles_touched loaded beside the parameters and the 2-D gradient row (one round trip after
      // the id, not two); the few big Gaussians (K5b64's) compute and drop their result
      const bool big = is_big(touched[i], opt.tile);
      GradAcc acc;
      grad_zero(acc);
      if (geometry_backward<float>(g, i, cam, opt, g2d, acc) && !big) grad_flush(acc, gr, i);
    } else if (!is_big(touched[i], opt.tile)) {  // else K5b64's
      GradAcc acc;
      grad_zero(acc);
      if (geometry_backward<float>(g, i, cam, opt, g2d, acc)) grad_flush(acc, gr, i);
    }
  }
  // launched as K5b64's programmatic dependent (the two write disjoint rows and overlap):
  // do not complete before K5b64 has, so stream order after K5b still covers both
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// K5b64: the same chain rule in fp64 for the Gaussians of K1's big list.
__global__ void __launch_bounds__(128) k_preprocess_bwd64(DevGauss g, DevCam cam, DevOpt opt,
                                                          const uint32_t* __restrict__ big, int64_t n_big,
                                                          const G2D* __restrict__ g2d, DevGrads gr) {
  asm volatile("griddepcontrol.launch_dependents;");  // K5b may start now (disjoint rows)
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_big) return;
  GradAcc acc;
  grad_zero(acc);
  if (geometry_backward<double>(g, big[p], cam, opt, g2d, acc)) grad_flush(acc, gr, big[p]);
}

// The geometry parts of a round of views in one launch each (blockIdx.y = view): no tail and
// launch gap between the views' kernels. Same per-thread work as k_preprocess_bwd(64).
struct ViewsGeo {
  DevCam cam[kMaxBatchViews];
  const uint32_t* touched[kMaxBatchViews];
  const uint32_t* list[kMaxBatchViews];  // visible list (K5b) / big list (K5b64)
  int64_t n[kMaxBatchViews];
  const G2D* g2d[kMaxBatchViews];
};
__global__ void __launch_bounds__(RD_K5_THREADS, RD_K5_MINB) k_preprocess_bwd_geo_views(DevGauss g, DevOpt opt,
                                                                             const __grid_constant__ ViewsGeo vg,
                                                                             DevGrads gr) {
  const int v = (int)blockIdx.y;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < vg.n[v]) {
    const uint32_t i = vg.list[v][p];
    const bool big = is_big(vg.touched[v][i], opt.tile);
    GradAcc acc;
    grad_zero(acc);
    if (geometry_backward<float>(g, i, vg.cam[v], opt, vg.g2d[v], acc) && !big) grad_flush(acc, gr, i);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__global__ void __launch_bounds__(128) k_preprocess_bwd64_views(DevGauss g, DevOpt opt, const __grid_constant__ ViewsGeo vg,
                                                                DevGrads gr) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int v = (int)blockIdx.y;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= vg.n[v]) return;
  const uint32_t i = vg.list[v][p];
  GradAcc acc;
  grad_zero(acc);
  if (geometry_backward<double>(g, i, vg.cam[v], opt, vg.g2d[v], acc)) grad_flush(acc, gr, i);
}

// ---------------------------------------------------------------------------- K5, B views
// rd_preprocess_bwd_views: the views of a step share the Gaussians. The SH part of K5 — the
// HBM-bound one (per view it read each visible Gaussian's 192-B coefficient row and reduced
// into its 192-B gradient row: ~0.55 GB per C3 view) — runs ONCE for all the views: each
// Gaussian's row is read once, every view's colour gradient is accumulated on chip, and the
// gradient row gets one reduction. The geometry part (K5b / K5b64) stays per view: it is
// latency-bound on its gathers, and its per-(Gaussian, view) thread parallelism beats fusing
// (measured: a fused geometry pass, one thread looping over the views or lane groups with a
// shuffle reduction, was 1.5x slower than the per-view kernels).
struct ViewsBwd {
  int nv;
  DevCam cam[kMaxBatchViews];
  const uint32_t* touched[kMaxBatchViews];
  const G2D* g2d[kMaxBatchViews];
};

#ifndef RD_K5AV_TOUCHED_UNROLL
#define RD_K5AV_TOUCHED_UNROLL 1
#endif
#ifndef RD_K5AV_MINB
#define RD_K5AV_MINB 8  // ≤ 128 registers (16 warps per SM): 12 and 10 spilled and measured slower
#endif
// K5a over B views: as k_preprocess_bwd_sh_coop, but each warp owns 32 consecutive ids (the
// SH rows of a warp are one contiguous 6-KB block), copies the rows of the ids visible in any
// view once, and accumulates every view's SH and view-direction gradients before one
// reduction per row.
template <int DEG>
__global__ void __launch_bounds__(64, RD_K5AV_MINB) k_preprocess_bwd_sh_views(DevGauss g, DevOpt opt,
                                                                const __grid_constant__ ViewsBwd vb, DevGrads gr,
                                                                Counter* __restrict__ counters, bool set_sh) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int NV = 3 * K, NV4 = (NV + 3) / 4, P = NV4 + 1;
  __shared__ float4 s_coef[2][32 * P];
  __shared__ float4 s_grad[2][32 * P];
#ifndef RD_K5AV_PRE
#define RD_K5AV_PRE 2  // views whose colour gradients are prefetched into shared memory
#endif
  // the colour gradient (G2D f[1..3]) of the first RD_K5AV_PRE views, copied in with the SH rows
  // (cp.async: no registers) instead of one dependent load per view inside the view loop
  __shared__ float s_drgb[RD_K5AV_PRE > 0 ? 2 : 1][RD_K5AV_PRE > 0 ? RD_K5AV_PRE : 1][3][32];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned mask = 0u;
  if (id < g.n) {
#if RD_K5AV_TOUCHED_UNROLL
    // every view's load issued before the first use: one round trip, not one per view
    uint32_t t[kMaxBatchViews];
#pragma unroll
    for (int v = 0; v < kMaxBatchViews; ++v) t[v] = v < vb.nv ? vb.touched[v][id] : 0u;
#pragma unroll
    for (int v = 0; v < kMaxBatchViews; ++v) mask |= (t[v] > 0u ? 1u : 0u) << v;
#else
#pragma unroll 1
    for (int v = 0; v < vb.nv; ++v) mask |= (vb.touched[v][id] > 0u ? 1u : 0u) << v;
#endif
  }
  const unsigned vmask = __ballot_sync(0xffffffffu, mask != 0u);
  const int64_t base = id - lane;
  const int L4 = g.sh_coeffs * 3 / 4;  // global row pitch in float4
  // the warp's 32 rows: one block of 32·L4 float4 from here (32-bit offsets within it)
  float4* gsh4 = reinterpret_cast<float4*>(gr.sh) + base * L4;
  const int nrows = g.n - base < 32 ? (int)(g.n - base) : 32;  // rows of the warp that exist
  if (vmask == 0u) {  // warp-uniform: none of the 32 Gaussians is visible in any view
    if (set_sh) {  // set mode: their SH gradient rows are 0
      for (int f = lane; f < nrows * L4; f += 32) gsh4[f] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return;
  }
  if (counters && lane == 0) atomicAdd(counters + 4, (Counter)__popc(vmask));
  float4* sc = s_coef[warp];
  float4* sg = s_grad[warp];
  const float4* sh4 = reinterpret_cast<const float4*>(g.sh) + base * L4;
  if (L4 == NV4) {  // rows of exactly the active coefficients: the warp's block is contiguous
    const float4* src = sh4 + lane;
#pragma unroll
    for (int it = 0; it < NV4; ++it) {
      const unsigned f = (unsigned)(it * 32 + lane), row = f / (unsigned)NV4;
      if ((vmask >> row) & 1u) cp_async16(&sc[f + row], src + it * 32);
    }
  } else {
#pragma unroll
    for (int it = 0; it < NV4; ++it) {
      const int f = it * 32 + lane, row = f / NV4, c = f - row * NV4;
      if ((vmask >> row) & 1u) cp_async16(&sc[row * P + c], &sh4[row * L4 + c]);
    }
  }
  if (RD_K5AV_PRE > 0) {
#pragma unroll
    for (int v = 0; v < (RD_K5AV_PRE > 0 ? RD_K5AV_PRE : 1); ++v)
      if (v < vb.nv && ((mask >> v) & 1u)) {
        const float* f = vb.g2d[v][id].f + 1;
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async4(&s_drgb[warp][v][c][lane], f + c);
      }
  }
  cp_async_commit();
#pragma unroll
  for (int q = 0; q < NV4; ++q) sg[lane * P + q] = make_float4(0.f, 0.f, 0.f, 0.f);
  float mu0 = 0.f, mu1 = 0.f, mu2 = 0.f;
  if (mask) {
    mu0 = g.means[3 * id];
    mu1 = g.means[3 * id + 1];
    mu2 = g.means[3 * id + 2];
  }
  cp_async_wait<0>();
  __syncwarp();
  if (mask) {
    const float* coef = reinterpret_cast<const float*>(sc + lane * P);  // the row, read from shared memory
    float dmu[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
    for (int v = 0; v < vb.nv; ++v) {
      if (!((mask >> v) & 1u)) continue;
      const DevCam& cam = vb.cam[v];
      float d_rgb[3];
      if (v < RD_K5AV_PRE) {
#pragma unroll
        for (int c = 0; c < 3; ++c) d_rgb[c] = s_drgb[warp][v < RD_K5AV_PRE ? v : 0][c][lane];
      } else {
        const G2D* row = vb.g2d[v] + id;
        d_rgb[0] = row->f[1];
        d_rgb[1] = row->f[2];
        d_rgb[2] = row->f[3];
      }
      const float ex = mu0 - cam.campos[0], ey = mu1 - cam.campos[1], ez = mu2 - cam.campos[2];
      const float idl = rsqrtf(ex * ex + ey * ey + ez * ez);
      const float hx = ex * idl, hy = ey * idl, hz = ez * idl;
      float Y[16];
      sh_basis(hx, hy, hz, DEG, Y);
      float rgb[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) rgb[ch] += Y[k] * coef[k * 3 + ch];
      float drgb[3];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) drgb[ch] = rgb[ch] < 0.f ? 0.f : d_rgb[ch];  // clamp: zero grad
#pragma unroll
      for (int q = 0; q < NV4; ++q) {
        float d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) d[e] = (4 * q + e) < NV ? Y[(4 * q + e) / 3] * drgb[(4 * q + e) % 3] : 0.f;
        float4 a = sg[lane * P + q];
        a.x += d[0];
        a.y += d[1];
        a.z += d[2];
        a.w += d[3];
        sg[lane * P + q] = a;
      }
      float c16[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        c16[k] = k < K ? drgb[0] * coef[3 * k] + drgb[1] * coef[3 * k + 1] + drgb[2] * coef[3 * k + 2] : 0.f;
      float gx, gy, gz;
      sh_basis_grad(hx, hy, hz, DEG, c16, gx, gy, gz);
      const float dot = gx * hx + gy * hy + gz * hz;  // through the normalisation of dir
      dmu[0] += (gx - hx * dot) * idl;
      dmu[1] += (gy - hy * dot) * idl;
      dmu[2] += (gz - hz * dot) * idl;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) red_add(gr.means + 3 * id + k, dmu[k]);
  }
  __syncwarp();
  if (set_sh) {  // set mode: every row of the warp is written (0 where visible in no view), the
    // old values never read (the rows' 192-B read of the reduction disappears)
    if (nrows == 32 && L4 == NV4) {  // the usual case: the warp's rows are one contiguous block
      float4* dst = gsh4 + lane;
#pragma unroll
      for (int it = 0; it < NV4; ++it) {
        const unsigned f = (unsigned)(it * 32 + lane), row = f / (unsigned)NV4;
        dst[it * 32] = sg[f + row];  // row·P + c = f + row (P = NV4 + 1)
      }
      return;
    }
#pragma unroll
    for (int it = 0; it < NV4; ++it) {
      const int f = it * 32 + lane, row = f / NV4, c = f - row * NV4;
      if (row < nrows) gsh4[row * L4 + c] = sg[row * P + c];
    }
    // coefficients above the active degree get no gradient: 0
    if (L4 > NV4) {
      const int W = L4 - NV4;
      for (int f = lane; f < nrows * W; f += 32) {
        const int row = f / W, c = NV4 + (f - row * W);
        gsh4[row * L4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < NV4; ++it) {
    const int f = it * 32 + lane, row = f / NV4, c = f - row * NV4;
    if ((vmask >> row) & 1u) red_add4(&gsh4[row * L4 + c], sg[row * P + c]);
  }
}

__global__ void __launch_bounds__(256) k_g2d_to_f32(const G2D* __restrict__ g2d, int64_t n, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float* o = out + 16 * i;
#pragma unroll
  for (int k = 0; k < 5; ++k) o[k] = (float)g2d[i].m[k];
#pragma unroll
  for (int k = 0; k < 10; ++k) o[5 + k] = g2d[i].f[k];
  o[15] = 0.f;
}

// K5a (cooperative, rows of a multiple of 4 floats): each warp owns 32 VISIBLE Gaussians —
// 32 consecutive entries of K1's visible list — and moves their SH coefficient rows and
// SH gradient rows between HBM and shared
// memory cooperatively: each warp-wide 16-B load covers ~3 whole 192-B rows (full sectors,
// vs 32 scattered half-sectors for per-thread row loads), 2·NV4 loads per lane are in
// flight at once, and only visible rows are touched. Lane l then works on row l (pitch
// NV4+1 float4: conflict-free), and the updated gradient rows are stored back the same way.
template <int DEG>
__global__ void __launch_bounds__(64) k_preprocess_bwd_sh_coop(DevGauss g, DevCam cam, DevOpt opt,
                                                               const uint32_t* __restrict__ vis, int64_t n_vis,
                                                               const G2D* __restrict__ g2d, DevGrads gr) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int NV = 3 * K, NV4 = (NV + 3) / 4, P = NV4 + 1;
  __shared__ float4 s_coef[2][32 * P];
  __shared__ float4 s_grad[2][32 * P];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = p < n_vis;
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  if (vmask == 0) return;  // warp-uniform: past the end of the list
  const uint32_t id = valid ? vis[p] : 0u;
  const int64_t L4 = g.sh_coeffs * 3 / 4;  // global row pitch in float4
  float mu0 = 0.f, mu1 = 0.f, mu2 = 0.f, d_rgb[3] = {0.f, 0.f, 0.f};
  if (valid) {
    d_rgb[0] = g2d[id].f[1];
    d_rgb[1] = g2d[id].f[2];
    d_rgb[2] = g2d[id].f[3];
    mu0 = g.means[3 * (size_t)id];
    mu1 = g.means[3 * (size_t)id + 1];
    mu2 = g.means[3 * (size_t)id + 2];
  }
  float4* sc = s_coef[warp];
  float4* sg = s_grad[warp];
  const float4* sh4 = reinterpret_cast<const float4*>(g.sh);
  float4* gsh4 = reinterpret_cast<float4*>(gr.sh);
#pragma unroll
  for (int it = 0; it < NV4; ++it) {  // all 2·NV4 copies per lane in flight at once
    const int f = it * 32 + lane, row = f / NV4, c = f - row * NV4;
    const uint32_t rid = __shfl_sync(0xffffffffu, id, row);
    if ((vmask >> row) & 1u) cp_async16(&sc[row * P + c], &sh4[(int64_t)rid * L4 + c]);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  if (valid) {
    float ex = mu0 - cam.campos[0], ey = mu1 - cam.campos[1], ez = mu2 - cam.campos[2];
    const float idl = rsqrtf(ex * ex + ey * ey + ez * ez);
    const float hx = ex * idl, hy = ey * idl, hz = ez * idl;
    float Y[16];
    sh_basis(hx, hy, hz, DEG, Y);
    float coef[NV4 * 4];
#pragma unroll
    for (int q = 0; q < NV4; ++q) {
      const float4 v = sc[lane * P + q];
      coef[4 * q] = v.x;
      coef[4 * q + 1] = v.y;
      coef[4 * q + 2] = v.z;
      coef[4 * q + 3] = v.w;
    }
    float rgb[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) rgb[ch] += Y[k] * coef[k * 3 + ch];
    float drgb[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) drgb[ch] = rgb[ch] < 0.f ? 0.f : d_rgb[ch];  // clamp: zero grad
#pragma unroll
    for (int q = 0; q < NV4; ++q) {
      float d[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) d[e] = (4 * q + e) < NV ? Y[(4 * q + e) / 3] * drgb[(4 * q + e) % 3] : 0.f;
      sg[lane * P + q] = make_float4(d[0], d[1], d[2], d[3]);
    }
    float c16[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      c16[k] = k < K ? drgb[0] * coef[3 * k] + drgb[1] * coef[3 * k + 1] + drgb[2] * coef[3 * k + 2] : 0.f;
    float gx, gy, gz;
    sh_basis_grad(hx, hy, hz, DEG, c16, gx, gy, gz);
    const float dot = gx * hx + gy * hy + gz * hz;  // through the normalisation of dir
    red_add(gr.means + 3 * (size_t)id, (gx - hx * dot) * idl);
    red_add(gr.means + 3 * (size_t)id + 1, (gy - hy * dot) * idl);
    red_add(gr.means + 3 * (size_t)id + 2, (gz - hz * dot) * idl);
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < NV4; ++it) {
    const int f = it * 32 + lane, row = f / NV4, c = f - row * NV4;
    const uint32_t rid = __shfl_sync(0xffffffffu, id, row);
    if ((vmask >> row) & 1u) red_add4(&gsh4[(int64_t)rid * L4 + c], sg[row * P + c]);
  }
}


}  // namespace

void launch_preprocess_fwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, int tiles_x, Record* rec,
                           uint2* rect, uint32_t* tiles_touched, uint32_t* dkey, uint32_t* count,
                           uint32_t* vis, uint32_t* big, G2D* g2d, Counter* counters, cudaStream_t s) {
  if (g.n == 0) return;
  const int threads = RD_K1_THREADS;
  const unsigned blocks = (unsigned)((g.n + threads - 1) / threads);
#define RD_K1(D)                                                                                                 \
  k_preprocess_fwd<D><<<blocks, threads, 0, s>>>(g, cam, opt, tiles_x, rec, rect, tiles_touched, dkey, \
                                                 count, vis, big, g2d, counters)
  switch (opt.sh_degree) {
    case 0: RD_K1(0); break;
    case 1: RD_K1(1); break;
    case 2: RD_K1(2); break;
    default: RD_K1(3); break;
  }
#undef RD_K1
}

void launch_preprocess_fwd_views(const DevGauss& g, const DevOpt& opt, const K1Views& kv, cudaStream_t s) {
  if (g.n == 0 || kv.nv <= 0) return;
  const int threads = RD_K1_THREADS;
  const unsigned blocks = (unsigned)((g.n + threads - 1) / threads);
  switch (opt.sh_degree) {
    case 0: k_preprocess_fwd_views<0><<<blocks, threads, 0, s>>>(g, opt, kv); break;
    case 1: k_preprocess_fwd_views<1><<<blocks, threads, 0, s>>>(g, opt, kv); break;
    case 2: k_preprocess_fwd_views<2><<<blocks, threads, 0, s>>>(g, opt, kv); break;
    default: k_preprocess_fwd_views<3><<<blocks, threads, 0, s>>>(g, opt, kv); break;
  }
}

void launch_preprocess_bwd(const DevGauss& g, const DevCam& cam, const DevOpt& opt, const uint32_t* tiles_touched,
                           const uint32_t* vis, int64_t n_vis, const uint32_t* big, int64_t n_big, const G2D* g2d,
                           DevGrads grads, cudaStream_t s, int parts) {
  if (g.n == 0) return;
  const int threads = 128;
  const unsigned blocks = (unsigned)((g.n + threads - 1) / threads);
  if (!(parts & kK5Sh)) {
  } else if ((g.sh_coeffs * 3) % 4 == 0) {
    const unsigned cblocks = (unsigned)((n_vis + 63) / 64);
#define RD_K5A(D) \
  if (cblocks) k_preprocess_bwd_sh_coop<D><<<cblocks, 64, 0, s>>>(g, cam, opt, vis, n_vis, g2d, grads)
    switch (opt.sh_degree) {
      case 0: RD_K5A(0); break;
      case 1: RD_K5A(1); break;
      case 2: RD_K5A(2); break;
      default: RD_K5A(3); break;
    }
#undef RD_K5A
  } else {
#define RD_K5A(D) k_preprocess_bwd_sh<D><<<blocks, threads, 0, s>>>(g, cam, opt, tiles_touched, g2d, grads)
    switch (opt.sh_degree) {
      case 0: RD_K5A(0); break;
      case 1: RD_K5A(1); break;
      case 2: RD_K5A(2); break;
      default: RD_K5A(3); break;
    }
#undef RD_K5A
  }
  // K5b64 (few, fp64, latency-bound) first; K5b as its programmatic dependent, so the two
  // run side by side instead of K5b64's ~11 µs trailing K5b
  if (!(parts & kK5Geometry)) return;
  if (n_big > 0)
    k_preprocess_bwd64<<<(unsigned)((n_big + 127) / 128), 128, 0, s>>>(g, cam, opt, big, n_big, g2d, grads);
  if (n_vis > 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((n_vis + RD_K5_THREADS - 1) / RD_K5_THREADS));
    cfg.blockDim = dim3(RD_K5_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = n_big > 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_preprocess_bwd, g, cam, opt, tiles_touched, vis, n_vis, g2d, grads);
  }
}

void launch_preprocess_bwd_views(const DevGauss& g, const DevOpt& opt, int nv, const DevCam* cams,
                                 const uint32_t* const* touched, const G2D* const* g2d, const uint32_t* const* vis,
                                 const int64_t* n_vis, const uint32_t* const* big, const int64_t* n_big,
                                 DevGrads grads, Counter* counters, cudaStream_t s, int parts) {
  if (g.n == 0 || nv <= 0) return;
  ViewsBwd vb{};
  vb.nv = nv;
  for (int v = 0; v < nv; ++v) {
    vb.cam[v] = cams[v];
    vb.touched[v] = touched[v];
    vb.g2d[v] = g2d[v];
  }
  if (!(parts & kK5Sh)) {
  } else if ((g.sh_coeffs * 3) % 4 == 0) {
    const unsigned cblocks = (unsigned)((g.n + 63) / 64);
#define RD_K5AV(D) k_preprocess_bwd_sh_views<D><<<cblocks, 64, 0, s>>>(g, opt, vb, grads, counters, (parts & kK5ShSet) != 0)
    switch (opt.sh_degree) {
      case 0: RD_K5AV(0); break;
      case 1: RD_K5AV(1); break;
      case 2: RD_K5AV(2); break;
      default: RD_K5AV(3); break;
    }
#undef RD_K5AV
  } else {  // rows not 16-B multiples: the per-view SH kernel, once per view
    const unsigned blocks = (unsigned)((g.n + 127) / 128);
    for (int v = 0; v < nv; ++v) {
#define RD_K5A(D) k_preprocess_bwd_sh<D><<<blocks, 128, 0, s>>>(g, cams[v], opt, touched[v], g2d[v], grads)
      switch (opt.sh_degree) {
        case 0: RD_K5A(0); break;
        case 1: RD_K5A(1); break;
        case 2: RD_K5A(2); break;
        default: RD_K5A(3); break;
      }
#undef RD_K5A
    }
  }
  // geometry per view: its fp64 big list, then the fp32 pass over its visible list as the big
  // list's programmatic dependent (rows are only ever added by reductions)
  if (!(parts & kK5Geometry)) return;
#ifndef RD_K5_GEO_BATCH
#define RD_K5_GEO_BATCH 1
#endif
  if (RD_K5_GEO_BATCH) {
    ViewsGeo vb64{}, vbv{};
    int64_t max_big = 0, max_vis = 0;
    for (int v = 0; v < nv; ++v) {
      vb64.cam[v] = vbv.cam[v] = cams[v];
      vb64.touched[v] = vbv.touched[v] = touched[v];
      vb64.g2d[v] = vbv.g2d[v] = g2d[v];
      vb64.list[v] = big[v];
      vb64.n[v] = n_big[v];
      vbv.list[v] = vis[v];
      vbv.n[v] = n_vis[v];
      max_big = n_big[v] > max_big ? n_big[v] : max_big;
      max_vis = n_vis[v] > max_vis ? n_vis[v] : max_vis;
    }
    if (max_big > 0)
      k_preprocess_bwd64_views<<<dim3((unsigned)((max_big + 127) / 128), (unsigned)nv), 128, 0, s>>>(g, opt, vb64, grads);
    if (max_vis > 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)((max_vis + RD_K5_THREADS - 1) / RD_K5_THREADS), (unsigned)nv);
      cfg.blockDim = dim3(RD_K5_THREADS);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = max_big > 0 ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_preprocess_bwd_geo_views, g, opt, vbv, grads);
    }
    return;
  }
  for (int v = 0; v < nv; ++v) {
    if (n_big[v] > 0)
      k_preprocess_bwd64<<<(unsigned)((n_big[v] + 127) / 128), 128, 0, s>>>(g, cams[v], opt, big[v], n_big[v], g2d[v],
                                                                          grads);
    if (n_vis[v] > 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)((n_vis[v] + RD_K5_THREADS - 1) / RD_K5_THREADS));
      cfg.blockDim = dim3(RD_K5_THREADS);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = n_big[v] > 0 ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_preprocess_bwd, g, cams[v], opt, touched[v], vis[v], n_vis[v], g2d[v], grads);
    }
  }
}

void launch_g2d_to_f32(const G2D* g2d, int64_t n, float* out, cudaStream_t s) {
  if (n == 0) return;
  k_g2d_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g2d, n, out);
}

}  // namespace rade
