/*
 * RaDe-GS CPU ORACLE (arXiv 2406.01467) — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2406_01467_b200/) never does:
 * it shares no code, header, helper or constant table with this file.
 *
 * What it computes: a plain, slow, per-pixel brute-force renderer in fp64 that follows
 * the paper's method section in the paper's order and notation (PAPER.md lines cited
 * as PAPER:n; readings of silent / garbled points are DESIGN.md §"Readings" S1..S20):
 *
 *   per Gaussian   Σ = R S Sᵀ Rᵀ                                 PAPER:408 (Eq.1)
 *                  x_c = W μ + t ; (u_c, v_c) pinhole ; t_c = ‖x_c‖ PAPER:486-490, S2, S4
 *                  J = ∂(u, v, t)/∂x at x_c                      PAPER:417, 488 (S2)
 *                  Σ′ = J W Σ Wᵀ Jᵀ                              PAPER:413-416 (Eq.2)
 *                  2D covariance = Σ′[0:2,0:2] (+ dilation, S5)
 *                  q̂ = v′ᵀΣ′⁻¹ / (v′ᵀΣ′⁻¹v′), v′ = (0,0,1)       PAPER:519-522 (Eq.13)
 *                  p̂ = (z_c/t_c) q̂ ; q, p = first two entries
 *                  n′ = −(q, 1)ᵀ ; n = Jᵀ n′ / ‖Jᵀ n′‖             PAPER:617-627 (Eq.21-22)
 *                  colour from SH at the Gaussian's view dir      PAPER:426 (S14)
 *   order          all surviving Gaussians by centre depth        PAPER:422, 440 (S7)
 *   per pixel      α = min(α_max, o·exp(−½ Δᵀ conic Δ))           PAPER:406, 425 (S1, S8)
 *                  t* = v′ᵀΣ′⁻¹(u_c − u_o) / (v′ᵀΣ′⁻¹v′)          PAPER:514-517 (Eq.11-12),
 *                                                                 evaluated PER PIXEL (S13)
 *                  d = (z_c/t_c) t*                               PAPER:527-531 (Eq.15, S12)
 *                  c = Σ c_i α_i Π_{j<i}(1 − α_j)                 PAPER:423-425 (Eq.3)
 *                  normal map N = Σ ω_i n_i (unnormalised)        PAPER:30 (S10)
 *                  median depth = d of the first blended splat at
 *                  which T crosses median_T                       PAPER:30 (S9)
 *                  depth distortion L_d = Σ_i Σ_j ω_i ω_j (d_i − d_j)² over the
 *                  blended splats, ω detached in the gradient     PAPER:635-639 (S21)
 *   gradients      forward-mode dual numbers through all of the above (exact derivative of
 *                  this definition; independent of the GPU's hand-derived backward).
 *
 * Scalar type is templated: double for values, Dual<59> for gradients. No blocking,
 * tiling, fusion or reordering: every pixel walks the whole globally sorted list.
 * The only fp32 arithmetic is the sort key z_key (contract S7: both sides order by the
 * same fp32 value so that the ordering decision is taken in the same precision).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// dual slots per Gaussian: μ 3, s 3, q 4, o 1, sh 16*3 (the 59 parameters), then 2 for an
// offset of the projected centre (u_c, v_c) — zero-valued inputs whose derivative is the
// screen-space ("means2d") gradient, the other per-splat quantities held fixed
constexpr int NP = 61;

// ------------------------------------------------------------------ dual numbers
struct Dual {
  double v;
  double d[NP];
  Dual() : v(0.0) { std::memset(d, 0, sizeof(d)); }
  Dual(double x) : v(x) { std::memset(d, 0, sizeof(d)); }
};
inline double val(double x) { return x; }
inline double val(const Dual& x) { return x.v; }

inline Dual operator+(const Dual& a, const Dual& b) { Dual r(a.v + b.v); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] + b.d[k]; return r; }
inline Dual operator-(const Dual& a, const Dual& b) { Dual r(a.v - b.v); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] - b.d[k]; return r; }
inline Dual operator*(const Dual& a, const Dual& b) { Dual r(a.v * b.v); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] * b.v + a.v * b.d[k]; return r; }
inline Dual operator/(const Dual& a, const Dual& b) { Dual r(a.v / b.v); double ib = 1.0 / b.v; for (int k = 0; k < NP; ++k) r.d[k] = (a.d[k] - r.v * b.d[k]) * ib; return r; }
inline Dual operator+(const Dual& a, double b) { Dual r = a; r.v += b; return r; }
inline Dual operator+(double a, const Dual& b) { return b + a; }
inline Dual operator-(const Dual& a, double b) { Dual r = a; r.v -= b; return r; }
inline Dual operator-(double a, const Dual& b) { Dual r(a - b.v); for (int k = 0; k < NP; ++k) r.d[k] = -b.d[k]; return r; }
inline Dual operator*(const Dual& a, double b) { Dual r(a.v * b); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] * b; return r; }
inline Dual operator*(double a, const Dual& b) { return b * a; }
inline Dual operator/(const Dual& a, double b) { return a * (1.0 / b); }
inline Dual operator/(double a, const Dual& b) { return Dual(a) / b; }
inline Dual operator-(const Dual& a) { return 0.0 - a; }
inline Dual& operator+=(Dual& a, const Dual& b) { a = a + b; return a; }
inline Dual& operator+=(Dual& a, double b) { a.v += b; return a; }
inline Dual exp(const Dual& a) { Dual r(std::exp(a.v)); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] * r.v; return r; }
inline Dual sqrt(const Dual& a) { Dual r(std::sqrt(a.v)); double h = 0.5 / r.v; for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] * h; return r; }
inline Dual log(const Dual& a) { Dual r(std::log(a.v)); for (int k = 0; k < NP; ++k) r.d[k] = a.d[k] / a.v; return r; }
using std::exp;
using std::log;
using std::sqrt;

// ------------------------------------------------------------------ inputs
struct Cam {
  double fx, fy, cx, cy;
  int W, H;
  double R[9], t[3];
  double znear;
};
struct Opt {
  double alpha_min, alpha_max, T_min, median_T, dilation;
  double bg[3];
  int sh_degree;
  double eps[5];  // ambiguity-flag bands F1..F5 (see or_render)
  double guard_band;  // reading S6b: 0 = off; g > 0: cull centres outside the band
};

// SH basis constants of the 3DGS real-SH convention (reading S14; PAPER:426 only says
// "computed from its spherical harmonics coefficients and viewing direction").
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};

template <class S>
void sh_basis(const S dir[3], S Y[16]) {
  const S &x = dir[0], &y = dir[1], &z = dir[2];
  Y[0] = S(SH_C0);
  Y[1] = -SH_C1 * y;
  Y[2] = SH_C1 * z;
  Y[3] = -SH_C1 * x;
  S xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = SH_C2[0] * xy;
  Y[5] = SH_C2[1] * yz;
  Y[6] = SH_C2[2] * (2.0 * zz - xx - yy);
  Y[7] = SH_C2[3] * xz;
  Y[8] = SH_C2[4] * (xx - yy);
  Y[9] = SH_C3[0] * y * (3.0 * xx - yy);
  Y[10] = SH_C3[1] * xy * z;
  Y[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
  Y[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  Y[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
  Y[14] = SH_C3[5] * z * (xx - yy);
  Y[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

// Full per-Gaussian projection (everything the pins look at).
template <class S>
struct PG {
  bool valid = false;
  float zkey = 0.f;
  S x[3], z, tc, u, v;
  S Sigma[9], Sc[9], J[9], Sp[9], Spi[9];
  S A2[3];      // dilated 2D covariance (a, b, c)
  S conic[3];   // its inverse (a, b, c)
  S qhat[3], q[2], p[2], n[3];
  S rgb[3];
  bool rgb_clamped[3] = {false, false, false};
  S o;
  double ndotx = 0.0;  // n · x̂_c (grazing measure, F5)
};

template <class S>
void mat3mul(const S* A, const S* B, S* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      S s = A[3 * i] * B[j];
      s = s + A[3 * i + 1] * B[3 + j];
      s = s + A[3 * i + 2] * B[6 + j];
      C[3 * i + j] = s;
    }
}
template <class S>
void transpose3(const S* A, S* T) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * j + i] = A[3 * i + j];
}
// explicit inverse by adjugate / determinant (fp64)
template <class S>
bool inverse3(const S* m, S* inv) {
  S c00 = m[4] * m[8] - m[5] * m[7];
  S c01 = m[5] * m[6] - m[3] * m[8];
  S c02 = m[3] * m[7] - m[4] * m[6];
  S det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  if (!(val(det) != 0.0) || !std::isfinite(val(det))) return false;
  S id = 1.0 / det;
  inv[0] = c00 * id;
  inv[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  inv[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  inv[3] = c01 * id;
  inv[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  inv[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  inv[6] = c02 * id;
  inv[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  inv[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  return true;
}

struct SceneIn {
  int64_t n;
  const double *means, *scales, *rot, *opac, *sh;  // SoA, see scenegen
  int sh_coeffs;                                   // K = (deg+1)^2 stored per channel
};

template <class S>
void load_params(const SceneIn& sc, int64_t i, S P[NP]) {
  int64_t n = sc.n;
  for (int k = 0; k < 3; ++k) P[k] = S(sc.means[k * n + i]);
  for (int k = 0; k < 3; ++k) P[3 + k] = S(sc.scales[k * n + i]);
  for (int k = 0; k < 4; ++k) P[6 + k] = S(sc.rot[k * n + i]);
  P[10] = S(sc.opac[i]);
  for (int k = 0; k < 48; ++k) P[11 + k] = S(0.0);
  for (int k = 0; k < sc.sh_coeffs * 3; ++k) P[11 + k] = S(sc.sh[k * n + i]);
  P[59] = S(0.0);  // centre offsets (means2d slots)
  P[60] = S(0.0);
}

// Contract S7: z_key = fmaf(W20, μx, fmaf(W21, μy, fmaf(W22, μz, t2))) in IEEE fp32.
float zkey_of(const Cam& cam, float mx, float my, float mz) {
  return std::fmaf((float)cam.R[6], mx, std::fmaf((float)cam.R[7], my, std::fmaf((float)cam.R[8], mz, (float)cam.t[2])));
}

// Reading S6b (optional, off unless g = opt.guard_band > 0): the centre must
// project into the guard band of the image, u_c ∈ [−g W, (1+g) W] and v_c ∈ [−g H, (1+g) H],
// decided in fp32 as fx·x_k ∈ [g_u0·z_k, g_u1·z_k] (and likewise for y) with x_k, y_k formed
// like z_k and g_u0 = float(−g W − cx), g_u1 = float((1+g) W − cx), ... rounded once from double.
bool in_guard_band(const Cam& cam, double g, float mx, float my, float mz, float zk) {
  const float xk = std::fmaf((float)cam.R[0], mx, std::fmaf((float)cam.R[1], my, std::fmaf((float)cam.R[2], mz, (float)cam.t[0])));
  const float yk = std::fmaf((float)cam.R[3], mx, std::fmaf((float)cam.R[4], my, std::fmaf((float)cam.R[5], mz, (float)cam.t[1])));
  const float gu0 = (float)(-g * cam.W - cam.cx), gu1 = (float)((1.0 + g) * cam.W - cam.cx);
  const float gv0 = (float)(-g * cam.H - cam.cy), gv1 = (float)((1.0 + g) * cam.H - cam.cy);
  const float fu = (float)cam.fx * xk, fv = (float)cam.fy * yk;
  return fu >= gu0 * zk && fu <= gu1 * zk && fv >= gv0 * zk && fv <= gv1 * zk;
}

template <class S>
bool project(const S P[NP], const double raw[11], const Cam& cam, const Opt& opt, PG<S>& g) {
  g.valid = false;
  // validity (cull rules): finite inputs, s > 0, |q| > 0
  for (int k = 0; k < 11; ++k)
    if (!std::isfinite(raw[k])) return false;
  if (!(raw[3] > 0.0 && raw[4] > 0.0 && raw[5] > 0.0)) return false;
  double qn2 = raw[6] * raw[6] + raw[7] * raw[7] + raw[8] * raw[8] + raw[9] * raw[9];
  if (!(qn2 > 0.0)) return false;
  g.zkey = zkey_of(cam, (float)raw[0], (float)raw[1], (float)raw[2]);
  if (!(g.zkey > (float)cam.znear)) return false;
  if (opt.guard_band > 0.0 && !in_guard_band(cam, opt.guard_band, (float)raw[0], (float)raw[1], (float)raw[2], g.zkey))
    return false;
  if (!(raw[10] >= opt.alpha_min)) return false;
  g.o = P[10];

  // Σ = R S Sᵀ Rᵀ, R from the normalised quaternion (w, x, y, z) (S15)
  S qn = sqrt(P[6] * P[6] + P[7] * P[7] + P[8] * P[8] + P[9] * P[9]);
  S w = P[6] / qn, a = P[7] / qn, b = P[8] / qn, c = P[9] / qn;
  S Rq[9] = {1.0 - 2.0 * (b * b + c * c), 2.0 * (a * b - w * c), 2.0 * (a * c + w * b),
             2.0 * (a * b + w * c), 1.0 - 2.0 * (a * a + c * c), 2.0 * (b * c - w * a),
             2.0 * (a * c - w * b), 2.0 * (b * c + w * a), 1.0 - 2.0 * (a * a + b * b)};
  S Sm[9] = {P[3], S(0.0), S(0.0), S(0.0), P[4], S(0.0), S(0.0), S(0.0), P[5]};
  S RS[9], RSt[9];
  mat3mul(Rq, Sm, RS);
  transpose3(RS, RSt);
  mat3mul(RS, RSt, g.Sigma);

  // camera space: x_c = W μ + t
  for (int i = 0; i < 3; ++i) g.x[i] = cam.R[3 * i] * P[0] + cam.R[3 * i + 1] * P[1] + cam.R[3 * i + 2] * P[2] + cam.t[i];
  g.z = g.x[2];
  g.tc = sqrt(g.x[0] * g.x[0] + g.x[1] * g.x[1] + g.x[2] * g.x[2]);
  g.u = cam.fx * g.x[0] / g.z + cam.cx + P[59];  // + 0: carries d/du_c (means2d)
  g.v = cam.fy * g.x[1] / g.z + cam.cy + P[60];

  // J = ∂(u, v, t)/∂x  (reading S2: t = ‖x‖)
  S z2 = g.z * g.z;
  g.J[0] = cam.fx / g.z; g.J[1] = S(0.0); g.J[2] = -cam.fx * g.x[0] / z2;
  g.J[3] = S(0.0); g.J[4] = cam.fy / g.z; g.J[5] = -cam.fy * g.x[1] / z2;
  g.J[6] = g.x[0] / g.tc; g.J[7] = g.x[1] / g.tc; g.J[8] = g.x[2] / g.tc;

  // Σ′ = J W Σ Wᵀ Jᵀ (Eq.2)
  S Wm[9], Wt[9], T1[9], T2[9], Jt[9];
  for (int k = 0; k < 9; ++k) Wm[k] = S(cam.R[k]);
  transpose3(Wm, Wt);
  mat3mul(Wm, g.Sigma, T1);
  mat3mul(T1, Wt, g.Sc);
  mat3mul(g.J, g.Sc, T2);
  transpose3(g.J, Jt);
  mat3mul(T2, Jt, g.Sp);

  // 2D covariance = top-left 2x2 of Σ′ + dilation h·I (reading S5, α only)
  g.A2[0] = g.Sp[0] + opt.dilation;
  g.A2[1] = g.Sp[1];
  g.A2[2] = g.Sp[4] + opt.dilation;
  S det = g.A2[0] * g.A2[2] - g.A2[1] * g.A2[1];
  if (!(val(det) > 0.0)) return false;
  g.conic[0] = g.A2[2] / det;
  g.conic[1] = -g.A2[1] / det;
  g.conic[2] = g.A2[0] / det;

  // q̂ = v′ᵀΣ′⁻¹ / (v′ᵀΣ′⁻¹v′) (Eq.13), Σ′⁻¹ by explicit inverse
  if (!inverse3(g.Sp, g.Spi)) return false;
  for (int k = 0; k < 3; ++k) g.qhat[k] = g.Spi[6 + k] / g.Spi[8];
  g.q[0] = g.qhat[0];
  g.q[1] = g.qhat[1];
  // p̂ = (z_c/t_c) q̂, p = first two entries
  g.p[0] = (g.z / g.tc) * g.q[0];
  g.p[1] = (g.z / g.tc) * g.q[1];
  // n′ = −(q, 1)ᵀ; n = Jᵀ n′ normalised
  S np_[3] = {-g.q[0], -g.q[1], S(-1.0)};
  S nn[3];
  for (int j = 0; j < 3; ++j) nn[j] = g.J[j] * np_[0] + g.J[3 + j] * np_[1] + g.J[6 + j] * np_[2];
  S nl = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
  for (int j = 0; j < 3; ++j) g.n[j] = nn[j] / nl;
  g.ndotx = (val(g.n[0]) * val(g.x[0]) + val(g.n[1]) * val(g.x[1]) + val(g.n[2]) * val(g.x[2])) / val(g.tc);

  // colour from SH (reading S14): dir = normalize(μ − campos), campos = −Wᵀt
  double campos[3];
  for (int i = 0; i < 3; ++i) campos[i] = -(cam.R[i] * cam.t[0] + cam.R[3 + i] * cam.t[1] + cam.R[6 + i] * cam.t[2]);
  S dir[3] = {P[0] - campos[0], P[1] - campos[1], P[2] - campos[2]};
  S dl = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
  for (int i = 0; i < 3; ++i) dir[i] = dir[i] / dl;
  S Y[16];
  sh_basis(dir, Y);
  int K = (opt.sh_degree + 1) * (opt.sh_degree + 1);
  for (int ch = 0; ch < 3; ++ch) {
    S s = S(0.5);
    for (int k = 0; k < K; ++k) s = s + Y[k] * P[11 + k * 3 + ch];
    g.rgb_clamped[ch] = !(val(s) >= 0.0);
    g.rgb[ch] = g.rgb_clamped[ch] ? S(0.0) : s;
  }
  g.valid = true;
  return true;
}

// ------------------------------------------------------------------ per-pixel composite
template <class S>
struct Splat {  // what the per-pixel loop reads (a compact copy of PG)
  S u, v, o, conic[3], rgb[3], n[3], z, tc, r2[3];  // r2 = third row of Σ′⁻¹
  double ndotx;
  float zkey;
  int64_t id;
};
template <class S>
Splat<S> compact(const PG<S>& g, int64_t id) {
  Splat<S> s;
  s.u = g.u; s.v = g.v; s.o = g.o;
  for (int k = 0; k < 3; ++k) { s.conic[k] = g.conic[k]; s.rgb[k] = g.rgb[k]; s.n[k] = g.n[k]; s.r2[k] = g.Spi[6 + k]; }
  s.z = g.z; s.tc = g.tc; s.ndotx = g.ndotx; s.zkey = g.zkey; s.id = id;
  return s;
}

template <class S>
struct Pix {
  S T, C[3], N[3], D;
  bool Dset = false, done = false;
  int nblend = 0;
  int64_t median_id = -1;
  uint8_t flags = 0;
  double median_ndotx = 1.0;
  std::vector<double> wl;  // ω_i of the blended splats (values only: detached, S21)
  std::vector<S> dl;       // their per-pixel depths d_i
};

// Depth distortion: the plain double sum over the blended splats.
template <class S>
S distortion(const Pix<S>& px) {
  S L = S(0.0);
  for (size_t i = 0; i < px.dl.size(); ++i)
    for (size_t j = 0; j < px.dl.size(); ++j) {
      S dd = px.dl[i] - px.dl[j];
      L = L + (px.wl[i] * px.wl[j]) * (dd * dd);
    }
  return L;
}
template <class S>
void pix_init(Pix<S>& px) {
  px.T = S(1.0);
  for (int k = 0; k < 3; ++k) { px.C[k] = S(0.0); px.N[k] = S(0.0); }
  px.D = S(0.0);
}
template <class SS, class SG>
void promote(const Pix<SG>& a, Pix<SS>& b) {
  b.T = SS(val(a.T));
  for (int k = 0; k < 3; ++k) { b.C[k] = SS(val(a.C[k])); b.N[k] = SS(val(a.N[k])); }
  b.D = SS(val(a.D));
  b.Dset = a.Dset; b.done = a.done; b.nblend = a.nblend; b.median_id = a.median_id; b.flags = a.flags;
  b.median_ndotx = a.median_ndotx;
  b.wl = a.wl;
  b.dl.clear();
  for (const auto& d : a.dl) b.dl.push_back(SS(val(d)));
}

// One splat against one pixel, front to back (Eq.3; readings S1, S8, S9).
// Returns false when the pixel terminates (stop rule).
template <class SS, class SG>
bool blend(Pix<SS>& px, const Splat<SG>& s, double u, double v, const Opt& opt) {
  SG du = s.u - u, dv = s.v - v;  // Δ = centre − pixel
  SG power = -0.5 * (s.conic[0] * du * du + 2.0 * s.conic[1] * du * dv + s.conic[2] * dv * dv);
  double lna = std::log(val(s.o)) + val(power);
  if (std::fabs(lna - std::log(opt.alpha_min)) < opt.eps[0]) px.flags |= 1;
  SG G = exp(power);
  SG a_raw = s.o * G;
  bool clamp = val(a_raw) > opt.alpha_max;
  SG alpha = clamp ? SG(opt.alpha_max) : a_raw;
  if (val(alpha) < opt.alpha_min) return true;  // skipped
  if (std::fabs(lna - std::log(opt.alpha_max)) < opt.eps[1]) px.flags |= 2;
  SS Tn = px.T * (1.0 - alpha);
  if (std::fabs(val(Tn) / opt.T_min - 1.0) < opt.eps[2]) px.flags |= 4;
  if (val(Tn) < opt.T_min) { px.done = true; return false; }
  if (std::fabs(val(Tn) - opt.median_T) < opt.eps[3]) px.flags |= 8;
  // t* = v′ᵀΣ′⁻¹(u_c − u_o)/(v′ᵀΣ′⁻¹v′), u_c − u_o = (Δu, Δv, t_c)
  SG tstar = (s.r2[0] * du + s.r2[1] * dv + s.r2[2] * s.tc) / s.r2[2];
  SG d = (s.z / s.tc) * tstar;  // d = cosθ_c t* = (z_c/t_c) t*
  SS w = alpha * px.T;
  for (int k = 0; k < 3; ++k) { px.C[k] += w * s.rgb[k]; px.N[k] += w * s.n[k]; }
  px.wl.push_back(val(w));
  px.dl.push_back(SS(0.0) + d);
  if (!px.Dset && val(px.T) > opt.median_T && val(Tn) <= opt.median_T) {
    px.D = SS(0.0) + d;
    px.Dset = true;
    px.median_id = s.id;
    px.median_ndotx = s.ndotx;
    if (std::fabs(s.ndotx) < opt.eps[4]) px.flags |= 16;
  }
  px.T = Tn;
  px.nblend++;
  return true;
}

struct Prepared {
  std::vector<Splat<double>> splats;  // globally sorted by (z_key, id)
  std::vector<PG<double>> full;       // indexed by Gaussian id (only if keep_full)
  std::vector<int64_t> pos_of;        // position in sorted order, −1 if culled
};

void prepare(const SceneIn& sc, const Cam& cam, const Opt& opt, Prepared& pr) {
  int64_t n = sc.n;
  std::vector<Splat<double>> tmp(n);
  std::vector<char> ok(n, 0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double P[NP], raw[11];
    load_params(sc, i, P);
    for (int k = 0; k < 11; ++k) raw[k] = P[k];
    PG<double> g;
    if (project(P, raw, cam, opt, g)) { tmp[i] = compact(g, i); ok[i] = 1; }
  }
  pr.splats.clear();
  for (int64_t i = 0; i < n; ++i)
    if (ok[i]) pr.splats.push_back(tmp[i]);
  // order: centre depth ascending, ties by index (reading S7)
  std::sort(pr.splats.begin(), pr.splats.end(), [](const Splat<double>& a, const Splat<double>& b) {
    if (a.zkey != b.zkey) return a.zkey < b.zkey;
    return a.id < b.id;
  });
  pr.pos_of.assign(n, -1);
  for (size_t k = 0; k < pr.splats.size(); ++k) pr.pos_of[pr.splats[k].id] = (int64_t)k;
}

double wall() {
#ifdef _OPENMP
  return omp_get_wtime();
#else
  return 0.0;
#endif
}

Cam make_cam(const double* c) {
  Cam cam;
  cam.fx = c[0]; cam.fy = c[1]; cam.cx = c[2]; cam.cy = c[3];
  cam.W = (int)c[4]; cam.H = (int)c[5];
  for (int k = 0; k < 9; ++k) cam.R[k] = c[6 + k];
  for (int k = 0; k < 3; ++k) cam.t[k] = c[15 + k];
  cam.znear = c[18];
  return cam;
}
Opt make_opt(const double* o) {
  Opt opt;
  opt.alpha_min = o[0]; opt.alpha_max = o[1]; opt.T_min = o[2]; opt.median_T = o[3]; opt.dilation = o[4];
  opt.bg[0] = o[5]; opt.bg[1] = o[6]; opt.bg[2] = o[7];
  opt.sh_degree = (int)o[8];
  for (int k = 0; k < 5; ++k) opt.eps[k] = o[9 + k];
  opt.guard_band = o[14];
  return opt;
}
SceneIn make_scene(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
                   const double* sh, int sh_coeffs) {
  SceneIn s{n, means, scales, rot, opac, sh, sh_coeffs};
  return s;
}

}  // namespace

extern "C" {

/* Layouts shared with oracle/__init__.py only:
 *   cam[19]  = fx, fy, cx, cy, W, H, R[9] (world->camera, row-major), t[3], znear
 *   opt[15]  = alpha_min, alpha_max, T_min, median_T, dilation, bg[3], sh_degree, eps[5], guard_band
 *   scene    = double SoA: means[3][n], scales[3][n], rot[4][n] (w,x,y,z), opac[n], sh[K*3][n]
 */

#define OR_PG_STRIDE 96
/* or_project: per Gaussian, out[i*96 + ...]:
 *  0 valid, 1 zkey, 2..4 x_c, 5 z, 6 t_c, 7 u, 8 v, 9..17 Σ (world), 18..26 Σ_c, 27..35 J,
 *  36..44 Σ′, 45..53 Σ′⁻¹, 54..56 A′ (a,b,c), 57..59 conic, 60..62 q̂, 63..64 q, 65..66 p,
 *  67..69 n, 70..72 rgb, 73..75 rgb_clamped, 76 o, 77 n·x̂_c */
int or_project(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
               const double* sh, int sh_coeffs, const double* camv, const double* optv, double* out) {
  SceneIn sc = make_scene(n, means, scales, rot, opac, sh, sh_coeffs);
  Cam cam = make_cam(camv);
  Opt opt = make_opt(optv);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double P[NP], raw[11];
    load_params(sc, i, P);
    for (int k = 0; k < 11; ++k) raw[k] = P[k];
    PG<double> g;
    double* o = out + i * OR_PG_STRIDE;
    for (int k = 0; k < OR_PG_STRIDE; ++k) o[k] = 0.0;
    bool ok = project(P, raw, cam, opt, g);
    o[0] = ok ? 1.0 : 0.0;
    o[1] = (double)g.zkey;
    if (!ok) continue;
    for (int k = 0; k < 3; ++k) o[2 + k] = g.x[k];
    o[5] = g.z; o[6] = g.tc; o[7] = g.u; o[8] = g.v;
    for (int k = 0; k < 9; ++k) { o[9 + k] = g.Sigma[k]; o[18 + k] = g.Sc[k]; o[27 + k] = g.J[k]; o[36 + k] = g.Sp[k]; o[45 + k] = g.Spi[k]; }
    for (int k = 0; k < 3; ++k) { o[54 + k] = g.A2[k]; o[57 + k] = g.conic[k]; o[60 + k] = g.qhat[k]; o[67 + k] = g.n[k]; o[70 + k] = g.rgb[k]; o[73 + k] = g.rgb_clamped[k] ? 1.0 : 0.0; }
    o[63] = g.q[0]; o[64] = g.q[1]; o[65] = g.p[0]; o[66] = g.p[1];
    o[76] = g.o; o[77] = g.ndotx;
  }
  return 0;
}

/* or_sh_basis: the 16 real-SH basis values of reading S14 at unit direction dir. */
void or_sh_basis(const double* dir, double* out16) {
  double d[3] = {dir[0], dir[1], dir[2]};
  sh_basis(d, out16);
}

/* or_splat_eval: one Gaussian against a list of (u, v) image points.
 *  out[k*6 + ...]: 0 alpha (unclamped o·exp(power)), 1 t* (Eq.12, ray space), 2 d (Eq.15),
 *  3 t*_persp (Eq.7, true perspective ray through (u,v)), 4 depth of that point, 5 power. */
int or_splat_eval(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
                  const double* sh, int sh_coeffs, const double* camv, const double* optv, int64_t gid,
                  int64_t npts, const double* uv, double* out) {
  SceneIn sc = make_scene(n, means, scales, rot, opac, sh, sh_coeffs);
  Cam cam = make_cam(camv);
  Opt opt = make_opt(optv);
  double P[NP], raw[11];
  load_params(sc, gid, P);
  for (int k = 0; k < 11; ++k) raw[k] = P[k];
  PG<double> g;
  if (!project(P, raw, cam, opt, g)) return 1;
  double Sci[9];
  if (!inverse3(g.Sc, Sci)) return 2;
  for (int64_t k = 0; k < npts; ++k) {
    double u = uv[2 * k], v = uv[2 * k + 1];
    double du = g.u - u, dv = g.v - v;
    double power = -0.5 * (g.conic[0] * du * du + 2.0 * g.conic[1] * du * dv + g.conic[2] * dv * dv);
    double tstar = (g.Spi[6] * du + g.Spi[7] * dv + g.Spi[8] * g.tc) / g.Spi[8];
    // Eq.7: t* = vᵀΣ⁻¹(x_c − o) / (vᵀΣ⁻¹v), camera frame (o = 0), v through pixel (u, v)
    double r[3] = {(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, 1.0};
    double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (int i = 0; i < 3; ++i) r[i] /= rl;
    double Sr[3], Sx[3];
    for (int i = 0; i < 3; ++i) {
      Sr[i] = Sci[3 * i] * r[0] + Sci[3 * i + 1] * r[1] + Sci[3 * i + 2] * r[2];
      Sx[i] = Sci[3 * i] * g.x[0] + Sci[3 * i + 1] * g.x[1] + Sci[3 * i + 2] * g.x[2];
    }
    double tp = (r[0] * Sx[0] + r[1] * Sx[1] + r[2] * Sx[2]) / (r[0] * Sr[0] + r[1] * Sr[1] + r[2] * Sr[2]);
    double* o = out + 6 * k;
    o[0] = g.o * std::exp(power);
    o[1] = tstar;
    o[2] = (g.z / g.tc) * tstar;
    o[3] = tp;
    o[4] = tp * r[2];
    o[5] = power;
  }
  return 0;
}

/* or_render: brute-force per-pixel render. pix == NULL renders the full W×H frame
 * (npix = W*H, pixel k = (k % W, k / W)); otherwise pix[k] is a linear pixel index.
 * Outputs per listed pixel k (planar by channel):
 *   color[3*npix] (color[c*npix+k]), depth[npix] (median, 0 = none), normal[3*npix],
 *   alpha[npix] = 1 − T_final, flags[npix] (bit0 F1 α-cutoff, bit1 F2 α-clamp, bit2 F3
 *   T-stop, bit3 F4 median crossing, bit4 F5 grazing median splat), nblend[npix] (number
 *   of blended splats), median_id[npix] (Gaussian id of the median splat or −1),
 *   distortion[npix] = L_d of the pixel (S21). */
int or_render(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
              const double* sh, int sh_coeffs, const double* camv, const double* optv, int64_t npix,
              const int64_t* pix, double* color, double* depth, double* normal, double* alpha, uint8_t* flags,
              int32_t* nblend, int64_t* median_id, double* distortion_out, double* timing) {
  SceneIn sc = make_scene(n, means, scales, rot, opac, sh, sh_coeffs);
  Cam cam = make_cam(camv);
  Opt opt = make_opt(optv);
  Prepared pr;
  double t0 = wall();
  prepare(sc, cam, opt, pr);
  double t1 = wall();
  const int64_t ns = (int64_t)pr.splats.size();
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < npix; ++k) {
    int64_t lin = pix ? pix[k] : k;
    double u = (double)(lin % cam.W) + 0.5, v = (double)(lin / cam.W) + 0.5;  // pixel centre (S4)
    Pix<double> px;
    pix_init(px);
    for (int64_t s = 0; s < ns; ++s)
      if (!blend(px, pr.splats[s], u, v, opt)) break;
    for (int c = 0; c < 3; ++c) {
      color[c * npix + k] = px.C[c] + px.T * opt.bg[c];  // + T_final·bg (S17)
      normal[c * npix + k] = px.N[c];
    }
    depth[k] = px.D;
    alpha[k] = 1.0 - px.T;
    flags[k] = px.flags;
    nblend[k] = px.nblend;
    median_id[k] = px.median_id;
    distortion_out[k] = distortion(px);
  }
  if (timing) {  // [0] project + sort seconds, [1] per-pixel loop seconds, [2] surviving Gaussians
    timing[0] = t1 - t0;
    timing[1] = wall() - t1;
    timing[2] = (double)ns;
  }
  return 0;
}

/* or_grad: exact gradient of L = Σ_px g·(C, D, N, A, L_d) w.r.t. the 59 parameters of each
 * listed Gaussian, by forward-mode dual numbers through or_render's definition (ω detached
 * in L_d, S21), and w.r.t. its projected centre (u_c, v_c) with every other per-splat
 * quantity held fixed (the screen-space gradient of 3DGS's densification).
 *   cot[9][H][W] planar: dL/dC (3), dL/dD, dL/dN (3), dL/dA, dL/dL_d.
 *   out[k*61 + j]: j = μ 0..2, s 3..5, q(w,x,y,z) 6..9, o 10, sh 11 + coeff*3 + channel,
 *   59..60 = dL/d(u_c, v_c).
 *   culled Gaussians get zero. */
int or_grad(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
            const double* sh, int sh_coeffs, const double* camv, const double* optv, const double* cot,
            int64_t ng, const int64_t* gids, double* out, double* timing) {
  SceneIn sc = make_scene(n, means, scales, rot, opac, sh, sh_coeffs);
  Cam cam = make_cam(camv);
  Opt opt = make_opt(optv);
  Prepared pr;
  double t0 = wall();
  prepare(sc, cam, opt, pr);
  double t1 = wall();
  const int64_t ns = (int64_t)pr.splats.size();
  const int64_t npx = (int64_t)cam.W * cam.H;
  for (int64_t gk = 0; gk < ng; ++gk) {
    int64_t gid = gids[gk];
    double* res = out + gk * NP;
    for (int j = 0; j < NP; ++j) res[j] = 0.0;
    int64_t pos = pr.pos_of[gid];
    if (pos < 0) continue;
    Dual P[NP];
    double raw[11];
    load_params(sc, gid, P);
    for (int k = 0; k < 11; ++k) raw[k] = P[k].v;
    for (int j = 0; j < NP; ++j) P[j].d[j] = 1.0;
    PG<Dual> gd;
    if (!project(P, raw, cam, opt, gd)) continue;
    Splat<Dual> sd = compact(gd, gid);
    const Splat<double>& sv = pr.splats[pos];
#pragma omp parallel
    {
      double acc[NP] = {0};
#pragma omp for schedule(dynamic, 16)
      for (int64_t lin = 0; lin < npx; ++lin) {
        double u = (double)(lin % cam.W) + 0.5, v = (double)(lin / cam.W) + 0.5;
        // does g contribute here at all?  (α_g < α_min ⇒ outputs locally independent of g)
        double du = sv.u - u, dv = sv.v - v;
        double pw = -0.5 * (sv.conic[0] * du * du + 2.0 * sv.conic[1] * du * dv + sv.conic[2] * dv * dv);
        if (std::min(opt.alpha_max, sv.o * std::exp(pw)) < opt.alpha_min) continue;
        Pix<double> pd;
        pix_init(pd);
        bool alive = true;
        for (int64_t s = 0; s < pos && alive; ++s) alive = blend(pd, pr.splats[s], u, v, opt);
        if (!alive) continue;
        Pix<Dual> px;
        promote(pd, px);
        if (blend(px, sd, u, v, opt))
          for (int64_t s = pos + 1; s < ns; ++s)
            if (!blend(px, pr.splats[s], u, v, opt)) break;
        Dual L = px.D * cot[3 * npx + lin] + (1.0 - px.T) * cot[7 * npx + lin];
        if (cot[8 * npx + lin] != 0.0) L = L + distortion(px) * cot[8 * npx + lin];
        for (int c = 0; c < 3; ++c)
          L = L + (px.C[c] + px.T * opt.bg[c]) * cot[c * npx + lin] + px.N[c] * cot[(4 + c) * npx + lin];
        for (int j = 0; j < NP; ++j) acc[j] += L.d[j];
      }
#pragma omp critical
      for (int j = 0; j < NP; ++j) res[j] += acc[j];
    }
  }
  if (timing) {  // [0] project + sort seconds, [1] dual-number loop seconds, [2] surviving Gaussians
    timing[0] = t1 - t0;
    timing[1] = wall() - t1;
    timing[2] = (double)ns;
  }
  return 0;
}

/* or_order: the global front-to-back order of the surviving Gaussians (reading
 * S7: z_key ascending, ties by index) — out[0 .. *n_out) are Gaussian ids. */
int or_order(int64_t n, const double* means, const double* scales, const double* rot, const double* opac,
             const double* sh, int sh_coeffs, const double* camv, const double* optv, int64_t* out, int64_t* n_out) {
  SceneIn sc = make_scene(n, means, scales, rot, opac, sh, sh_coeffs);
  Cam cam = make_cam(camv);
  Opt opt = make_opt(optv);
  Prepared pr;
  prepare(sc, cam, opt, pr);
  for (size_t k = 0; k < pr.splats.size(); ++k) out[k] = pr.splats[k].id;
  *n_out = (int64_t)pr.splats.size();
  return 0;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
