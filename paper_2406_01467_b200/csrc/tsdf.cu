// tsdf.cu — NEXT-4 of the RaDe-GS hot path, sm_100a: TSDF fusion of rendered median depth
// maps ("We render depth maps for all training views and construct a TSDF";
// reading S24 in DESIGN.md).
//
// One thread per voxel of the [Z][Y][X] grid (x fastest: coalesced), and up to kViews views
// per launch fused in registers: the voxel's (tsdf, weight) is read once, updated by every
// view of the batch in view order, and written once — 8 B in + 8 B out per voxel per batch
// instead of per view (the HBM roofline of fusion), plus a 4-B depth gather per voxel and
// view that the 126 MB L2 mostly serves. The voxel centre, camera-space point and projection
// are formed in fp32 without FMA in the oracle's fixed order, so the pixel a voxel reads is
// the same decision on both sides.
#include "rade_internal.cuh"

namespace rade {
namespace {

constexpr int kViews = 32;

struct TsdfCam {
  float R[9], t[3];
  float fx, fy, cx, cy, znear;
};
struct TsdfCams {
  TsdfCam c[kViews];
};

__global__ void __launch_bounds__(256) k_tsdf_integrate(TsdfCams cams, int n_views, const float* __restrict__ depths,
                                                        int W, int H, float ox, float oy, float oz, float vs,
                                                        float trunc, float max_depth, int X, int Y, int Z,
                                                        float* __restrict__ tsdf, float* __restrict__ weight) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nvox = (int64_t)X * Y * Z;
  if (idx >= nvox) return;
  const int x = (int)(idx % X), y = (int)((idx / X) % Y), z = (int)(idx / ((int64_t)X * Y));
  const float Xw = __fadd_rn(__fmul_rn(__fadd_rn((float)x, 0.5f), vs), ox);
  const float Yw = __fadd_rn(__fmul_rn(__fadd_rn((float)y, 0.5f), vs), oy);
  const float Zw = __fadd_rn(__fmul_rn(__fadd_rn((float)z, 0.5f), vs), oz);
  float ts = tsdf[idx], w = weight[idx];
  const float itr = 1.f / trunc;
  // fully unrolled over the batch: every camera field is then a constant-bank operand of its
  // instruction instead of a dynamically indexed parameter load (17 LDC per view, MIO-bound)
#pragma unroll
  for (int v = 0; v < kViews; ++v) {
    if (v >= n_views) break;
    const TsdfCam& c = cams.c[v];
    const float xc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[0], Xw), __fmul_rn(c.R[1], Yw)), __fmul_rn(c.R[2], Zw)), c.t[0]);
    const float yc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[3], Xw), __fmul_rn(c.R[4], Yw)), __fmul_rn(c.R[5], Zw)), c.t[1]);
    const float zc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(c.R[6], Xw), __fmul_rn(c.R[7], Yw)), __fmul_rn(c.R[8], Zw)), c.t[2]);
    if (!(zc > c.znear)) continue;
    const float u = __fadd_rn(__fdiv_rn(__fmul_rn(c.fx, xc), zc), c.cx);
    const float vv = __fadd_rn(__fdiv_rn(__fmul_rn(c.fy, yc), zc), c.cy);
    if (!(u >= 0.f && vv >= 0.f && u < (float)W && vv < (float)H)) continue;
    const float D = __ldg(depths + ((int64_t)v * H + (int)vv) * W + (int)u);
    if (!(D > 0.f && D <= max_depth)) continue;
    const float sdf = __fsub_rn(D, zc);
    if (!(sdf > -trunc)) continue;
    const float nw = fminf(fmaxf(sdf * itr, -1.f), 1.f);
    ts = (w * ts + nw) / (w + 1.f);
    w += 1.f;
  }
  tsdf[idx] = ts;
  weight[idx] = w;
}

}  // namespace

int tsdf_views_per_launch() { return kViews; }

void launch_tsdf_integrate(const float* cam_rows, int n_views, const float* depths, int W, int H, const float origin[3],
                           float voxel, float trunc, float max_depth, const int dims[3], float* tsdf, float* weight,
                           cudaStream_t s) {
  // cam_rows: n_views × 17 floats (R[9], t[3], fx, fy, cx, cy, znear), n_views ≤ kViews
  TsdfCams cams;
  for (int v = 0; v < n_views; ++v) {
    const float* r = cam_rows + 17 * v;
    TsdfCam& c = cams.c[v];
    for (int k = 0; k < 9; ++k) c.R[k] = r[k];
    for (int k = 0; k < 3; ++k) c.t[k] = r[9 + k];
    c.fx = r[12]; c.fy = r[13]; c.cx = r[14]; c.cy = r[15]; c.znear = r[16];
  }
  const int64_t nvox = (int64_t)dims[0] * dims[1] * dims[2];
  if (nvox == 0 || n_views == 0) return;
  k_tsdf_integrate<<<(unsigned)((nvox + 255) / 256), 256, 0, s>>>(cams, n_views, depths, W, H, origin[0], origin[1],
                                                                  origin[2], voxel, trunc, max_depth, dims[0],
                                                                  dims[1], dims[2], tsdf, weight);
}

}  // namespace rade
