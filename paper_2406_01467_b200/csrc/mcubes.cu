// mcubes.cu — NEXT-4 of the RaDe-GS hot path, sm_100a: marching-cubes extraction of the
// fused TSDF's zero level set ("with the Marching Cube algorithm"; reading S25).
//
// The triangulation table is built on the host at first use by walking the cube faces: on
// every face each maximal run of inside corners (value < iso) is cut off by one segment from
// the crossing where the run is entered to the crossing where it is left (walking the face
// counter-clockwise seen from outside), so diagonal inside corners are always separated — a
// decision that depends on the face alone, hence shared by the two cells on either side of
// it, which makes the surface watertight. The segments chain into closed loops through the
// crossing edges; each loop is fanned into triangles whose winding makes the normal point
// from the inside corners to the outside ones.
//
// Extraction is three passes over the (X−1)(Y−1)(Z−1) cells: count triangles per cell (0 if
// a corner has weight 0), exclusive scan (binning.cu's single-pass look-back scan), emit each
// cell's triangles at its offset —
// a deterministic triangle soup in cell order (x fastest), triangles in table order.
// Degenerate triangles are dropped (reading S25): a vertex lands exactly on a cube corner only
// when that corner's value equals iso (then s = (iso − v_a)/(v_b − v_a) is exactly 0 or 1),
// and a triangle is degenerate exactly when two of its vertices land on the same corner
// (three distinct corner / edge-interior points of a cube cannot be collinear here).
#include "rade_internal.cuh"

#include <cmath>
#include <vector>

namespace rade {
namespace {

constexpr int kMaxTri = 5;  // the face-walking rule never needs more per cell

__constant__ int8_t c_tri[256][3 * kMaxTri];
__constant__ uint8_t c_ntri[256];

// cube corner c at (c & 1, c >> 1 & 1, c >> 2 & 1); edge e joins kEdge[e][0] → kEdge[e][1]
constexpr int kEdge[12][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3},
                              {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
__constant__ int c_edge[12][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3},
                                  {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};

struct McTable {
  int8_t tri[256][3 * kMaxTri];
  uint8_t ntri[256];
};

int edge_between(int a, int b) {
  for (int e = 0; e < 12; ++e)
    if ((kEdge[e][0] == a && kEdge[e][1] == b) || (kEdge[e][0] == b && kEdge[e][1] == a)) return e;
  return -1;
}

McTable build_table() {
  // the six faces as corner cycles, counter-clockwise seen from outside the cube
  const int face[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4}, {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
  McTable t{};
  for (int cfg = 0; cfg < 256; ++cfg) {
    auto in = [&](int c) { return ((cfg >> c) & 1) != 0; };
    int next[12];
    for (int e = 0; e < 12; ++e) next[e] = -1;
    for (int f = 0; f < 6; ++f)
      for (int i = 0; i < 4; ++i) {
        const int prev = face[f][(i + 3) % 4], cur = face[f][i];
        if (!in(cur) || in(prev)) continue;  // not the first corner of an inside run
        int j = i;
        while (in(face[f][(j + 1) % 4])) j = (j + 1) % 4;
        next[edge_between(prev, cur)] = edge_between(face[f][j], face[f][(j + 1) % 4]);
      }
    double cin[3] = {0, 0, 0}, cout[3] = {0, 0, 0};
    int nin = 0, nout = 0;
    for (int c = 0; c < 8; ++c) {
      const double p[3] = {(double)(c & 1), (double)((c >> 1) & 1), (double)((c >> 2) & 1)};
      for (int k = 0; k < 3; ++k) (in(c) ? cin : cout)[k] += p[k];
      (in(c) ? nin : nout) += 1;
    }
    int ntri = 0;
    bool used[12] = {false};
    for (int e0 = 0; e0 < 12; ++e0) {
      if (next[e0] < 0 || used[e0]) continue;
      int loop[12], n = 0;
      for (int e = e0; !used[e]; e = next[e]) {
        used[e] = true;
        loop[n++] = e;
      }
      // Newell normal of the loop through the edge midpoints vs inside → outside
      double nrm[3] = {0, 0, 0};
      for (int k = 0; k < n; ++k) {
        double p[3], q[3];
        for (int d = 0; d < 3; ++d) {
          const int a = kEdge[loop[k]][0], b = kEdge[loop[k]][1];
          const int a2 = kEdge[loop[(k + 1) % n]][0], b2 = kEdge[loop[(k + 1) % n]][1];
          p[d] = 0.5 * (((a >> d) & 1) + ((b >> d) & 1));
          q[d] = 0.5 * (((a2 >> d) & 1) + ((b2 >> d) & 1));
        }
        nrm[0] += (p[1] - q[1]) * (p[2] + q[2]);
        nrm[1] += (p[2] - q[2]) * (p[0] + q[0]);
        nrm[2] += (p[0] - q[0]) * (p[1] + q[1]);
      }
      double dir = 0;
      for (int k = 0; k < 3; ++k) dir += nrm[k] * (cout[k] / (nout ? nout : 1) - cin[k] / (nin ? nin : 1));
      if (dir < 0)
        for (int k = 0; k < n / 2; ++k) std::swap(loop[k], loop[n - 1 - k]);
      for (int k = 1; k + 1 < n; ++k) {
        t.tri[cfg][3 * ntri] = (int8_t)loop[0];
        t.tri[cfg][3 * ntri + 1] = (int8_t)loop[k];
        t.tri[cfg][3 * ntri + 2] = (int8_t)loop[k + 1];
        ++ntri;
      }
    }
    t.ntri[cfg] = (uint8_t)ntri;
  }
  return t;
}

struct Vol {
  float ox, oy, oz, vs;
  int X, Y, Z;
  const float* tsdf;
  const float* weight;
};

__device__ __forceinline__ int cell_config(const Vol& v, int i, int j, int k, float iso, float (&val)[8]) {
  int cfg = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int64_t idx = ((int64_t)(k + ((c >> 2) & 1)) * v.Y + (j + ((c >> 1) & 1))) * v.X + (i + (c & 1));
    if (v.weight[idx] == 0.f) return -1;
    val[c] = v.tsdf[idx];
    cfg |= (val[c] < iso ? 1 : 0) << c;
  }
  return cfg;
}

// The cube corner a vertex on edge e sits on (s = 0: its first corner, s = 1: its second), −1
// for an edge-interior vertex.
__device__ __forceinline__ int vertex_corner(int e, const float (&val)[8], float iso) {
  const int a = c_edge[e][0], b = c_edge[e][1];
  const float s = (iso - val[a]) / (val[b] - val[a]);
  return s == 0.f ? a : (s == 1.f ? b : -1);
}
__device__ __forceinline__ bool tri_degenerate(int cfg, int t, const float (&val)[8], float iso) {
  const int c0 = vertex_corner(c_tri[cfg][3 * t], val, iso), c1 = vertex_corner(c_tri[cfg][3 * t + 1], val, iso),
            c2 = vertex_corner(c_tri[cfg][3 * t + 2], val, iso);
  return (c0 >= 0 && (c0 == c1 || c0 == c2)) || (c1 >= 0 && c1 == c2);
}

__global__ void __launch_bounds__(256) k_mc_count(Vol v, float iso, uint32_t* __restrict__ count) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int CX = v.X - 1, CY = v.Y - 1;
  const int64_t ncell = (int64_t)CX * CY * (v.Z - 1);
  if (cell >= ncell) return;
  const int i = (int)(cell % CX), j = (int)((cell / CX) % CY), k = (int)(cell / ((int64_t)CX * CY));
  float val[8];
  const int cfg = cell_config(v, i, j, k, iso, val);
  uint32_t n = 0;
  if (cfg >= 0)
    for (int t = 0; t < c_ntri[cfg]; ++t) n += tri_degenerate(cfg, t, val, iso) ? 0u : 1u;
  count[cell] = n;
}

__global__ void __launch_bounds__(256) k_mc_emit(Vol v, float iso, const uint32_t* __restrict__ offset,
                                                 float* __restrict__ out) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int CX = v.X - 1, CY = v.Y - 1;
  const int64_t ncell = (int64_t)CX * CY * (v.Z - 1);
  if (cell >= ncell) return;
  const int i = (int)(cell % CX), j = (int)((cell / CX) % CY), k = (int)(cell / ((int64_t)CX * CY));
  float val[8];
  const int cfg = cell_config(v, i, j, k, iso, val);
  if (cfg < 0) return;
  const int n = c_ntri[cfg];
  float* o = out + (int64_t)offset[cell] * 9;
  for (int t = 0, w = 0; t < n; ++t) {
    if (tri_degenerate(cfg, t, val, iso)) continue;
    for (int q = 0; q < 3; ++q) {
      const int e = c_tri[cfg][3 * t + q], a = c_edge[e][0], b = c_edge[e][1];
      const float s = (iso - val[a]) / (val[b] - val[a]);
      const int ia[3] = {i + (a & 1), j + ((a >> 1) & 1), k + ((a >> 2) & 1)};
      const int ib[3] = {i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1)};
      const float org[3] = {v.ox, v.oy, v.oz};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const float pa = __fadd_rn(__fmul_rn((float)ia[d] + 0.5f, v.vs), org[d]);
        const float pb = __fadd_rn(__fmul_rn((float)ib[d] + 0.5f, v.vs), org[d]);
        o[9 * w + 3 * q + d] = pa + s * (pb - pa);
      }
    }
    ++w;
  }
}

}  // namespace

namespace {
// Per host thread, grow-only scratch reused across calls (count, offset, scan temp) and a
// pinned slot for the count read-back: a fresh cudaMallocAsync / cudaMallocHost per call cost
// milliseconds (and cudaFreeHost synchronises the device). `done` is recorded after the last
// use of the scratch (the emit reads offset asynchronously); the next call — possibly on
// another stream — waits for it before rewriting count / offset, and before freeing them.
struct McScratch {
  uint32_t *count = nullptr, *offset = nullptr, *host = nullptr;
  unsigned long long* status = nullptr;  // the scan's look-back words (zeroed when allocated)
  size_t cells = 0, status_words = 0;
  uint32_t epoch = 0;
  cudaEvent_t done = nullptr;
};
thread_local McScratch t_mc;

// The triangulation table goes to constant memory once per process (every call used to
// rewrite it asynchronously while an earlier emit on another stream could be reading it).
cudaError_t upload_table() {
  static cudaError_t status = [] {
    const McTable table = build_table();
    cudaError_t e = cudaMemcpyToSymbol(c_tri, table.tri, sizeof(table.tri));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_ntri, table.ntri, sizeof(table.ntri));
    return e;
  }();
  return status;
}
}  // namespace

cudaError_t launch_marching_cubes(const float origin[3], float voxel, const int dims[3], const float* tsdf,
                                  const float* weight, float iso, float* triangles, int64_t capacity,
                                  int64_t* n_triangles, cudaStream_t s) {
  cudaError_t e = upload_table();  // thread-safe one-time construction and upload
  if (e != cudaSuccess) return e;
  *n_triangles = 0;
  if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2) return cudaSuccess;
  const Vol v{origin[0], origin[1], origin[2], voxel, dims[0], dims[1], dims[2], tsdf, weight};
  const int64_t ncell = (int64_t)(dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1);
  if (ncell > 0x7fffffffLL) return cudaErrorInvalidValue;
  McScratch& m = t_mc;
  if (!m.host) {
    e = cudaMallocHost(&m.host, 8);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  } else {
    e = cudaStreamWaitEvent(s, m.done, 0);  // the previous call's emit has read offset
    if (e != cudaSuccess) return e;
  }
  if (m.cells < (size_t)ncell) {
    e = cudaEventSynchronize(m.done);  // the old buffers may still be in use
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (m.count) cudaFree(m.count);
    if (m.offset) cudaFree(m.offset);
    m.count = m.offset = nullptr;
    m.cells = 0;
    if (e == cudaSuccess) e = cudaMalloc(&m.count, (size_t)ncell * 4);
    if (e == cudaSuccess) e = cudaMalloc(&m.offset, (size_t)ncell * 4);
    if (e != cudaSuccess) return e;
    m.cells = (size_t)ncell;
  }
  const size_t words = scan_status_words(ncell);
  if (m.status_words < words) {
    e = cudaEventSynchronize(m.done);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (m.status) cudaFree(m.status);
    m.status = nullptr;
    m.status_words = 0;
    if (e == cudaSuccess) e = cudaMalloc(&m.status, words * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(m.status, 0, words * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    m.status_words = words;
  }
  const unsigned grid = (unsigned)((ncell + 255) / 256);
  k_mc_count<<<grid, 256, 0, s>>>(v, iso, m.count);
  BinSort bs{m.status, m.epoch};
  launch_scan_excl_u32(m.count, m.offset, ncell, bs, s);
  m.epoch = bs.epoch;
  cudaMemcpyAsync(m.host, m.offset + (ncell - 1), 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(m.host + 1, m.count + (ncell - 1), 4, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *n_triangles = (int64_t)m.host[0] + m.host[1];
  if (triangles && capacity >= *n_triangles) k_mc_emit<<<grid, 256, 0, s>>>(v, iso, m.offset, triangles);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventRecord(m.done, s);
  return e;
}

}  // namespace rade
