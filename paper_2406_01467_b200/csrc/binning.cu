// binning.cu — stage 2 (K2) of the RaDe-GS rasterizer, sm_100a.
//
// The depth sort of PAPER:422 per tile, as a two-stage stable sort whose result is
// bit-identical to one LSD radix sort of 64-bit keys (tile << 32 | float_bits(z_c)) over
// (Gaussian, tile) pairs emitted in id order (reading S7):
//
//   K2a  depth sort: stable radix sort of the N pairs (float_bits(z_c), id) — culled or
//        off-screen Gaussians carry key 0xFFFFFFFF and sink to the end. Order (z_c, id).
//   K2b  inclusive scan of tiles_touched gathered in that order → offsets; M = offsets[N−1]
//   K2c  duplicate: each Gaussian, in depth order, emits (tile, id) for every tile of its
//        rect (warp-cooperative, coalesced stores)
//   K2d  stable radix sort of the M pairs by tile on ceil(log2 T) bits (2 passes at 4096
//        tiles instead of 6 passes over 12-byte pairs): within a tile the (z_c, id) order
//        of K2a is preserved
//   K2e  ranges[tile] = [first, last) in the sorted list
//
// z_c > znear > 0, so the IEEE bit pattern orders like the value. Integer work: checked
// bit-exactly against a CPU std::stable_sort of the 64-bit keys.
#include "rade_internal.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/dispatch/dispatch_radix_sort.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

namespace rade {
namespace {

// CUB's onesweep radix sort with 512-thread × 12-key tiles (tools/sort_bench.cu on B200: 96 vs
// 107 µs for the 1.5 M depth keys, 129 vs 141 µs for 5.6 M 12-bit tile keys against CUB's
// default 384 × 23), 8-bit digits.
struct SortHub {
  using Base = cub::detail::radix::policy_hub<uint32_t, uint32_t, uint32_t>;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    using B = typename Base::Policy1000;
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = typename B::HistogramPolicy;
    using ExclusiveSumPolicy = typename B::ExclusiveSumPolicy;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<512, 12, uint32_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
    using ScanPolicy = typename B::ScanPolicy;
    using DownsweepPolicy = typename B::DownsweepPolicy;
    using AltDownsweepPolicy = typename B::AltDownsweepPolicy;
    using UpsweepPolicy = typename B::UpsweepPolicy;
    using AltUpsweepPolicy = typename B::AltUpsweepPolicy;
    using SingleTilePolicy = typename B::SingleTilePolicy;
    using SegmentedPolicy = typename B::SegmentedPolicy;
    using AltSegmentedPolicy = typename B::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy1000;
};
using Sort = cub::DispatchRadixSort<false, uint32_t, uint32_t, uint32_t, SortHub>;

struct CountOf {
  const uint32_t* __restrict__ touched;
  __host__ __device__ __forceinline__ uint32_t operator()(const uint32_t id) const { return touched[id]; }
};

// First index p in [0, n) with a[p] > target (n if none), searched by a whole warp: each
// round probes 32 evenly spaced positions and keeps the bracket (4 rounds for n = 1.5M).
__device__ __forceinline__ uint32_t warp_upper_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t target,
                                                     int lane) {
  uint32_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t probe = lo + (uint32_t)lane * step;
    const bool gt = probe < hi ? (a[probe] > target) : true;
    const unsigned m = __ballot_sync(0xffffffffu, gt);
    if (m == 0) {
      lo = lo + 31 * step + 1;
    } else {
      const int f = __ffs(m) - 1;
      if (f == 0) return lo;
      const uint32_t nlo = lo + (uint32_t)(f - 1) * step + 1;
      hi = min(hi, lo + (uint32_t)f * step);
      lo = nlo;
    }
  }
  const uint32_t probe = lo + (uint32_t)lane;
  const bool gt = probe < hi ? (a[probe] > target) : true;
  const unsigned m = __ballot_sync(0xffffffffu, gt);
  return m ? min(hi, lo + (uint32_t)(__ffs(m) - 1)) : hi;
}

constexpr int kDupThreads = 256;
constexpr int kDupPer = 8;     // consecutive outputs per thread
constexpr int kDupOut = kDupThreads * kDupPer;  // outputs per block (2048)

// Load-balanced emission over OUTPUTS: block b writes duplicates [b·2048, (b+1)·2048). In
// depth order every visible Gaussian touches ≥ 1 tile, so the block's outputs come from at
// most 2048 consecutive positions [g0, g1], found by one warp-wide search of the inclusive
// offsets. Their offsets, ids and rects are staged in shared memory; each output finds its
// owner by binary search there. Stores are coalesced and a huge near-camera splat is spread
// over as many blocks as its tiles need (no per-thread or per-warp serialisation). Per
// Gaussian the tiles are emitted row-major over its rect.
__global__ void __launch_bounds__(kDupThreads) k_duplicate(int64_t n, int64_t m, const uint32_t* __restrict__ offsets,
                                                            const uint32_t* __restrict__ sorted_ids,
                                                            const uint2* __restrict__ rect, int tiles_x,
                                                            uint32_t* __restrict__ tile_keys,
                                                            uint32_t* __restrict__ vals) {
  __shared__ uint32_t s_end[kDupOut + 1];
  __shared__ uint32_t s_id[kDupOut];
  __shared__ uint2 s_rect[kDupOut];
  __shared__ uint32_t s_g[2];
  const uint32_t o0 = blockIdx.x * (uint32_t)kDupOut;
  const uint32_t o1 = min((uint32_t)m, o0 + (uint32_t)kDupOut);
  if (threadIdx.x < 32) {
    const uint32_t g0 = warp_upper_bound(offsets, (uint32_t)n, o0, (int)threadIdx.x);
    const uint32_t g1 = warp_upper_bound(offsets, (uint32_t)n, o1 - 1, (int)threadIdx.x);
    if (threadIdx.x == 0) {
      s_g[0] = g0;
      s_g[1] = g1;
    }
  }
  __syncthreads();
  const uint32_t g0 = s_g[0];
  const int ng = (int)(s_g[1] - g0) + 1;  // ≤ kDupOut
  // s_end[0] = start of g0; s_end[k + 1] = end of g0 + k
  if (threadIdx.x == 0) s_end[0] = g0 == 0 ? 0u : offsets[g0 - 1];
  for (int k = threadIdx.x; k < ng; k += kDupThreads) {
    s_end[k + 1] = offsets[g0 + k];
    const uint32_t id = sorted_ids[g0 + k];
    s_id[k] = id;
    s_rect[k] = rect[id];
  }
  __syncthreads();
  // thread t writes the kDupPer consecutive outputs o0 + kDupPer·t ..: one binary search for
  // the first one's owner, then a walk (every staged Gaussian has ≥ 1 tile, so the owner
  // advances by at most one per output) with the tile stepped row-major over the rect, and
  // two 16-B stores per array (a warp writes 1 KB contiguous per array)
  const uint32_t o = o0 + (uint32_t)threadIdx.x * kDupPer;
  if (o >= o1) return;
  int lo = 0, hi = ng - 1;  // owner k: s_end[k] <= o < s_end[k + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_end[mid] <= o) lo = mid; else hi = mid - 1;
  }
  int k = lo;
  uint2 r = s_rect[k];
  uint32_t x0 = r.x & 0xffffu, x1 = r.y & 0xffffu;
  const uint32_t li = o - s_end[k], w = x1 - x0;
  uint32_t ty = (r.x >> 16) + li / w, tx = x0 + li % w;
  uint32_t key[kDupPer], val[kDupPer];
#pragma unroll
  for (int j = 0; j < kDupPer; ++j) {
    const uint32_t oj = o + (uint32_t)j;
    if (oj < o1) {
      if (oj >= s_end[k + 1]) {  // the next Gaussian starts here, at its rect's first tile
        ++k;
        r = s_rect[k];
        x0 = r.x & 0xffffu;
        x1 = r.y & 0xffffu;
        tx = x0;
        ty = r.x >> 16;
      }
      key[j] = ty * (uint32_t)tiles_x + tx;
      val[j] = s_id[k];
      if (++tx == x1) {
        tx = x0;
        ++ty;
      }
    }
  }
  if (o + kDupPer <= o1) {
    uint4* kk = reinterpret_cast<uint4*>(tile_keys + o);
    uint4* vv = reinterpret_cast<uint4*>(vals + o);
    kk[0] = make_uint4(key[0], key[1], key[2], key[3]);
    kk[1] = make_uint4(key[4], key[5], key[6], key[7]);
    vv[0] = make_uint4(val[0], val[1], val[2], val[3]);
    vv[1] = make_uint4(val[4], val[5], val[6], val[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kDupPer; ++j)
      if (o + (uint32_t)j < o1) {
        tile_keys[o + j] = key[j];
        vals[o + j] = val[j];
      }
  }
}

// 8 consecutive sorted keys per thread (two 16-B loads) + the next one; a boundary between
// positions k and k+1 closes tile keys[k] and opens tile keys[k+1].
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, int64_t m,
                                                 uint2* __restrict__ ranges) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (b >= m) return;
  uint32_t k[9];
  if (b + 8 <= m) {
    const uint4 q0 = *reinterpret_cast<const uint4*>(keys + b);
    const uint4 q1 = *reinterpret_cast<const uint4*>(keys + b + 4);
    k[0] = q0.x; k[1] = q0.y; k[2] = q0.z; k[3] = q0.w;
    k[4] = q1.x; k[5] = q1.y; k[6] = q1.z; k[7] = q1.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) k[j] = b + j < m ? keys[b + j] : 0xffffffffu;
  }
  k[8] = b + 8 < m ? keys[b + 8] : 0xffffffffu;
  if (b == 0) ranges[k[0]].x = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t p = b + j;
    if (p < m && k[j] != k[j + 1]) {
      ranges[k[j]].y = (uint32_t)(p + 1);
      if (p + 1 < m) ranges[k[j + 1]].x = (uint32_t)(p + 1);
    }
  }
}

__global__ void __launch_bounds__(256) k_keys64(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ ids,
                                                 const Record* __restrict__ rec, int64_t m,
                                                 uint64_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  out[k] = ((uint64_t)tiles[k] << 32) | (uint64_t)__float_as_uint(rec[ids[k]].r3.x);
}

}  // namespace

size_t binning_temp_bytes(int64_t n, int64_t m, int tile_bits) {
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr), v(nullptr, nullptr);
  Sort::Dispatch(nullptr, a, k, v, (uint32_t)n, 0, 32, true, 0);
  cub::TransformInputIterator<uint32_t, CountOf, const uint32_t*> it(nullptr, CountOf{nullptr});
  cub::DeviceScan::InclusiveSum(nullptr, b, it, (uint32_t*)nullptr, (int)n);
  if (m > 0) Sort::Dispatch(nullptr, c, k, v, (uint32_t)m, 0, tile_bits, true, 0);
  size_t r = a > b ? a : b;
  return r > c ? r : c;
}

int launch_depth_sort(uint32_t* dkey0, uint32_t* dkey1, uint32_t* idx0, uint32_t* idx1, int64_t n, void* temp,
                      size_t temp_bytes, cudaStream_t s) {
  if (n == 0) return 0;
  cub::DoubleBuffer<uint32_t> k(dkey0, dkey1), v(idx0, idx1);
  Sort::Dispatch(temp, temp_bytes, k, v, (uint32_t)n, 0, 32, true, s);
  return k.selector;
}

void launch_scan(const uint32_t* sorted_ids, const uint32_t* tiles_touched, uint32_t* offsets, int64_t n, void* temp,
                 size_t temp_bytes, cudaStream_t s) {
  if (n == 0) return;
  cub::TransformInputIterator<uint32_t, CountOf, const uint32_t*> it(sorted_ids, CountOf{tiles_touched});
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, it, offsets, (int)n, s);
}

void launch_duplicate(int64_t n, int64_t m, const uint32_t* offsets, const uint32_t* sorted_ids, const uint2* rect,
                      int tiles_x, uint32_t* tile_keys, uint32_t* vals, cudaStream_t s) {
  if (n == 0 || m == 0) return;
  k_duplicate<<<(unsigned)((m + kDupOut - 1) / kDupOut), kDupThreads, 0, s>>>(n, m, offsets, sorted_ids, rect, tiles_x,
                                                                            tile_keys, vals);
}

int launch_tile_sort(uint32_t* keys0, uint32_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t m, int tile_bits,
                     void* temp, size_t temp_bytes, cudaStream_t s) {
  if (m == 0) return 0;
  cub::DoubleBuffer<uint32_t> k(keys0, keys1), v(vals0, vals1);
  Sort::Dispatch(temp, temp_bytes, k, v, (uint32_t)m, 0, tile_bits, true, s);
  return k.selector;
}

void launch_ranges(const uint32_t* keys, int64_t m, int n_tiles, uint2* ranges, cudaStream_t s) {
  cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
  if (m == 0) return;
  const int threads = 256;
  const int64_t items = (m + 7) / 8;
  k_ranges<<<(unsigned)((items + threads - 1) / threads), threads, 0, s>>>(keys, m, ranges);
}

void launch_keys64(const uint32_t* tiles, const uint32_t* ids, const Record* rec, int64_t m, uint64_t* out,
                   cudaStream_t s) {
  if (m == 0) return;
  const int threads = 256;
  k_keys64<<<(unsigned)((m + threads - 1) / threads), threads, 0, s>>>(tiles, ids, rec, m, out);
}

}  // namespace rade
