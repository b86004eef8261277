// binning.cu — stage 2 (K2) of the RaDe-GS rasterizer, sm_100a.
//
//   K2a  inclusive scan of tiles_touched → offsets; M = offsets[n−1]
//   K2b  duplicate: for each Gaussian (id order) and each tile of its rect, emit
//        key = (tile << 32) | float_bits(z_c), value = id         (PAPER:422 depth sort)
//   K2c  stable LSD radix sort of (key, id) on bits [0, 32 + ceil(log2 T))
//   K2d  ranges[tile] = [first, last) in the sorted list
//
// z_c > znear > 0, so the IEEE bit pattern of z_c orders like its value; with the stable
// sort over input in id order the final order is (tile, z_c, id) — reading S7.
// Integer work: the result is checked bit-exactly against a CPU std::stable_sort.
#include "rade_internal.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace rade {
namespace {

// Warp-cooperative emission: a warp owns 32 consecutive Gaussians, whose outputs are
// contiguous in [start(first), end(last)). The warp walks that span 32 outputs at a time;
// output t belongs to the first lane whose inclusive warp-prefix exceeds t (a 5-step binary
// search over shuffled prefixes),
// whose rect / key are fetched by shuffle. Stores are fully coalesced and a large splat no
// longer serialises one thread. Per-Gaussian output order is row-major over its rect.
__global__ void __launch_bounds__(256) k_duplicate(int64_t n, const uint32_t* __restrict__ offsets,
                                                    const uint2* __restrict__ rect, const float* __restrict__ zkey,
                                                    int tiles_x, uint64_t* __restrict__ keys,
                                                    uint32_t* __restrict__ vals) {
  const int lane = (int)(threadIdx.x & 31);
  const int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  if (base >= n) return;  // whole warp out of range
  const int64_t i = base + lane;
  uint32_t start = 0, end = 0;
  if (i < n) {
    end = offsets[i];
    start = i == 0 ? 0u : offsets[i - 1];
  } else {
    end = start = offsets[n - 1];
  }
  const uint32_t cnt = end - start;
  uint32_t x0 = 0, y0 = 0, w = 1, zb = 0;
  if (cnt) {
    const uint2 r = rect[i];
    x0 = r.x & 0xffffu;
    y0 = r.x >> 16;
    w = (r.y & 0xffffu) - x0;
    zb = __float_as_uint(zkey[i]);
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t excl = incl - cnt;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t wstart = __shfl_sync(0xffffffffu, start, 0);
  for (uint32_t t0 = 0; t0 < total; t0 += 32) {
    const uint32_t t = t0 + lane;
    // owner = first lane whose inclusive prefix exceeds t (binary search over shuffled prefixes)
    int owner = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, owner + s - 1);
      if (v <= t) owner += s;
    }
    owner &= 31;
    const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, owner);
    const uint32_t o_x0 = __shfl_sync(0xffffffffu, x0, owner);
    const uint32_t o_y0 = __shfl_sync(0xffffffffu, y0, owner);
    const uint32_t o_w = __shfl_sync(0xffffffffu, w, owner);
    const uint32_t o_zb = __shfl_sync(0xffffffffu, zb, owner);
    if (t < total) {
      const uint32_t li = t - o_excl;
      const uint32_t ty = o_y0 + li / o_w, tx = o_x0 + li % o_w;
      const uint64_t tile = (uint64_t)ty * (uint64_t)tiles_x + tx;
      keys[wstart + t] = (tile << 32) | (uint64_t)o_zb;
      vals[wstart + t] = (uint32_t)(base + owner);
    }
  }
}

__global__ void __launch_bounds__(256) k_ranges(const uint64_t* __restrict__ keys, int64_t m,
                                                 uint2* __restrict__ ranges) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint32_t tile = (uint32_t)(keys[k] >> 32);
  if (k == 0 || (uint32_t)(keys[k - 1] >> 32) != tile) ranges[tile].x = (uint32_t)k;
  if (k == m - 1 || (uint32_t)(keys[k + 1] >> 32) != tile) ranges[tile].y = (uint32_t)(k + 1);
}

}  // namespace

size_t binning_scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return bytes;
}

void launch_scan(const uint32_t* tiles_touched, uint32_t* offsets, int64_t n, void* temp, size_t temp_bytes,
                 cudaStream_t s) {
  if (n == 0) return;
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, tiles_touched, offsets, (int)n, s);
}

void launch_duplicate(int64_t n, const uint32_t* offsets, const uint2* rect, const float* zkey, int tiles_x,
                      uint64_t* keys, uint32_t* vals, cudaStream_t s) {
  if (n == 0) return;
  const int threads = 256;
  k_duplicate<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(n, offsets, rect, zkey, tiles_x, keys, vals);
}

size_t binning_sort_temp_bytes(int64_t m, int end_bit) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint64_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)m, 0, end_bit);
  return bytes;
}

int launch_sort(uint64_t* keys0, uint64_t* keys1, uint32_t* vals0, uint32_t* vals1, int64_t m, int end_bit, void* temp,
                size_t temp_bytes, cudaStream_t s) {
  if (m == 0) return 0;
  cub::DoubleBuffer<uint64_t> k(keys0, keys1);
  cub::DoubleBuffer<uint32_t> v(vals0, vals1);
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)m, 0, end_bit, s);
  return k.selector;
}

void launch_ranges(const uint64_t* keys, int64_t m, int n_tiles, uint2* ranges, cudaStream_t s) {
  cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
  if (m == 0) return;
  const int threads = 256;
  k_ranges<<<(unsigned)((m + threads - 1) / threads), threads, 0, s>>>(keys, m, ranges);
}

}  // namespace rade
