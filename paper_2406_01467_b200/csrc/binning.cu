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

__global__ void __launch_bounds__(256) k_duplicate(int64_t n, const uint32_t* __restrict__ offsets,
                                                    const uint2* __restrict__ rect, const float* __restrict__ zkey,
                                                    int tiles_x, uint64_t* __restrict__ keys,
                                                    uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t end = offsets[i];
  const uint32_t start = i == 0 ? 0u : offsets[i - 1];
  if (start == end) return;
  const uint2 r = rect[i];
  const uint32_t x0 = r.x & 0xffffu, y0 = r.x >> 16, x1 = r.y & 0xffffu, y1 = r.y >> 16;
  const uint64_t zb = (uint64_t)__float_as_uint(zkey[i]);
  uint32_t o = start;
  for (uint32_t ty = y0; ty < y1; ++ty)
    for (uint32_t tx = x0; tx < x1; ++tx) {
      const uint64_t tile = (uint64_t)ty * (uint64_t)tiles_x + tx;
      keys[o] = (tile << 32) | zb;
      vals[o] = (uint32_t)i;
      ++o;
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
