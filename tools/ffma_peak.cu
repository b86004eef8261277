// ffma_peak.cu — measured FP32 FFMA throughput of this B200 (the roofline denominator of the
// ALU-bound blend kernels K3/K4: "the FP32 FFMA peak from our own
// microbenchmark").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma_peak.bin tools/ffma_peak.cu
//   tools/ffma_peak.bin > profiles/fp32_peak.json
//
// Every thread runs 8 independent FFMA chains (enough ILP to cover the 4-cycle FMA latency at
// full occupancy), 4096 iterations × 8 chains × 8 unrolled FFMAs; the grid is a multiple of
// the SM count at 2 × 1024-thread CTAs per SM. Result: flop = 2 × FFMAs executed, divided by
// the CUDA-event time of the launch (median of 9 launches after 3 warm-ups). The SM clock
// during the run is read from nvidia-smi by the caller (tools/gpu_peaks.sh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

constexpr int kIters = 4096;
constexpr int kChains = 8;
constexpr int kUnroll = 8;

__global__ void __launch_bounds__(1024, 2) k_ffma(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = (float)(threadIdx.x + c) * 1e-7f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(a), "f"(b));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[blockIdx.x] = s;  // never true; keeps the chains alive
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int blocks = sms * 2 * 8;  // 8 waves of 2 CTAs per SM
  const int threads = 1024;
  float* out = nullptr;
  cudaMalloc(&out, blocks * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_ffma<<<blocks, threads>>>(out, 0.9999f, 1e-6f);
  cudaDeviceSynchronize();
  std::vector<float> ms;
  for (int r = 0; r < 9; ++r) {
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, 0.9999f, 1e-6f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    ms.push_back(t);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(err));
    return 1;
  }
  std::sort(ms.begin(), ms.end());
  const double med = ms[ms.size() / 2];
  const double ffma = (double)blocks * threads * kIters * kUnroll * kChains;
  const double tflops = 2.0 * ffma / (med * 1e-3) / 1e12;
  // the formula peak at the attribute clock, for comparison
  const double formula = (double)sms * 128 * 2 * clk_khz * 1e3 / 1e12;
  printf("{\"fp32_ffma_tflops\": %.3f, \"median_ms\": %.4f, \"ffma_per_launch\": %.0f, \"sms\": %d, "
         "\"attr_clock_mhz\": %.0f, \"formula_tflops_at_attr_clock\": %.3f, \"launches\": %zu}\n",
         tflops, med, ffma, sms, clk_khz / 1e3, formula, ms.size());
  return 0;
}
