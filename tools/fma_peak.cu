// Measured CUDA-core FMA peaks on this B200 (the compute denominators of the
// evaluator / cfg2 / ePIE flop rooflines, and of cfg1's FP64 check):
//   FFMA2  packed fma.rn.f32x2 (2 FP32 FMAs = 4 FLOP per lane per instruction)
//   FFMA   scalar fma.rn.f32
//   DFMA   fma.rn.f64
// 8 independent accumulator chains per thread, 148 x k CTAs of 256 threads,
// CUDA events around a timed launch after warm-up; prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_peak tools/fma_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;

__global__ void k_ffma2(float* out, float s) {
  unsigned long long a[8];
  const float x = threadIdx.x * 1e-7f;
  for (int k = 0; k < 8; ++k) {
    float2 v = make_float2(x + k, x - k);
    a[k] = *reinterpret_cast<unsigned long long*>(&v);
  }
  float2 bb = make_float2(s, s), cc = make_float2(1e-7f, -1e-7f);
  const unsigned long long b = *reinterpret_cast<unsigned long long*>(&bb);
  const unsigned long long c = *reinterpret_cast<unsigned long long*>(&cc);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(b), "l"(c));
  }
  float acc = 0;
  for (int k = 0; k < 8; ++k) {
    float2 v = *reinterpret_cast<float2*>(&a[k]);
    acc += v.x + v.y;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_ffma(float* out, float s) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(s), "f"(1e-7f));
  }
  float acc = 0;
  for (int k = 0; k < 8; ++k) acc += a[k];
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_dfma(double* out, double s) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7 + k;
  for (int i = 0; i < kIters / 8; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(s), "d"(1e-7));
  }
  double acc = 0;
  for (int k = 0; k < 8; ++k) acc += a[k];
  if (acc == 12345.0) out[0] = acc;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch();
  float best = 1e30f;
  for (int t = 0; t < 10; ++t) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* f;
  double* d;
  cudaMalloc(&f, 16);
  cudaMalloc(&d, 16);
  const int grid = sms * 8, block = 256;
  const double thr = (double)grid * block;
  const float t2 = best_ms([&] { k_ffma2<<<grid, block>>>(f, 0.999f); });
  const float t1 = best_ms([&] { k_ffma<<<grid, block>>>(f, 0.999f); });
  const float td = best_ms([&] { k_dfma<<<grid, block>>>(d, 0.999); });
  const double ffma2 = thr * kIters * 8 * 4 / (t2 * 1e-3) / 1e12;  // 2 FMA x 2 FLOP per lane-instruction
  const double ffma = thr * kIters * 8 * 2 / (t1 * 1e-3) / 1e12;
  const double dfma = thr * (kIters / 8) * 8 * 2 / (td * 1e-3) / 1e12;
  const double nominal = (double)sms * 128 * 2 * clk * 1e3 / 1e12;
  std::printf(
      "{\"fp32_ffma2_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f, \"sms\": %d, "
      "\"clock_mhz_attr\": %d, \"fp32_nominal_tflops\": %.2f, \"how\": \"%d CTAs x %d threads, 8 independent chains, "
      "best of 10 (CUDA events) after 3 warm-ups\"}\n",
      ffma2, ffma, dfma, sms, clk / 1000, nominal, grid, block);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
