// PCIe probe: pinned host <-> device copy rates, one direction alone and both
// directions at once, over a range of copy sizes (the e2e host pipeline's
// ceiling).  nvcc -O2 -o tools/pcie_probe tools/pcie_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  const size_t total = 512ull << 20;
  char *h_in, *h_out, *d_in, *d_out;
  CK(cudaMallocHost(&h_in, total));
  CK(cudaMallocHost(&h_out, total));
  CK(cudaMalloc(&d_in, total));
  CK(cudaMalloc(&d_out, total));
  for (size_t i = 0; i < total; i += 4096) h_in[i] = 1, h_out[i] = 1;
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const size_t sizes[] = {1ull << 20, 4ull << 20, 8ull << 20, 16ull << 20, 32ull << 20, 64ull << 20};
  for (int rep = 0; rep < 2; ++rep)
    for (size_t cs : sizes) {
      float ms[3];
      for (int mode = 0; mode < 3; ++mode) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, 0));
        CK(cudaStreamWaitEvent(s0, a));
        CK(cudaStreamWaitEvent(s1, a));
        for (size_t o = 0; o < total; o += cs) {
          if (mode != 1) CK(cudaMemcpyAsync(d_in + o, h_in + o, cs, cudaMemcpyHostToDevice, s0));
          if (mode != 0) CK(cudaMemcpyAsync(h_out + o, d_out + o, cs, cudaMemcpyDeviceToHost, s1));
        }
        cudaEvent_t j;
        CK(cudaEventCreate(&j));
        CK(cudaEventRecord(j, s1));
        CK(cudaStreamWaitEvent(s0, j));
        CK(cudaEventRecord(b, s0));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms[mode], a, b));
        cudaEventDestroy(j);
      }
      if (rep)
        printf("chunk %3zu MB: H2D %.1f GB/s, D2H %.1f GB/s, both %.1f + %.1f GB/s (%.2f ms for 512+512 MB)\n", cs >> 20,
               total / ms[0] / 1e6, total / ms[1] / 1e6, total / ms[2] / 1e6, total / ms[2] / 1e6, ms[2]);
    }
  // the cfg2 streamed call's copy pattern (64 fields: 8 MiB in; 8 MiB + 0.5 MiB
  // out per field) without compute: one stream per direction, chunk = c fields
  const size_t fz = 8ull << 20, fb = 512ull << 10;
  for (int c : {1, 2, 4, 8}) {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, 0));
      CK(cudaStreamWaitEvent(s0, a));
      CK(cudaStreamWaitEvent(s1, a));
      for (int f = 0; f < 64; f += c) {
        CK(cudaMemcpyAsync(d_in + f * fz % total, h_in + f * fz % total, c * fz, cudaMemcpyHostToDevice, s0));
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, s0));
        CK(cudaStreamWaitEvent(s1, ev));
        CK(cudaMemcpyAsync(h_out + f * fz % total, d_out + f * fz % total, c * fz, cudaMemcpyDeviceToHost, s1));
        CK(cudaMemcpyAsync(h_out + f * fb, d_out + f * fb, c * fb, cudaMemcpyDeviceToHost, s1));
        cudaEventDestroy(ev);
      }
      cudaEvent_t j;
      CK(cudaEventCreate(&j));
      CK(cudaEventRecord(j, s1));
      CK(cudaStreamWaitEvent(s0, j));
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = ms < best ? ms : best;
      cudaEventDestroy(j);
    }
    printf("cfg2 copy pattern, %d fields per chunk: %.2f ms = %.0f transforms/s ceiling\n", c, best, 128 / best * 1e3);
  }
  return 0;
}
