// Cost of one grid-wide barrier (148 co-resident CTAs x 256 threads, atomic
// arrive with release + acquire spin) on this GPU: K barriers in one launch.
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_barriers(unsigned* ctr, int K, int* sink) {
  unsigned target = 0;
  int acc = 0;
  for (int k = 0; k < K; ++k) {
    acc += threadIdx.x ^ k;
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
  }
  if (acc == 123456789) sink[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* ctr;
  int* sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int K : {1, 10000}) {
    cudaMemset(ctr, 0, 4);
    void* args[] = {&ctr, &K, &sink};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_barriers, dim3(sms), dim3(256), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("{\"ctas\": %d, \"barriers\": %d, \"us_total\": %.2f, \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n", sms, K,
                1e3 * ms, 1e3 * ms / K, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
