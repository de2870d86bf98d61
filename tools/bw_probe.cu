// HBM read-bandwidth probe for the rows-pass streaming structure (tool, not
// product code). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// gpurun_out/bw_probe tools/bw_probe.cu -I paper_2408_03532_b200/csrc
// Prints GB/s for: plain LDG.128 grid-stride reads; a persistent 1-CTA/SM
// bulk-copy ring (slot = 2 x 8 KB rows, like kt2_fwd_rows) at several depths;
// the same ring with 2 CTAs per SM.
#include <cstdio>
#include <cstdint>
#include <vector>
#include "tma.cuh"

using namespace pftg;

__global__ void k_ldg(const float4* __restrict__ x, size_t n, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(x + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// ntiles tiles of 32 rows x rowb bytes; slot = 2 rows
__global__ void k_ring(const char* __restrict__ z, int ntiles, int rowb, int NS, int ncons, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  char* ring = reinterpret_cast<char*>(sm) + 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int slotb = 2 * rowb;
  if (threadIdx.x >= ncons) {
    if (threadIdx.x != ncons) return;
    uint32_t seq = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int pi = 0; pi < 16; ++pi, ++seq) {
        const int s = seq % NS;
        if (seq >= (uint32_t)NS) mbar_wait(&empty[s], ((seq / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], 2 * rowb);
        const char* base = z + (size_t)t * 32 * rowb;
        bulk_g2s(ring + (size_t)s * slotb, base + (size_t)pi * rowb, rowb, &full[s]);
        bulk_g2s(ring + (size_t)s * slotb + rowb, base + (size_t)(31 - pi) * rowb, rowb, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (int pi = 0; pi < 16; ++pi) {
      mbar_wait(&full[s], ph);
      const float4 v = *reinterpret_cast<const float4*>(ring + (size_t)s * slotb + 16 * threadIdx.x);
      acc += v.x;
      mbar_arrive(&empty[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)36 << 23;  // 36 fields of 1024^2 complex64 (302 MB)
  char* z;
  float* out;
  cudaMalloc(&z, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(z, 0, bytes);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes / (ms / 20 * 1e-3) / 1e9;
  };
  for (int bpsm : {4, 8, 16}) {
    const double gbs = timeit([&] { k_ldg<<<nsm * bpsm, 256>>>((const float4*)z, bytes / 16, out); });
    printf("ldg128 grid=%d x 256: %.0f GB/s\n", nsm * bpsm, gbs);
  }
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int rowb = 8192, ntiles = (int)(bytes / (32 * rowb));
  for (int ctas : {1, 2})
    for (int NS : {4, 6, 8, 12}) {
      const size_t smem = 1024 + (size_t)NS * 2 * rowb;
      if (smem * ctas > 228 * 1024) continue;
      const int ncons = 512;  // 16 B per consumer thread per slot row
      const double gbs = timeit([&] { k_ring<<<nsm * ctas, ncons + 32, smem>>>(z, ntiles, rowb, NS, ncons, out); });
      printf("ring ctas/SM=%d NS=%d (%d KB in flight/SM): %.0f GB/s\n", ctas, NS, ctas * NS * 2 * rowb / 1024, gbs);
    }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
