// ncu duration floor of a trivial kernel on this GPU (launch + one wave)
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (threadIdx.x == 1234567) p[0] = 1; }
int main() { int* p; cudaMalloc(&p, 4); for (int i = 0; i < 5; ++i) k_empty<<<256, 256>>>(p); cudaDeviceSynchronize(); return 0; }
