// Device-side timing of the cfg1 step (one 512^2 complex128 field, forward +
// adjoint) straight through the C-ABI, without Python in the loop:
//   eager: K back-to-back (apply, adjoint) pairs on one stream, CUDA events;
//   graph: the pair captured once into a CUDA graph, K replays.
// Build: g++ -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include tools/cfg1_time.cpp \
//          -Lpaper_2408_03532_b200 -lpftg -L/usr/local/cuda/lib64 -lcudart \
//          -Wl,-rpath,'$ORIGIN/../paper_2408_03532_b200' -o tools/cfg1_time
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pftg.h"

#define CK(x)                                                                    \
  do {                                                                           \
    int rc_ = (x);                                                               \
    if (rc_) {                                                                   \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, rc_, pftg_last_error()); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(int argc, char** argv) {
  const char* table = argc > 1 ? argv[1] : "paper_2408_03532_b200/data/scope_table_xi4_r12.txt";
  const int K = argc > 2 ? std::atoi(argv[2]) : 200;
  pftg_table* t = nullptr;
  pftg_plan* p = nullptr;
  CK(pftg_table_load(table, &t));
  CK(pftg_plan_2d(t, 512, 512, 64, 64, 16, 16, 1.0, &p));
  const size_t nz = 512 * 512, nb = 128 * 128;
  std::vector<double> hz(2 * nz);
  for (size_t i = 0; i < hz.size(); ++i) hz[i] = (double)((i * 2654435761u) % 1000) / 500.0 - 1.0;
  void *z, *b, *y;
  cudaMalloc(&z, 16 * nz);
  cudaMalloc(&b, 16 * nb);
  cudaMalloc(&y, 16 * nz);
  cudaMemcpy(z, hz.data(), 16 * nz, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < 20; ++i) {
    CK(pftg_apply_2d_dev(p, PFTG_C128, z, b, 1, st));
    CK(pftg_adjoint_2d_dev(p, PFTG_C128, b, y, 1, st));
  }
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < K; ++i) {
    CK(pftg_apply_2d_dev(p, PFTG_C128, z, b, 1, st));
    CK(pftg_adjoint_2d_dev(p, PFTG_C128, b, y, 1, st));
  }
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms_eager;
  cudaEventElapsedTime(&ms_eager, e0, e1);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  CK(pftg_apply_2d_dev(p, PFTG_C128, z, b, 1, st));
  CK(pftg_adjoint_2d_dev(p, PFTG_C128, b, y, 1, st));
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(e0, st);
  for (int i = 0; i < K; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms_graph;
  cudaEventElapsedTime(&ms_graph, e0, e1);
  std::printf("{\"eager_us_per_step\": %.2f, \"graph_us_per_step\": %.2f, \"steps\": %d, \"err\": \"%s\"}\n",
              1e3 * ms_eager / K, 1e3 * ms_graph / K, K, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
