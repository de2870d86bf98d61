// Host-side internals shared by the CUDA translation units of libpftg.
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "fft_kernels.cuh"
#include "host.hpp"
#include "pft_kernels.cuh"

namespace pftg {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
#define PFTG_CUDA(x)                                                        \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) ::pftg::throw_cuda(e_, #x, __FILE__, __LINE__);  \
  } while (0)
#define PFTG_LAUNCH_CHECK() PFTG_CUDA(cudaGetLastError())

// Runtime switches, read from the environment ONCE per process (knobs()):
// alternative (correct) kernel choices used for A/B measurements, and -- in a
// -DPFTG_PROFILING build only -- the stage-skipping profiling experiments
// (debug_*), which are forced to 0 in the product build. PFTG_CHUNK_MB (the G
// budget per chunk) is the one knob read per call (chunk_fields in capi.cu).
struct Knobs {
  bool no_pdl, no_tma, no_ws, no_wide, no_split, no_local_cols, eval_lanefft, epie_lanefft;
  int tma_ns, cols_grid;  // 0 = unset
  int eval_chunk;         // evaluator positions per chunk (0 = 64 MB of spectra)
  int eval_pchunk;        // evaluator positions per band-chain chunk (0 = 2 x eval chunk)
  bool eval_one_stream;   // evaluator: FFT and PFT chains on one stream
  int eval_band_old;      // eval_band.cu off: bit 0 = forward rows (evaluator, launch_fwd_rows), bit 1 = evaluator cols, bit 2 = launch_fwd_cols, bit 3 = launch_adj_rows (ePIE band stage, pft_apply_2d / pft_adjoint_2d)
  bool no_tile, force_tile;  // small-batch tile path (pft_tile.cu): off / forced
  int host_chunk_mb;         // host-buffer pipelines: MB per copy (0 = 32)
  bool no_persist;           // ePIE full-FFT stage: per-position kernel graph instead of the persistent sweep
  bool no_prefetch;          // ePIE adjoint-rows epilogue without the shared-memory prefetch
  int debug_tma, debug_ws, debug_adj, debug_cols, debug_adjcols;
  bool debug_wide_adj;
};
const Knobs& knobs();

template <class R>
struct DevTables {
  R* Bv1 = nullptr;
  R* Bv2 = nullptr;
  typename CT<R>::C* W1t = nullptr;
  typename CT<R>::C* W2t = nullptr;
  typename CT<R>::C* tw1 = nullptr;
  typename CT<R>::C* tw2 = nullptr;
};

}  // namespace pftg

namespace pftg {
// Device copy of a plan's tables on one device, in one precision.
template <class R>
struct DevPlan {
  DevTables<R> t;
  PftDev<R> pd{};
};
}  // namespace pftg

// pft::PftPlan2D (pft.hpp:44-47): host tables + lazily uploaded device tables,
// one immutable copy per (device, precision): a plan shared by threads that
// drive different GPUs never frees tables another thread may still read.
struct pftg_plan {
  pftg::Axis a1, a2;
  mutable std::mutex mu;
  mutable std::map<int, std::unique_ptr<pftg::DevPlan<float>>> dev32;
  mutable std::map<int, std::unique_ptr<pftg::DevPlan<double>>> dev64;
  mutable std::vector<double> hbv1, hbv2;  // nonzero parts of B1, B2 (host; kernel-parameter tables)
  ~pftg_plan();
};

struct pftg_table {
  pftg::Table t;
};

namespace pftg {

// Validates the GPU constraints and returns the device descriptor (uploads
// the tables on first use).
template <class R>
const PftDev<R>& plan_dev(const pftg_plan& p);

// ---- PFT building blocks (pft_launch_*.cu); all stream-ordered ----
// Returns true when G was written in the strip-major layout (only if
// want_strip and the persistent cols kernel handles the plan); pass that
// flag to launch_fwd_cols.
template <class R>
bool launch_fwd_rows(const PftDev<R>& pd, const Src<R>& src, typename CT<R>::C* G, int batch,
                     cudaStream_t st, bool want_strip = false);
// mode 0: band out; 1: residual -> Gout; 2: evaluator partials [batch][cols_strips]
template <class R>
void launch_fwd_cols(const PftDev<R>& pd, int mode, const typename CT<R>::C* G, typename CT<R>::C* band,
                     const R* dcrop, long long dstride, typename CT<R>::C* Gout, double* partial, int batch,
                     cudaStream_t st, bool strip = false);
// G elements per field needed by either layout
template <class R>
long long g_field_elems(const PftDev<R>& pd);
template <class R>
int cols_strips(const PftDev<R>& pd);
template <class R>
void launch_adj_cols(const PftDev<R>& pd, const typename CT<R>::C* band, typename CT<R>::C* Gt, int batch,
                     cudaStream_t st);
template <class R>
void launch_adj_rows(const PftDev<R>& pd, int epi, const typename CT<R>::C* Gt, const EpiArgs& ep,
                     int batch, cudaStream_t st);

// ---- evaluator band chain for the q = 8, r = 9 complex64 plans (eval_band.cu) ----
// Axis 2 first: rows -> G[f][k1][j1][b] (the row-block layout of launch_fwd_rows),
// cols (strips of nb = 8 or 4 columns) -> band / residual partials [batch][M2 / nb] / residual + adjoint cols -> Gout.
bool eval_band_rows_ok(const PftDev<float>& pd);
bool eval_band_cols_ok(const PftDev<float>& pd);
void launch_eval_band_rows(const PftDev<float>& pd, const float2* frame, long long ld, long long bstride,
                           const long long* offs, const float2* probe, float2* G, int batch, cudaStream_t st);
void launch_eval_band_cols(const PftDev<float>& pd, int nb, const float2* G, float2* band, const float* dcrop,
                           long long dstride, float2* Gout, double* partial, int batch, cudaStream_t st);

// adjoint rows (+ ePIE epilogues and the fused forward rows pass), axis 1 first; Gt in the row-block layout
bool eval_band_adj_rows_ok(const PftDev<float>& pd);
void launch_eval_band_adj_rows(const PftDev<float>& pd, int epi, const float2* Gt, const EpiArgs& ep, int batch,
                               cudaStream_t st);

// ---- small-batch tile path (pft_tile.cu) ----
template <class R>
bool tile_path_ok(const PftDev<R>& pd, std::size_t batch);
template <class R>
void tile_apply(const PftDev<R>& pd, const void* z, long long bstride, void* band, int batch, cudaStream_t st);
template <class R>
void tile_adjoint(const PftDev<R>& pd, const void* band, void* z, long long bstride, int batch, cudaStream_t st);

// ---- full FFT building blocks (fft_launch_*.cu) ----
template <class R>
const typename CT<R>::C* fft_twiddles(int n);  // device table exp(-2 pi i k/n), k < n/2
template <class R>
void launch_fft_rows(int mode, int epi, int n1, int n2, const RowSrc<R>& src, typename CT<R>::C* X,
                     long long x_bstride, int sign, double scale, const RowEpiArgs& ep, int batch,
                     cudaStream_t st);
template <class R>
void launch_fft_cols(int mode, int n1, int n2, typename CT<R>::C* X, long long x_bstride, const R* d,
                     long long d_bstride, const long long* d_index, int dmode, int sign,
                     double* partial, int batch, cudaStream_t st);
template <class R>
int fft_cols_strips(int n2);

// Stream-ordered scratch allocation (cudaMallocAsync on the default pool).
struct Scratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  Scratch() = default;
  Scratch(std::size_t bytes, cudaStream_t s);
  ~Scratch();
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

void ensure_device();
void set_error(const std::string& m);  // thread-local message behind pftg_last_error (capi.cu)
void check_fft_len(std::size_t n);

// Optional per-kernel timing (pftg_profile_*): CUDA events recorded around
// each launch on its own stream while profiling is on (never inside a graph
// capture). Kernel ids:
enum KernelId { K_FWD_ROWS = 0, K_FWD_COLS, K_ADJ_COLS, K_ADJ_ROWS, K_FFT_ROWS, K_FFT_COLS, K_NUM };
// launch counters: snapshot (K_NUM ints) and credit replays of a captured graph
void prof_launch_snapshot(int* out);
void prof_add_launches(const int* delta);
struct ProfScope {
  int kid;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  ProfScope(cudaStream_t s, int k);
  ~ProfScope();
};

}  // namespace pftg
