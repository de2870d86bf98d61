// Launchers for the full 2-D FFT passes; included once per precision by
// fft_launch_f32.cu / fft_launch_f64.cu (PFTG_REAL = float | double).
#include <cmath>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "internal.hpp"

namespace pftg {

namespace {

template <int V>
using IC = std::integral_constant<int, V>;

template <class F>
void dispatch_slots(int S, F&& f) {
  switch (S) {
    case 1: f(IC<1>{}); break;
    case 2: f(IC<2>{}); break;
    case 4: f(IC<4>{}); break;
    case 8: f(IC<8>{}); break;
    case 16: f(IC<16>{}); break;
    case 32: f(IC<32>{}); break;
    default: throw std::invalid_argument("pftg: FFT length out of range");
  }
}

template <class K>
void allow_smem_fft(K kernel) {
  // one-time (per kernel and device) opt-in to 227 KB of dynamic shared memory
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({reinterpret_cast<const void*>(kernel), dev}).second)
    PFTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
}

int slots_for(int n) { return n <= 32 ? 1 : n / 32; }

}  // namespace

using R_ = PFTG_REAL;
using C_ = typename CT<R_>::C;

template <>
const C_* fft_twiddles<R_>(int n) {
  // One device table per (device, length); built once, never freed (tiny).
  static std::mutex mu;
  static C_* tabs[64][11] = {};
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  const int lg = ilog2(n);
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 64) throw std::runtime_error("pftg: device index out of range");
  if (!tabs[dev][lg]) {
    const int h = n / 2 > 0 ? n / 2 : 1;
    std::vector<C_> host(static_cast<size_t>(h));
    for (int k = 0; k < h; ++k) {
      const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
      host[k] = CT<R_>::mk(static_cast<R_>(std::cos(a)), static_cast<R_>(std::sin(a)));
    }
    C_* d = nullptr;
    PFTG_CUDA(cudaMalloc(&d, sizeof(C_) * h));
    PFTG_CUDA(cudaMemcpyAsync(d, host.data(), sizeof(C_) * h, cudaMemcpyHostToDevice, cudaStreamPerThread));
    PFTG_CUDA(cudaStreamSynchronize(cudaStreamPerThread));  // before any non-blocking stream reads it
    tabs[dev][lg] = d;
  }
  return tabs[dev][lg];
}

template <>
void launch_fft_rows<R_>(int mode, int epi, int n1, int n2, const RowSrc<R_>& src, C_* X, long long x_bstride,
                         int sign, double scale, const RowEpiArgs& ep, int batch, cudaStream_t st) {
  const C_* tw = fft_twiddles<R_>(n2);
  const int S = slots_for(n2);
  const int P = n2 / S;
  // Small batches (one ePIE position) get narrower CTAs so the pass spreads
  // over the SMs instead of queueing rows behind a few blocks.
  int threads = 256;
  while (threads > 64 && (long long)((n1 + threads / 32 * (32 / P) - 1) / (threads / 32 * (32 / P))) * batch < 2 * 148)
    threads /= 2;
  const int rows_per_cta = threads / 32 * (32 / P);
  const dim3 grid((n1 + rows_per_cta - 1) / rows_per_cta, batch);
  size_t smem = sizeof(C_) * (n2 / 2 + 1);
  // ROW_DIT_NATURAL stages each row in shared memory for its bit-reversed gather
  if (mode == ROW_DIT_NATURAL) smem = sizeof(C_) * (((n2 / 2 + 2) & ~1) + (size_t)rows_per_cta * n2);
  ProfScope prof(st, K_FFT_ROWS);
  dispatch_slots(S, [&](auto s) {
    constexpr int SS = decltype(s)::value;
    if (mode == ROW_DIF_STORE) {
      k_fft_rows<R_, SS, ROW_DIF_STORE, EPI_STORE><<<grid, threads, smem, st>>>(n1, n2, ilog2(n2), tw, src, X,
                                                                           x_bstride, sign, scale, ep);
    } else if (mode == ROW_DIT_NATURAL) {
      auto k = k_fft_rows<R_, SS, ROW_DIT_NATURAL, EPI_STORE>;
      allow_smem_fft(k);
      k<<<grid, threads, smem, st>>>(n1, n2, ilog2(n2), tw, src, X, x_bstride, sign, scale, ep);
    } else if (epi == EPI_STORE) {
      k_fft_rows<R_, SS, ROW_DIT_PROJ, EPI_STORE><<<grid, threads, smem, st>>>(n1, n2, ilog2(n2), tw, src, X,
                                                                          x_bstride, sign, scale, ep);
    } else if (epi == EPI_OBJ) {
      k_fft_rows<R_, SS, ROW_DIT_PROJ, EPI_OBJ><<<grid, threads, smem, st>>>(n1, n2, ilog2(n2), tw, src, X,
                                                                        x_bstride, sign, scale, ep);
    } else {
      k_fft_rows<R_, SS, ROW_DIT_PROJ, EPI_PROBE><<<grid, threads, smem, st>>>(n1, n2, ilog2(n2), tw, src, X,
                                                                          x_bstride, sign, scale, ep);
    }
  });
  PFTG_LAUNCH_CHECK();
}

template <>
int fft_cols_strips<R_>(int n2) {
  const int nc0 = sizeof(R_) == 4 ? 16 : 8;
  const int nc = n2 < nc0 ? n2 : nc0;
  return n2 / nc;
}

template <>
void launch_fft_cols<R_>(int mode, int n1, int n2, C_* X, long long x_bstride, const R_* d, long long d_bstride,
                         const long long* d_index, int dmode, int sign, double* partial, int batch,
                         cudaStream_t st) {
  const C_* tw = fft_twiddles<R_>(n1);
  const int S = slots_for(n1);
  const int nc0 = sizeof(R_) == 4 ? 16 : 8;
  int nc = n2 < nc0 ? n2 : nc0;
  // Narrow strips for small batches (ePIE positions); the evaluation modes keep
  // the fixed strip count their per-CTA partial sums are laid out by.
  if (mode == COL_PROJECT || mode == COL_NATURAL)
    while (nc > 2 && (long long)(n2 / nc) * batch < 148) nc /= 2;
  const int threads = std::max(64, std::min(256, nc * (n1 / S)));  // one lane group per column
  const dim3 grid(n2 / nc, batch);
  size_t smem = sizeof(C_) * ((size_t)n1 * (nc + 1) + n1 / 2 + 1);
  if (mode != COL_NATURAL && dmode == 0) smem += sizeof(R_) * (size_t)n1 * (nc + 1);
  smem = (smem + 15) & ~size_t(15);
  if (smem < 64 * sizeof(double)) smem = 64 * sizeof(double);
  ProfScope prof(st, K_FFT_COLS);
  dispatch_slots(S, [&](auto s) {
    constexpr int SS = decltype(s)::value;
    if (mode == COL_PROJECT) {
      auto k = k_fft_cols<R_, SS, COL_PROJECT>;
      allow_smem_fft(k);
      k<<<grid, threads, smem, st>>>(n1, n2, ilog2(n1), ilog2(n2), nc, tw, X, x_bstride, d, d_bstride, d_index,
                                 dmode, sign, partial);
    } else if (mode == COL_EVAL) {
      auto k = k_fft_cols<R_, SS, COL_EVAL>;
      allow_smem_fft(k);
      k<<<grid, threads, smem, st>>>(n1, n2, ilog2(n1), ilog2(n2), nc, tw, X, x_bstride, d, d_bstride, d_index,
                                 dmode, sign, partial);
    } else if (mode == COL_EVAL_NAT) {
      auto k = k_fft_cols<R_, SS, COL_EVAL_NAT>;
      allow_smem_fft(k);
      k<<<grid, threads, smem, st>>>(n1, n2, ilog2(n1), ilog2(n2), nc, tw, X, x_bstride, d, d_bstride, d_index,
                                 dmode, sign, partial);
    } else {
      auto k = k_fft_cols<R_, SS, COL_NATURAL>;
      allow_smem_fft(k);
      k<<<grid, threads, smem, st>>>(n1, n2, ilog2(n1), ilog2(n2), nc, tw, X, x_bstride, d, d_bstride, d_index,
                                 dmode, sign, partial);
    }
  });
  PFTG_LAUNCH_CHECK();
}

}  // namespace pftg
