// Launchers for the PFT kernels; included once per precision by
// pft_launch_f32.cu / pft_launch_f64.cu (PFTG_REAL = float | double) so the two
// precisions compile in parallel.
#include <type_traits>

#include "internal.hpp"

namespace pftg {

namespace {

template <int V>
using IC = std::integral_constant<int, V>;

int rb_of(int r) {
  if (r <= 8) return 8;
  if (r <= 10) return 10;
  if (r <= 13) return 13;
  if (r <= 16) return 16;
  throw std::invalid_argument("pftg: GPU PFT supports r <= 16 coefficients per axis");
}

int slots_of(int p) {
  if (p <= 32) return 1;
  if (p == 64) return 2;
  if (p == 128) return 4;
  throw std::invalid_argument("pftg: GPU PFT supports power-of-two p in [2, 128]");
}

template <class F>
void dispatch_sr(int S, int RB, F&& f) {
  auto go = [&](auto s) {
    switch (RB) {
      case 8: f(s, IC<8>{}); break;
      case 10: f(s, IC<10>{}); break;
      case 13: f(s, IC<13>{}); break;
      default: f(s, IC<16>{}); break;
    }
  };
  switch (S) {
    case 1: go(IC<1>{}); break;
    case 2: go(IC<2>{}); break;
    default: go(IC<4>{}); break;
  }
}

template <class K>
void allow_smem(K kernel) {
  // one-time opt-in to the full 227 KB of dynamic shared memory per CTA
  PFTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
}

template <class R>
constexpr int rows_threads() { return sizeof(R) == 4 ? 512 : 256; }

}  // namespace

using R_ = PFTG_REAL;

template <>
void launch_fwd_rows<R_>(const PftDev<R_>& pd, const Src<R_>& src, typename CT<R_>::C* G, int batch,
                         cudaStream_t st) {
  const size_t smem = rows_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
  ProfScope prof(st, K_FWD_ROWS);
  dispatch_sr(slots_of(pd.p2), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    auto k = k_fwd_rows<R_, decltype(s)::value, decltype(rb)::value>;
    static bool once = (allow_smem(k), true);
    (void)once;
    k<<<dim3(pd.p1, batch), rows_threads<R_>(), smem, st>>>(pd, src, G);
  });
  PFTG_LAUNCH_CHECK();
}

template <>
int cols_strips<R_>(const PftDev<R_>& pd) {
  const int nb = strip_nb(pd.M2);
  return (pd.M2 + nb - 1) / nb;
}

template <>
void launch_fwd_cols<R_>(const PftDev<R_>& pd, int mode, const typename CT<R_>::C* G,
                         typename CT<R_>::C* band, const R_* dcrop, long long dstride,
                         typename CT<R_>::C* Gout, double* partial, int batch, cudaStream_t st) {
  const size_t smem = cols_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the cols pass (smem)");
  const dim3 grid(cols_strips(pd), batch);
  const R_* dc = dcrop;  // batch element f reads dcrop + f*dstride
  ProfScope prof(st, K_FWD_COLS);
  dispatch_sr(slots_of(pd.p1), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    constexpr int S = decltype(s)::value, RB = decltype(rb)::value;
    if (mode == 0) {
      auto k = k_fwd_cols<R_, S, RB, 0>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, 256, smem, st>>>(pd, G, band, dc, dstride, Gout, partial);
    } else if (mode == 1) {
      auto k = k_fwd_cols<R_, S, RB, 1>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, 256, smem, st>>>(pd, G, band, dc, dstride, Gout, partial);
    } else {
      auto k = k_fwd_cols<R_, S, RB, 2>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, 256, smem, st>>>(pd, G, band, dc, dstride, Gout, partial);
    }
  });
  PFTG_LAUNCH_CHECK();
}

template <>
void launch_adj_cols<R_>(const PftDev<R_>& pd, const typename CT<R_>::C* band, typename CT<R_>::C* Gt,
                         int batch, cudaStream_t st) {
  const size_t smem = cols_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the cols pass (smem)");
  ProfScope prof(st, K_ADJ_COLS);
  dispatch_sr(slots_of(pd.p1), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    auto k = k_adj_cols<R_, decltype(s)::value, decltype(rb)::value>;
    static bool once = (allow_smem(k), true);
    (void)once;
    k<<<dim3(cols_strips(pd), batch), 256, smem, st>>>(pd, band, Gt);
  });
  PFTG_LAUNCH_CHECK();
}

template <>
void launch_adj_rows<R_>(const PftDev<R_>& pd, int epi, const typename CT<R_>::C* Gt, const EpiArgs& ep,
                         int batch, cudaStream_t st) {
  const size_t smem = rows_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
  ProfScope prof(st, K_ADJ_ROWS);
  dispatch_sr(slots_of(pd.p2), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    constexpr int S = decltype(s)::value, RB = decltype(rb)::value;
    const dim3 grid(pd.p1, batch);
    if (epi == 0) {
      auto k = k_adj_rows<R_, S, RB, 0>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    } else if (epi == 1) {
      auto k = k_adj_rows<R_, S, RB, 1>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    } else {
      auto k = k_adj_rows<R_, S, RB, 2>;
      static bool once = (allow_smem(k), true);
      (void)once;
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    }
  });
  PFTG_LAUNCH_CHECK();
}

}  // namespace pftg
