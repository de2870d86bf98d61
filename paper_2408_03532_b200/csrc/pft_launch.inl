// Launchers for the PFT kernels; included by pft_launch_{f32,f64}_{fwd,adj,cols}.cu
// (PFTG_REAL = float | double; PFTG_PART = 1 forward rows, 2 adjoint rows,
// 3 cols passes) so the six kernel groups compile in parallel.
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include <cstdlib>

#include "internal.hpp"
#include "pft_fast.cuh"
#include "pft_tma.cuh"
#include "pft_cols.cuh"

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
  // one-time (per kernel and device) opt-in to the full 227 KB of dynamic shared memory per CTA
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({reinterpret_cast<const void*>(kernel), dev}).second)
    PFTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor in the stream drains; it calls
// griddep_wait() before touching global memory (tma.cuh). PFTG_NO_PDL=1: plain launch.
template <class... KA, class... A>
void launch_pdl(void (*kernel)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  const bool off = knobs().no_pdl;
  // not inside stream capture: the per-position ePIE graphs measured slower with programmatic edges
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (off || capturing) ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PFTG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

template <class R>
constexpr int rows_threads() { return sizeof(R) == 4 ? 512 : 256; }

// ---- specialized rows kernels (pft_fast.cuh) for the hot-path plan shapes ----
template <class R, int Q, int RR>
BPar<R, Q, RR> make_bpar(const PftDev<R>& pd) {
  BPar<R, Q, RR> b;
  for (int l = 0; l <= Q / 2; ++l)
    for (int j = 0; j < RR; ++j) {
      b.b1[l][j] = static_cast<R>(pd.hBv1[l * RR + j]);
      b.b2[l][j] = static_cast<R>(pd.hBv2[l * RR + j]);
    }
  return b;
}

// Calls f(IC<Q>, IC<RR>, IC<P>) when the (square) plan matches a specialized shape.
template <class R, class F>
bool dispatch_fast(const PftDev<R>& pd, F&& f) {
  if (pd.n1 != pd.n2 || pd.p1 != pd.p2 || pd.r1 != pd.r2 || pd.mt1 != pd.mt2 || pd.q1 != pd.q2) return false;
  const int q = pd.q1, r = pd.r1, p = pd.p1;
#define PFTG_FAST(QQ, RRR, PP)                      \
  if (q == QQ && r == RRR && p == PP) {             \
    f(IC<QQ>{}, IC<RRR>{}, IC<PP>{});               \
    return true;                                    \
  }
  if constexpr (sizeof(R) == 4) {
    PFTG_FAST(32, 10, 32)  // BASELINE cfg2 literal
    PFTG_FAST(8, 9, 32)    // cfg3 band (w=256, mt=p=32, eps 1e-3)
    PFTG_FAST(8, 9, 64)    // cfg4/5 band (w=512, mt=p=64)
    PFTG_FAST(8, 13, 64)   // scope-1 companion of cfg1 (eps 1e-7)
    PFTG_FAST(8, 13, 128)  // scope-1 companion of cfg2
  } else {
    PFTG_FAST(32, 12, 16)  // BASELINE cfg1 literal
    PFTG_FAST(32, 10, 32)  // cfg2 literal in complex128
    PFTG_FAST(8, 13, 64)   // scope-1 companion of cfg1
    PFTG_FAST(8, 9, 32)    // cfg3 band in complex128
    PFTG_FAST(8, 13, 8)    // SPEC ACC-4 dot-test shape (64^2, m~=p=8)
  }
#undef PFTG_FAST
  return false;
}

int sm_count() {
  int dev = 0, nsm = 148;
  PFTG_CUDA(cudaGetDevice(&dev));
  PFTG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  return nsm;
}

// The persistent cols kernels (pft_cols.cuh) handle this plan.
template <class R>
bool fast_cols_ok(const PftDev<R>& pd) {
  if (pd.M2 % kStripNB || pd.M1 * (kStripNB / 2) > kColsThreads * 8) return false;
  bool ok = false;
  dispatch_fast(pd, [&](auto, auto r, auto p) {
    constexpr int RR = decltype(r)::value, P = decltype(p)::value;
    ok = cols_fwd_smem<R>(P, RR, pd.M1) <= 227 * 1024 && cols_adj_smem<R>(P, RR, pd.M1) <= 227 * 1024 &&
         cols_fwd_local_smem<R>(RR, pd.M1) <= 227 * 1024 && cols_adj_local_smem<R>(RR, pd.M1) <= 227 * 1024 &&
         (P != kLocalP || pd.M1 <= 2 * 32 * kBandWarps);
  });
  return ok;
}

}  // namespace

using R_ = PFTG_REAL;

#ifndef PFTG_PART
#define PFTG_PART_FWD 1
#define PFTG_PART_ADJ 1
#define PFTG_PART_COLS 1
#else
#define PFTG_PART_FWD (PFTG_PART == 1)
#define PFTG_PART_ADJ (PFTG_PART == 2)
#define PFTG_PART_COLS (PFTG_PART == 3)
#endif

namespace {

#if PFTG_PART_FWD
bool fast_fwd_rows(const PftDev<R_>& pd, const Src<R_>& src, typename CT<R_>::C* G, int batch, cudaStream_t st) {
  return dispatch_fast(pd, [&](auto q, auto r, auto p) {
    constexpr int Q = decltype(q)::value, RR = decltype(r)::value, P = decltype(p)::value;
    const size_t smem = fast_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P);
    if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
    const auto bp = make_bpar<R_, Q, RR>(pd);
    const bool vec = sizeof(R_) == 4 && src.vec_ok && (pd.n2 % 2 == 0);
    constexpr int NT = fast_nt<RR, P>();
    if (vec) {
      auto k = kf_fwd_rows<R_, Q, RR, P, (sizeof(R_) == 4 ? 2 : 1)>;
      allow_smem(k);
      k<<<dim3(pd.p1, batch), NT, smem, st>>>(pd, bp, src, G);
    } else {
      auto k = kf_fwd_rows<R_, Q, RR, P, 1>;
      allow_smem(k);
      k<<<dim3(pd.p1, batch), NT, smem, st>>>(pd, bp, src, G);
    }
  });
}

// Persistent TMA-fed rows pass (pft_tma.cuh) for plain batched fields whose
// rows are whole 16-byte multiples and span exactly 512 x {1,2} columns.
bool tma_fwd_rows(const PftDev<R_>& pd, const Src<R_>& src, typename CT<R_>::C* G, int batch, cudaStream_t st,
                  bool strip) {
  const long long gstride = strip ? strip_field_elems(pd) : 0;
  const bool plain = !src.offs && !src.probe;  // scan windows / exit waves: warp-specialized kernel only
  // rows must share one 16-byte phase; windows off by 8 bytes (odd complex64
  // offsets) are handled by the one-column-per-consumer kernel (vc == 1)
  const bool base_ok = reinterpret_cast<uintptr_t>(src.base) % 16 == 0 && (src.ld * sizeof(typename CT<R_>::C)) % 16 == 0 &&
                       (src.bstride * sizeof(typename CT<R_>::C)) % 16 == 0 &&
                       (!src.probe || reinterpret_cast<uintptr_t>(src.probe) % 16 == 0);
  if (!base_ok) return false;
  if (knobs().no_tma) return false;
  int vc = 0;
  if (pd.n2 == kTmaConsumers) vc = 1;
  else if (sizeof(R_) == 4 && pd.n2 == 2 * kTmaConsumers) vc = 2;
  if (!vc || (vc == 2 && !src.vec_ok)) return false;
  bool launched = false;
  const bool matched = dispatch_fast(pd, [&](auto q, auto r, auto p) {
    constexpr int Q = decltype(q)::value, RR = decltype(r)::value, P = decltype(p)::value;
    int ns = 8;
    while (ns > 2 && tma_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns) > 227 * 1024) --ns;
    const size_t smem = tma_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns);
    if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the TMA rows pass");
    const auto bp = make_bpar<R_, Q, RR>(pd);
    int dev = 0, nsm = 148;
    PFTG_CUDA(cudaGetDevice(&dev));
    PFTG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int ntiles = pd.p1 * batch;
    const int grid = ntiles < nsm ? ntiles : nsm;
    const int dbg = knobs().debug_tma;
    if (knobs().tma_ns) ns = std::min(ns, knobs().tma_ns);
    // warp-specialized version when the double-buffered T still leaves >= 3 ring slots
    const bool wp = src.probe != nullptr;
    int ns2 = 12;
    while (ns2 > 3 && tma2_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns2, wp) > 227 * 1024) --ns2;
    if (knobs().tma_ns) ns2 = std::max(3, std::min(ns2, knobs().tma_ns));
    const int dbg2 = knobs().debug_ws;
    if constexpr (sizeof(R_) == 4 && Q == 32) {
      // wide variant: 256 group-A threads x 4 columns with setmaxnreg (plain complex64 fields, n2 = 1024)
      constexpr int AT = 256, NT = fwd_rows_threads<AT, RR, P>(true);
      constexpr int L = (65536 / NT) & ~7, RB = L < 72 ? L : 72;
      constexpr int RA0 = L + (((NT - AT) * (L - RB) / AT) & ~7), RA = RA0 > 248 ? 248 : RA0;
      const size_t smem2 = tma2_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns2, false);
      if (plain && src.vec_ok && pd.n2 == AT * 4 && !dbg && !knobs().no_ws && !knobs().no_wide &&
          smem2 <= 227 * 1024) {
        auto k = kt2_fwd_rows<R_, Q, RR, P, 4, AT, RA, RB>;
        cudaFuncAttributes fa{};
        PFTG_CUDA(cudaFuncGetAttributes(&fa, k));
        // the register hand-over must balance within the CTA's launch allocation
        if (fa.numRegs >= RB && fa.numRegs <= RA && AT * (RA - fa.numRegs) <= (NT - AT) * (fa.numRegs - RB)) {
          allow_smem(k);
          launch_pdl(k, grid, NT, smem2, st, pd, bp, src.base, src.ld, src.bstride, ntiles, ns2, G, gstride, dbg2,
                     (const long long*)nullptr, (const typename CT<R_>::C*)nullptr);
          launched = true;
          return;
        }
      }
    }
    if constexpr (sizeof(R_) == 4 && P == 64) {
      // q = 8 plans (p2 = 64, n2 = 512): two group-B warps per j1 (slot split); group A
      // becomes 256 threads x 2 columns so the block stays within 1024 threads
      constexpr int AT = 256, NT = fwd_rows_threads<AT, RR, P, 2>(false);
      const size_t smem2 = tma2_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns2, wp);
      if (pd.n2 == 2 * AT && NT <= 1024 && !dbg && !knobs().no_ws && !knobs().no_split && smem2 <= 227 * 1024) {
        auto k = kt2_fwd_rows<R_, Q, RR, P, 2, AT, 0, 0, 2>;
        {
          allow_smem(k);
          launch_pdl(k, grid, NT, smem2, st, pd, bp, src.base, src.ld, src.bstride, ntiles, ns2, G, gstride, dbg2,
                     src.offs, src.probe);
          launched = true;
          return;
        }
      }
    }
    if (!dbg && !knobs().no_ws && tma2_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns2, wp) <= 227 * 1024) {
      const size_t smem2 = tma2_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P, ns2, wp);
      constexpr int NT = kTmaConsumers + 32 * fwd_b_warps<RR, P>() + 32;
      auto k = kt2_fwd_rows<R_, Q, RR, P, (sizeof(R_) == 4 ? 2 : 1)>;
      if (vc == 2) {
        allow_smem(k);
        launch_pdl(k, grid, NT, smem2, st, pd, bp, src.base, src.ld, src.bstride, ntiles, ns2, G, gstride, dbg2,
                   src.offs, src.probe);
      } else {
        auto k1 = kt2_fwd_rows<R_, Q, RR, P, 1>;
        allow_smem(k1);
        launch_pdl(k1, grid, NT, smem2, st, pd, bp, src.base, src.ld, src.bstride, ntiles, ns2, G, gstride, dbg2,
                   src.offs, src.probe);
      }
      launched = true;
      return;
    }
    if (!plain || !src.vec_ok) return;  // the single-group kernels stream plain, aligned fields only
    launched = true;
    if (vc == 2) {
      auto k = kt_fwd_rows<R_, Q, RR, P, (sizeof(R_) == 4 ? 2 : 1)>;
      allow_smem(k);
      k<<<grid, kTmaConsumers + 32, smem, st>>>(pd, bp, src.base, src.ld, src.bstride, ntiles, ns, G, dbg,
                                                gstride);
    } else {
      auto k = kt_fwd_rows<R_, Q, RR, P, 1>;
      allow_smem(k);
      k<<<grid, kTmaConsumers + 32, smem, st>>>(pd, bp, src.base, src.ld, src.bstride, ntiles, ns, G, dbg,
                                                gstride);
    }
  });
  return matched && launched;
}

#endif  // PFTG_PART_FWD

#if PFTG_PART_ADJ
bool tma_adj_rows(const PftDev<R_>& pd, int epi, const typename CT<R_>::C* Gt, const EpiArgs& ep, int batch,
                  cudaStream_t st) {
  if (epi != 0 || !ep.vec_ok || knobs().no_tma) return false;
  // P2 owns column pairs (c64) or single columns (c128); any even n2 works
  const int vc = sizeof(R_) == 4 ? 2 : 1;
  if (pd.n2 % vc) return false;
  bool launched = false;
  const bool matched = dispatch_fast(pd, [&](auto q, auto r, auto p) {
    constexpr int Q = decltype(q)::value, RR = decltype(r)::value, P = decltype(p)::value;
    const size_t smem = tma_adj_smem<R_>(pd.n2, Q, RR, pd.M2, P);
    if (smem > 227 * 1024) return;  // double-buffered T does not fit: use kf_adj_rows
    const auto bp = make_bpar<R_, Q, RR>(pd);
    int dev = 0, nsm = 148;
    PFTG_CUDA(cudaGetDevice(&dev));
    PFTG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int ntiles = pd.p1 * batch;
    const int grid = ntiles < nsm ? ntiles : nsm;
    auto* out = reinterpret_cast<typename CT<R_>::C*>(ep.out);
    const int dbg = knobs().debug_adj;
    if constexpr (sizeof(R_) == 4 && Q == 32) {
      // wide variant: 8 P2 warps x 4 columns first, setmaxnreg hand-over (complex64, n2 = 1024)
      constexpr int P2T = 256, NT = adj_rows_threads<RR, P, P2T>(true);
      constexpr int L = (65536 / NT) & ~7, RB = L < 72 ? L : 72;
      constexpr int RA0 = L + (((NT - P2T) * (L - RB) / P2T) & ~7), RA = RA0 > 248 ? 248 : RA0;
      if (pd.n2 == P2T * 4 && (!dbg || knobs().debug_wide_adj) && !knobs().no_wide) {
        auto k = kt_adj_rows<R_, Q, RR, P, 4, P2T, RA, RB>;
        cudaFuncAttributes fa{};
        PFTG_CUDA(cudaFuncGetAttributes(&fa, k));
        if (fa.numRegs >= RB && fa.numRegs <= RA && P2T * (RA - fa.numRegs) <= (NT - P2T) * (fa.numRegs - RB)) {
          allow_smem(k);
          launch_pdl(k, grid, NT, smem, st, pd, bp, Gt, out, ntiles, dbg);
          launched = true;
          return;
        }
      }
    }
    constexpr int NT = 32 * (adj_p1_warps<RR, P>() + kAdjP2Warps);
    auto k = kt_adj_rows<R_, Q, RR, P, (sizeof(R_) == 4 ? 2 : 1)>;
    allow_smem(k);
    launch_pdl(k, grid, NT, smem, st, pd, bp, Gt, out, ntiles, dbg);
    launched = true;
  });
  return matched && launched;
}

bool fast_adj_rows(const PftDev<R_>& pd, int epi, const typename CT<R_>::C* Gt, const EpiArgs& ep, int batch,
                   cudaStream_t st) {
  return dispatch_fast(pd, [&](auto q, auto r, auto p) {
    constexpr int Q = decltype(q)::value, RR = decltype(r)::value, P = decltype(p)::value;
    constexpr int VV = sizeof(R_) == 4 ? 2 : 1;
    const size_t smem = fast_rows_smem<R_>(pd.n2, Q, RR, pd.M2, P);
    if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
    const auto bp = make_bpar<R_, Q, RR>(pd);
    const bool vec = sizeof(R_) == 4 && ep.vec_ok && (pd.n2 % 2 == 0);
    const dim3 grid(pd.p1, batch);
    // ePIE epilogues: prefetch the row block's probe / window rows when they fit
    const size_t smem_pf = smem + 16 + adj_prefetch_smem<R_>(pd.n2, Q);
    const bool pf = epi >= 1 && smem_pf <= 227 * 1024 && !knobs().no_prefetch;
    auto go = [&](auto kern, size_t sm) {
      allow_smem(kern);
      kern<<<grid, fast_nt<RR, P>(), sm, st>>>(pd, bp, Gt, ep);
    };
    if (epi == 0) {
      if (vec) go(kf_adj_rows<R_, Q, RR, P, VV, 0>, smem);
      else go(kf_adj_rows<R_, Q, RR, P, 1, 0>, smem);
    } else if (epi == 1) {
      if (pf) {
        if (vec) go(kf_adj_rows<R_, Q, RR, P, VV, 1, 1>, smem_pf);
        else go(kf_adj_rows<R_, Q, RR, P, 1, 1, 1>, smem_pf);
      } else {
        if (vec) go(kf_adj_rows<R_, Q, RR, P, VV, 1>, smem);
        else go(kf_adj_rows<R_, Q, RR, P, 1, 1>, smem);
      }
    } else {
      if (pf) {
        if (vec) go(kf_adj_rows<R_, Q, RR, P, VV, 2, 1>, smem_pf);
        else go(kf_adj_rows<R_, Q, RR, P, 1, 2, 1>, smem_pf);
      } else {
        if (vec) go(kf_adj_rows<R_, Q, RR, P, VV, 2>, smem);
        else go(kf_adj_rows<R_, Q, RR, P, 1, 2>, smem);
      }
    }
  });
}

#endif  // PFTG_PART_ADJ

}  // namespace

#if PFTG_PART_FWD
// complex64 q = 8, r = 9 plans: axis 2 first (kb_rows, eval_band.cu), for every batch size and
// source kind (batched fields, scan windows, exit waves); G in the row-block layout.
inline bool try_eb_fwd_rows(const PftDev<double>&, const Src<double>&, double2*, int, cudaStream_t) { return false; }
inline bool try_eb_fwd_rows(const PftDev<float>& pd, const Src<float>& src, float2* G, int batch, cudaStream_t st) {
  if (!eval_band_rows_ok(pd) || (knobs().eval_band_old & 1) || (reinterpret_cast<uintptr_t>(G) & 15)) return false;
  launch_eval_band_rows(pd, src.base, src.ld, src.bstride, src.offs, src.probe, G, batch, st);
  return true;
}

template <>
bool launch_fwd_rows<R_>(const PftDev<R_>& pd, const Src<R_>& src, typename CT<R_>::C* G, int batch,
                         cudaStream_t st, bool want_strip) {
  if (try_eb_fwd_rows(pd, src, G, batch, st)) return false;
  ProfScope prof(st, K_FWD_ROWS);
  // strip-major G only when the persistent cols kernel can consume it
  const bool strip = want_strip && fast_cols_ok(pd);
  if (tma_fwd_rows(pd, src, G, batch, st, strip)) {
    PFTG_LAUNCH_CHECK();
    return strip;
  }
  if (fast_fwd_rows(pd, src, G, batch, st)) {
    PFTG_LAUNCH_CHECK();
    return false;
  }
  const size_t smem = rows_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
  dispatch_sr(slots_of(pd.p2), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    auto k = k_fwd_rows<R_, decltype(s)::value, decltype(rb)::value>;
    allow_smem(k);
    k<<<dim3(pd.p1, batch), rows_threads<R_>(), smem, st>>>(pd, src, G);
  });
  PFTG_LAUNCH_CHECK();
  return false;
}

#endif  // PFTG_PART_FWD

#if PFTG_PART_COLS
template <>
long long g_field_elems<R_>(const PftDev<R_>& pd) {
  const long long rowblk = (long long)pd.p1 * pd.r1 * pd.M2;
  return fast_cols_ok(pd) ? std::max(rowblk, strip_field_elems(pd)) : rowblk;
}

template <>
int cols_strips<R_>(const PftDev<R_>& pd) {
  return (pd.M2 + pd.nb - 1) / pd.nb;
}

// complex64 p1 = 64, r = 9 plans (512-wide windows of the q = 8 family): radix-8
// shared-memory column transforms (eval_band.cu); 4-column strips for a single
// field (an ePIE position), 8 otherwise. MODE 2 partials keep the plan's strip count.
inline bool try_eb_cols(const PftDev<double>&, int, const double2*, double2*, const double*, long long, double2*,
                        double*, int, cudaStream_t) {
  return false;
}
inline bool try_eb_cols(const PftDev<float>& pd, int mode, const float2* G, float2* band, const float* dcrop,
                        long long dstride, float2* Gout, double* partial, int batch, cudaStream_t st) {
  const bool al = ((reinterpret_cast<uintptr_t>(G) | reinterpret_cast<uintptr_t>(Gout) |
                    reinterpret_cast<uintptr_t>(dcrop)) & 15) == 0 && dstride % 4 == 0;
  if (!al || !eval_band_cols_ok(pd) || (knobs().eval_band_old & 4) || (mode == 2 && pd.nb != 8)) return false;
  // one field: >= 32 CTAs (cfg3, M2 = 64: 2-column strips, band stage 56.5k -> 60.3k updates/s;
  // cfg4, M2 = 128: 4-column strips -- 2-column ones measured 2 % slower there)
  const int nb = (mode != 2 && batch == 1) ? ((mode == 1 && pd.M2 / 4 < 32) ? 2 : 4) : 8;
  launch_eval_band_cols(pd, nb, G, band, mode == 0 ? nullptr : dcrop, dstride, mode == 1 ? Gout : nullptr,
                        mode == 2 ? partial : nullptr, batch, st);
  return true;
}

template <>
void launch_fwd_cols<R_>(const PftDev<R_>& pd, int mode, const typename CT<R_>::C* G,
                         typename CT<R_>::C* band, const R_* dcrop, long long dstride,
                         typename CT<R_>::C* Gout, double* partial, int batch, cudaStream_t st,
                         bool strip) {
  if (strip) {
    // G in strip-major layout (written by the TMA rows pass): persistent cols kernel
    if (mode != 0) throw std::logic_error("pftg: strip-major G only feeds the plain forward cols pass");
    ProfScope prof(st, K_FWD_COLS);
    const bool ok = dispatch_fast(pd, [&](auto q, auto r, auto p) {
      constexpr int RR = decltype(r)::value, P = decltype(p)::value;
      const int nsf = pd.M2 / kStripNB, total = nsf * batch;
      int grid = std::min(total, 2 * sm_count());
      if (knobs().cols_grid) grid = std::min(total, knobs().cols_grid);
      if constexpr (P == kLocalP && sizeof(R_) == 4) {
        auto kl = kc_fwd_cols_local<R_, RR>;
        cudaFuncAttributes fa{};
        PFTG_CUDA(cudaFuncGetAttributes(&fa, kl));
        // setmaxnreg hand-over inside the kernel assumes the launch register count
        if (!knobs().no_local_cols && fa.numRegs == kColsRegLaunch) {
          allow_smem(kl);
          launch_pdl(kl, grid, 32 * (kFftWarps + kBandWarps), cols_fwd_local_smem<R_>(RR, pd.M1), st, pd, G,
                     (long long)strip_field_elems(pd), band, nsf, total, knobs().debug_cols);
          return;
        }
      }
      const size_t smem = cols_fwd_smem<R_>(P, RR, pd.M1);
      auto k = kc_fwd_cols<R_, RR, P>;
      allow_smem(k);
      launch_pdl(k, grid, kColsThreads, smem, st, pd, G, (long long)strip_field_elems(pd), band, nsf, total);
    });
    if (!ok) throw std::logic_error("pftg: strip-major G for an unspecialized plan");
    PFTG_LAUNCH_CHECK();
    return;
  }
  if (try_eb_cols(pd, mode, G, band, dcrop, dstride, Gout, partial, batch, st)) return;
  // Narrower strips when one launch covers few fields (an ePIE position): the
  // pass is latency-bound, so spread it over more SMs. MODE 2 keeps the plan's
  // strip count (its per-CTA partial sums are laid out by it).
  PftDev<R_> pl = pd;
  if (mode != 2)
    while (pl.nb > 1 && (long long)cols_strips(pl) * batch < 148) pl.nb /= 2;
  const size_t smem = cols_smem_bytes(pl);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the cols pass (smem)");
  const dim3 grid(cols_strips(pl), batch);
  const R_* dc = dcrop;  // batch element f reads dcrop + f*dstride
  ProfScope prof(st, K_FWD_COLS);
  dispatch_sr(slots_of(pd.p1), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    constexpr int S = decltype(s)::value, RB = decltype(rb)::value;
    if (mode == 0) {
      auto k = k_fwd_cols<R_, S, RB, 0>;
      allow_smem(k);
      k<<<grid, 256, smem, st>>>(pl, G, band, dc, dstride, Gout, partial);
    } else if (mode == 1) {
      if (pl.nb == 1 && pd.r1 > 8 && pd.r1 <= 10) {  // one warp per j1 (single-column strips)
        auto k = k_fwd_cols<R_, S, RB, 1, 320>;
        allow_smem(k);
        k<<<grid, 32 * pd.r1, smem, st>>>(pl, G, band, dc, dstride, Gout, partial);
      } else {
        auto k = k_fwd_cols<R_, S, RB, 1>;
        allow_smem(k);
        k<<<grid, 256, smem, st>>>(pl, G, band, dc, dstride, Gout, partial);
      }
    } else {
      auto k = k_fwd_cols<R_, S, RB, 2>;
      allow_smem(k);
      k<<<grid, 256, smem, st>>>(pl, G, band, dc, dstride, Gout, partial);
    }
  });
  PFTG_LAUNCH_CHECK();
}

template <>
void launch_adj_cols<R_>(const PftDev<R_>& pd, const typename CT<R_>::C* band, typename CT<R_>::C* Gt,
                         int batch, cudaStream_t st) {
  ProfScope prof(st, K_ADJ_COLS);
  if (fast_cols_ok(pd) && (long long)(pd.M2 / kStripNB) * batch >= 64 && !knobs().no_tma) {
    dispatch_fast(pd, [&](auto q, auto r, auto p) {
      constexpr int RR = decltype(r)::value, P = decltype(p)::value;
      const int nsf = pd.M2 / kStripNB, total = nsf * batch;
      const int grid = std::min(total, 2 * sm_count());
      if constexpr (P == kLocalP && sizeof(R_) == 4) {
        if (!knobs().no_local_cols && pd.M1 <= 256) {
          auto kl = kc_adj_cols_local<R_, RR>;
          allow_smem(kl);
          launch_pdl(kl, grid, kColsThreads, cols_adj_local_smem<R_>(RR, pd.M1), st, pd, band, Gt, nsf, total,
                     knobs().debug_adjcols);
          return;
        }
      }
      const size_t smem = cols_adj_smem<R_>(P, RR, pd.M1);
      auto k = kc_adj_cols<R_, RR, P>;
      allow_smem(k);
      launch_pdl(k, grid, kColsThreads, smem, st, pd, band, Gt, nsf, total);
    });
    PFTG_LAUNCH_CHECK();
    return;
  }
  PftDev<R_> pl = pd;
  while (pl.nb > 1 && (long long)cols_strips(pl) * batch < 148) pl.nb /= 2;
  const size_t smem = cols_smem_bytes(pl);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the cols pass (smem)");
  dispatch_sr(slots_of(pd.p1), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    auto k = k_adj_cols<R_, decltype(s)::value, decltype(rb)::value>;
    allow_smem(k);
    launch_pdl(k, dim3(cols_strips(pl), batch), 256, smem, st, pl, band, Gt);
  });
  PFTG_LAUNCH_CHECK();
}

#endif  // PFTG_PART_COLS

#if PFTG_PART_ADJ
// complex64 q = 8, r = 9 plans: one warp per output row, A-dagger on the band
// side, epilogue and fused forward in registers (eval_band.cu), for every batch size
// (the choice must not depend on how a host-buffer call or a multi-device call chunks the batch).
inline bool try_eb_adj_rows(const PftDev<double>&, int, const double2*, const EpiArgs&, int, cudaStream_t) {
  return false;
}
inline bool try_eb_adj_rows(const PftDev<float>& pd, int epi, const float2* Gt, const EpiArgs& ep, int batch,
                            cudaStream_t st) {
  if (!eval_band_adj_rows_ok(pd) || (knobs().eval_band_old & 8)) return false;  // any batch: results must not depend on chunking
  if ((reinterpret_cast<uintptr_t>(Gt) & 15) || (reinterpret_cast<uintptr_t>(ep.G2) & 15)) return false;
  launch_eval_band_adj_rows(pd, epi, Gt, ep, batch, st);
  return true;
}

template <>
void launch_adj_rows<R_>(const PftDev<R_>& pd, int epi, const typename CT<R_>::C* Gt, const EpiArgs& ep,
                         int batch, cudaStream_t st) {
  ProfScope prof(st, K_ADJ_ROWS);
  if (try_eb_adj_rows(pd, epi, Gt, ep, batch, st)) return;
  if (tma_adj_rows(pd, epi, Gt, ep, batch, st) || fast_adj_rows(pd, epi, Gt, ep, batch, st)) {
    PFTG_LAUNCH_CHECK();
    return;
  }
  const size_t smem = rows_smem_bytes(pd);
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: plan too large for the rows pass (smem)");
  dispatch_sr(slots_of(pd.p2), rb_of(std::max(pd.r1, pd.r2)), [&](auto s, auto rb) {
    constexpr int S = decltype(s)::value, RB = decltype(rb)::value;
    const dim3 grid(pd.p1, batch);
    if (epi == 0) {
      auto k = k_adj_rows<R_, S, RB, 0>;
      allow_smem(k);
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    } else if (epi == 1) {
      auto k = k_adj_rows<R_, S, RB, 1>;
      allow_smem(k);
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    } else {
      auto k = k_adj_rows<R_, S, RB, 2>;
      allow_smem(k);
      k<<<grid, rows_threads<R_>(), smem, st>>>(pd, Gt, ep);
    }
  });
  PFTG_LAUNCH_CHECK();
}

#endif  // PFTG_PART_ADJ

}  // namespace pftg
