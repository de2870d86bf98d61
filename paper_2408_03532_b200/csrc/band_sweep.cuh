// Persistent PFT-band ePIE sweep (blind, list order, complex64 q = 8 plans of
// BASELINE configs[2] / [3]): ONE cooperative launch per band sweep instead of
// four graph nodes per scan position. Per position j (solver.cpp:243-251):
//   cols    G -> band -> residual vs dcrop_j -> adjoint cols -> Gt     (k_fwd_cols_body MODE 1)
//   rows    Gt -> A-dagger -> z_j -= beta_pft conj(P) r; G = forward rows of P z_j   (EPI 1)
//   cols    G -> Gt
//   rows    Gt -> P -= gamma_pft conj(z_j) r2; G = forward rows of P z_{j+1}   (EPI 2, fused next)
// with a grid-wide barrier between the phases (esweep_barrier, 1.2 us). The
// work items run the same device bodies as the standalone kernels, so the
// trajectory is bit-identical; the forward rows pass of the sweep's first
// position is launched before this kernel.
#pragma once

#include "epie_sweep.cuh"
#include "pft_fast.cuh"

namespace pftg {

constexpr int kBandSweepThreads = 320;

template <class R, int Q, int RR, int P, int S1, int RB>
__global__ void __launch_bounds__(kBandSweepThreads, 1)
    kb_band_sweep(PftDev<R> pd, PftDev<R> pc, BPar<R, Q, RR> bp, typename CT<R>::C* frame, long long ld,
                  const long long* __restrict__ offs, int npos, typename CT<R>::C* probe, typename CT<R>::C* G,
                  typename CT<R>::C* Gt, const R* __restrict__ dcrop, long long mb, double beta_pft, double gamma_pft,
                  int vec_base, unsigned* bar) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int VV = sizeof(R) == 4 ? 2 : 1;
  unsigned target = 0;
  const int nstrips = (pc.M2 + pc.nb - 1) / pc.nb;
  auto cols = [&](const R* dc) {
    for (int bx = blockIdx.x; bx < nstrips; bx += gridDim.x)
      k_fwd_cols_body<R, S1, RB, 1>(pc, G, nullptr, dc, mb, Gt, nullptr, bx, 0, nstrips, smem_raw);
  };
  auto rows = [&](const EpiArgs& ep, auto epi_tag) {
    constexpr int EPI = decltype(epi_tag)::value;
    for (int t = blockIdx.x; t < pd.p1; t += gridDim.x) {
      if (ep.vec_ok) kf_adj_rows_body<R, Q, RR, P, VV, EPI, 1>(pd, bp, Gt, ep, t, 0, smem_raw);
      else kf_adj_rows_body<R, Q, RR, P, 1, EPI, 1>(pd, bp, Gt, ep, t, 0, smem_raw);
    }
  };
  for (int j = 0; j < npos; ++j) {
    const R* dc = dcrop + (size_t)j * mb;
    const long long off = offs[j];
    cols(dc);
    esweep_barrier(bar, target);
    EpiArgs ep{};
    ep.obj = frame;
    ep.obj_ld = ld;
    ep.obj_off = off;
    ep.probe = probe;
    ep.step = beta_pft;
    ep.G2 = G;
    ep.vec_ok = vec_base && (off % 2 == 0);
    rows(ep, std::integral_constant<int, 1>{});
    esweep_barrier(bar, target);
    cols(dc);
    esweep_barrier(bar, target);
    ep.step = gamma_pft;
    ep.G2 = j + 1 < npos ? G : nullptr;
    ep.obj_off2 = j + 1 < npos ? offs[j + 1] : 0;
    rows(ep, std::integral_constant<int, 2>{});
    esweep_barrier(bar, target);
  }
}

}  // namespace pftg
