// 2-D fast Partial Fourier Transform: forward, adjoint and the fused
// band-residual, as sm_100a CUDA kernels.
//
// Reference: /root/reference/proj/core/src/pft.cpp
//   pft_apply_2d   (pft.cpp:119-172): stage A  T = B1^T Z_blk        (133-136)
//                                     stage B  C = M B2              (137-144)
//                                     stage C  2-D FFT over (k1,k2)  (147)
//                                     stage D  band assembly         (149-170)
//   pft_adjoint_2d (pft.cpp:174-226): D^dagger, backward FFT, B^dagger, A^dagger.
//
// The operator is the tensor product of two 1-D PFT matrices, so the GPU
// evaluates it in two separable passes that each touch HBM once:
//
//   pass "rows"  (one CTA per (field, k1)): reads the q1 x n2 row block once,
//       stage A on the fly (T = B1^T Z_blk, T kept in shared memory),
//       stage B + the k2-FFT + the axis-2 half of stage D in registers:
//         G[k1][j1][b] = sum_j2 W2[b][j2] * FFT_k2( C[k1][k2][j1][j2] )[u2(b)]
//   pass "cols"  (one CTA per (field, strip of nb band columns)):
//         out[a][b] = sum_j1 W1[a][j1] * FFT_k1( G[k1][j1][b] )[u1(a)]
//
// Only the linear maps are re-associated (FFT over k1 moved after the j2
// contraction); the arithmetic per term is the reference's. B entries are
// purely real (even j) / imaginary (odd j) (minimax.cpp:326-330), so every B
// contraction is 2 FMA per complex MAC. The adjoint mirrors both passes
// (gather formulation of D^dagger, no atomics).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace pftg {

template <class R>
struct PftDev {
  using C = typename CT<R>::C;
  int n1, n2, p1, p2, q1, q2, mt1, mt2, r1, r2, M1, M2;
  int lp1, lp2;             // log2 p
  int nb;                   // band columns per cols-pass CTA (fits shared memory)
  const R* Bv1;             // [q1][r1] nonzero part of B1 (pft.cpp:52-61)
  const R* Bv2;             // [q2][r2]
  const C* W1t;             // [r1][M1] = W1[a][j1] for a < 2*mt1 (pft.cpp:63-74)
  const C* W2t;             // [r2][M2]
  const C* tw1;             // exp(-2 pi i k / p1), k < p1/2
  const C* tw2;
  const double* hBv1;       // HOST copies of Bv1/Bv2 (kernel-parameter B tables of the
  const double* hBv2;       // specialized kernels, pft_fast.cuh); never dereferenced on device
};

// Where the rows pass reads its field: base + off(f) + l*ld + c, optionally
// multiplied by probe[l*n2 + c] (exit wave = probe .* object window,
// solver.cpp:240). off(f) = offs ? offs[f] : f*bstride.
template <class R>
struct Src {
  using C = typename CT<R>::C;
  const C* base;
  long long ld;
  long long bstride;
  const long long* offs;
  const C* probe;
  int vec_ok;  // host-verified: base, ld, offsets and probe allow 16-byte column pairs
};

// ---------------------------------------------------------------- smem sizes
__host__ __device__ inline int ldT_of(int n2, int q2) { return n2 + n2 / q2; }

template <class R>
__host__ inline size_t rows_smem_bytes(const PftDev<R>& p) {
  using C = typename CT<R>::C;
  size_t b = 0;
  b += sizeof(C) * (size_t)p.r1 * ldT_of(p.n2, p.q2);  // T
  b += sizeof(C) * (size_t)p.r2 * p.M2;                // W2t
  b += sizeof(C) * (size_t)(p.p2 / 2 + 1);             // tw2
  b += sizeof(R) * (size_t)(p.q1 * p.r1 + p.q2 * p.r2);  // Bv1, Bv2
  return (b + 15) & ~size_t(15);
}

template <class R>
__host__ inline size_t cols_smem_bytes(const PftDev<R>& p, int nb) {
  using C = typename CT<R>::C;
  size_t b = 0;
  b += sizeof(C) * (size_t)p.r1 * nb * (p.p1 + 1);  // Gs
  b += sizeof(C) * (size_t)p.M1 * (nb + 1);        // band strip
  b += sizeof(C) * (size_t)(p.p1 / 2 + 1);         // tw1
  b += sizeof(double) * 64;                        // reduction scratch
  return (b + 15) & ~size_t(15);
}

template <class R>
__host__ inline size_t cols_smem_bytes(const PftDev<R>& p) {
  return cols_smem_bytes(p, p.nb);
}

// Widest strip (<= 16 band columns) whose working set fits in shared memory.
// 8 band columns per CTA keeps several CTAs resident per SM (the cols pass is
// latency-bound); fewer only when the strip does not fit.
template <class R>
__host__ inline int choose_nb(const PftDev<R>& p) {
  int nb = p.M2 < 8 ? p.M2 : 8;
  while (nb > 1 && cols_smem_bytes(p, nb) > 100 * 1024) nb /= 2;
  return nb;
}

// out[m] = sum_j W[j*M + a0 + m*step] * x[j] for the M/step band indices of one
// FFT output (4 independent accumulation chains at a time). emit(a, value).
template <int RB, class C, class Emit>
__device__ __forceinline__ void band_contract(const C* __restrict__ W, int M, int a0, int step, int r,
                                              const C (&x)[RB], Emit&& emit) {
  for (int a = a0; a < M; a += 4 * step) {
    C acc[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[m] = czero<C>();
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      if (j < r) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (a + m * step < M) cmac(acc[m], W[j * M + a + m * step], x[j]);
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (a + m * step < M) emit(a + m * step, acc[m]);
  }
}

// ------------------------------------------------------------ rows pass core
// Stage B + FFT over k2 + axis-2 band contraction for every j1 of this row
// block, reading T (padded [r1][ldT]) from shared memory and writing
// G[j1][b] (global, M2 contiguous per j1).
template <class R, int S2, int RB>
__device__ __forceinline__ void rows_stage_b_to_g(const PftDev<R>& pl, const typename CT<R>::C* T,
                                                  const R* Bv2, const typename CT<R>::C* W2t,
                                                  const typename CT<R>::C* tw2,
                                                  typename CT<R>::C* Gblk) {
  using C = typename CT<R>::C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P2 = pl.p2 < 32 ? pl.p2 : 32;
  const int gpw = 32 / P2;
  const int lig = lane & (P2 - 1), giw = lane / P2;
  const int ldT = ldT_of(pl.n2, pl.q2), q2 = pl.q2, r2 = pl.r2, M2 = pl.M2;
  for (int base = warp * gpw; base < pl.r1; base += nwarps * gpw) {
    const int j1 = base + giw;
    const bool valid = j1 < pl.r1;
    C x[S2][RB];
#pragma unroll
    for (int s = 0; s < S2; ++s) {
#pragma unroll
      for (int j = 0; j < RB; ++j) x[s][j] = czero<C>();
      if (valid) {
        const int k2 = s * P2 + lig;
        const C* trow = T + (size_t)j1 * ldT + (size_t)k2 * (q2 + 1);
        for (int l2 = 0; l2 < q2; ++l2) {
          const C t = trow[l2];
          const R* bv = Bv2 + l2 * r2;
#pragma unroll
          for (int j = 0; j < RB; ++j)
            if (j < r2) bmac(x[s][j], bv[j], t, (j & 1) != 0);
        }
      }
    }
    fft_dif<S2, RB>(x, pl.p2, P2, lig, tw2, -1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S2; ++s) {
      const int u2 = bitrev(s * P2 + lig, pl.lp2);
      band_contract<RB>(W2t, M2, mod_nonneg(u2 + pl.mt2, pl.p2), pl.p2, r2, x[s],
                        [&](int b, C v) { Gblk[(size_t)j1 * M2 + b] = v; });
    }
  }
}

// Load plan tables for the rows pass into shared memory.
template <class R>
__device__ __forceinline__ void rows_load_tables(const PftDev<R>& pl, R* Bv1s, R* Bv2s,
                                                 typename CT<R>::C* W2s, typename CT<R>::C* tw2s) {
  for (int i = threadIdx.x; i < pl.q1 * pl.r1; i += blockDim.x) Bv1s[i] = pl.Bv1[i];
  for (int i = threadIdx.x; i < pl.q2 * pl.r2; i += blockDim.x) Bv2s[i] = pl.Bv2[i];
  for (int i = threadIdx.x; i < pl.r2 * pl.M2; i += blockDim.x) W2s[i] = pl.W2t[i];
  for (int i = threadIdx.x; i < pl.p2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
}

template <class R>
struct RowsSmem {
  using C = typename CT<R>::C;
  C* T;
  C* W2s;
  C* tw2s;
  R* Bv1s;
  R* Bv2s;
  __device__ RowsSmem(unsigned char* raw, const PftDev<R>& pl) {
    C* c = reinterpret_cast<C*>(raw);
    T = c;
    c += (size_t)pl.r1 * ldT_of(pl.n2, pl.q2);
    W2s = c;
    c += (size_t)pl.r2 * pl.M2;
    tw2s = c;
    c += pl.p2 / 2 + 1;
    Bv1s = reinterpret_cast<R*>(c);
    Bv2s = Bv1s + pl.q1 * pl.r1;
  }
};

// Stage A for one column: acc[j1] += B1[l1][j1] * z[l1][c] over l1 < q1.
template <class R, int RB>
__device__ __forceinline__ void stage_a_column(const PftDev<R>& pl, const R* Bv1s,
                                               const typename CT<R>::C* zc, long long ld,
                                               const typename CT<R>::C* pc,
                                               typename CT<R>::C (&acc)[RB]) {
  using C = typename CT<R>::C;
#pragma unroll
  for (int j = 0; j < RB; ++j) acc[j] = czero<C>();
  const int q1 = pl.q1, r1 = pl.r1;
  int l1 = 0;
  for (; l1 + 8 <= q1; l1 += 8) {
    C v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(zc + (long long)(l1 + u) * ld);
    if (pc) {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = cmul(__ldg(pc + (long long)(l1 + u) * pl.n2), v[u]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const R* bv = Bv1s + (l1 + u) * r1;
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (j < r1) bmac(acc[j], bv[j], v[u], (j & 1) != 0);
    }
  }
  for (; l1 < q1; ++l1) {
    C v = __ldg(zc + (long long)l1 * ld);
    if (pc) v = cmul(__ldg(pc + (long long)l1 * pl.n2), v);
    const R* bv = Bv1s + l1 * r1;
#pragma unroll
    for (int j = 0; j < RB; ++j)
      if (j < r1) bmac(acc[j], bv[j], v, (j & 1) != 0);
  }
}

// Forward rows pass. grid = (p1, batch). G: [batch][p1][r1][M2].
template <class R, int S2, int RB>
__global__ void __launch_bounds__(sizeof(R) == 4 ? 512 : 256) k_fwd_rows(PftDev<R> pl, Src<R> src,
                                                  typename CT<R>::C* __restrict__ G) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RowsSmem<R> sm(smem_raw, pl);
  const int k1 = blockIdx.x, f = blockIdx.y;
  rows_load_tables(pl, sm.Bv1s, sm.Bv2s, sm.W2s, sm.tw2s);
  __syncthreads();
  const long long off = src.offs ? src.offs[f] : (long long)f * src.bstride;
  const C* zb = src.base + off + (long long)k1 * pl.q1 * src.ld;
  const C* pb = src.probe ? src.probe + (long long)k1 * pl.q1 * pl.n2 : nullptr;
  const int ldT = ldT_of(pl.n2, pl.q2);
  for (int c = threadIdx.x; c < pl.n2; c += blockDim.x) {
    C acc[RB];
    stage_a_column<R, RB>(pl, sm.Bv1s, zb + c, src.ld, pb ? pb + c : nullptr, acc);
    const int tc = c + c / pl.q2;
#pragma unroll
    for (int j = 0; j < RB; ++j)
      if (j < pl.r1) sm.T[(size_t)j * ldT + tc] = acc[j];
  }
  __syncthreads();
  C* Gblk = G + ((size_t)f * pl.p1 + k1) * pl.r1 * pl.M2;
  rows_stage_b_to_g<R, S2, RB>(pl, sm.T, sm.Bv2s, sm.W2s, sm.tw2s, Gblk);
}

// ------------------------------------------------------------ cols pass core
template <class R>
struct ColsSmem {
  using C = typename CT<R>::C;
  C* Gs;   // [r1][nb][p1+1]
  C* Ys;   // [M1][nb+1]  band strip
  const C* W1s;  // [r1][M1], read through L1 (shared by all CTAs; no per-CTA copy)
  C* tw1s;
  double* red;
  __device__ ColsSmem(unsigned char* raw, const PftDev<R>& pl, int nb) {
    C* c = reinterpret_cast<C*>(raw);
    Gs = c;
    c += (size_t)pl.r1 * nb * (pl.p1 + 1);
    Ys = c;
    c += (size_t)pl.M1 * (nb + 1);
    W1s = pl.W1t;
    tw1s = c;
    c += pl.p1 / 2 + 1;
    red = reinterpret_cast<double*>(c);
  }
};

template <class R>
__device__ __forceinline__ void cols_load_tables(const PftDev<R>& pl, ColsSmem<R>& sm) {
  for (int i = threadIdx.x; i < pl.p1 / 2; i += blockDim.x) sm.tw1s[i] = pl.tw1[i];
}

// Gs <- G[f][k1][j1][b0 + bb] for bb < nbv (coalesced along bb).
// One thread per (j1, k1) row segment of the strip, k1 fastest across threads:
// each thread reads its nb contiguous values (full 128-byte segments), and the
// shared-memory writes of a warp hit consecutive k1 (conflict-free). nb <= 16.
template <class R>
__device__ __forceinline__ void cols_load_g(const PftDev<R>& pl, ColsSmem<R>& sm,
                                            const typename CT<R>::C* Gf, int b0, int nb, int nbv) {
  using C = typename CT<R>::C;
  const int rows = pl.p1 * pl.r1;
  const int ld = pl.p1 + 1;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const int k1 = t & (pl.p1 - 1), j1 = t >> pl.lp1;
    const C* src = Gf + ((size_t)k1 * pl.r1 + j1) * pl.M2 + b0;
    C* dst = sm.Gs + (size_t)j1 * nb * ld + k1;
    C v[16];
#pragma unroll
    for (int bb = 0; bb < 16; ++bb) v[bb] = (bb < nbv) ? src[bb] : czero<C>();
#pragma unroll
    for (int bb = 0; bb < 16; ++bb)
      if (bb < nb) dst[(size_t)bb * ld] = v[bb];
  }
}

// Forward cols: FFT over k1 of Gs column bb and the axis-1 band contraction
// into Ys[a][bb].
template <class R, int S1, int RB>
__device__ __forceinline__ void cols_forward(const PftDev<R>& pl, ColsSmem<R>& sm, int nb) {
  using C = typename CT<R>::C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P1 = pl.p1 < 32 ? pl.p1 : 32;
  const int gpw = 32 / P1;
  const int lig = lane & (P1 - 1), giw = lane / P1;
  const int M1 = pl.M1, r1 = pl.r1;
  for (int base = warp * gpw; base < nb; base += nwarps * gpw) {
    const int bb = base + giw;
    const bool valid = bb < nb;
    C x[S1][RB];
#pragma unroll
    for (int s = 0; s < S1; ++s) {
      const int k1 = s * P1 + lig;
#pragma unroll
      for (int j = 0; j < RB; ++j)
        x[s][j] = (valid && j < r1) ? sm.Gs[((size_t)j * nb + bb) * (pl.p1 + 1) + k1] : czero<C>();
    }
    fft_dif<S1, RB>(x, pl.p1, P1, lig, sm.tw1s, -1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S1; ++s) {
      const int u1 = bitrev(s * P1 + lig, pl.lp1);
      auto emit = [&](int a, C v) { sm.Ys[(size_t)a * (nb + 1) + bb] = v; };
      if constexpr (sizeof(R) == 4) {
        // complex64: Horner form of the band rows (band_horner, pft_fast.cuh); padded x[j >= r1] are 0
        band_horner<RB>(sm.W1s, M1, mod_nonneg(u1 + pl.mt1, pl.p1), pl.p1, pl.mt1, R(1) / R(pl.p1), x[s], emit);
      } else {
        band_contract<RB>(sm.W1s, M1, mod_nonneg(u1 + pl.mt1, pl.p1), pl.p1, r1, x[s], emit);
      }
    }
  }
}

// Adjoint cols: gather conj(W1)^T over the a's of each u1, backward FFT over
// u1 -> k1, into Gs[j1][bb][k1]  (pft.cpp:184-205, axis-1 half).
template <class R, int S1, int RB>
__device__ __forceinline__ void cols_adjoint(const PftDev<R>& pl, ColsSmem<R>& sm, int nb) {
  using C = typename CT<R>::C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P1 = pl.p1 < 32 ? pl.p1 : 32;
  const int gpw = 32 / P1;
  const int lig = lane & (P1 - 1), giw = lane / P1;
  const int M1 = pl.M1, r1 = pl.r1;
  for (int base = warp * gpw; base < nb; base += nwarps * gpw) {
    const int bb = base + giw;
    const bool valid = bb < nb;
    C x[S1][RB];
#pragma unroll
    for (int s = 0; s < S1; ++s) {
#pragma unroll
      for (int j = 0; j < RB; ++j) x[s][j] = czero<C>();
      if (valid) {
        const int u1 = s * P1 + lig;
        for (int a = mod_nonneg(u1 + pl.mt1, pl.p1); a < M1; a += pl.p1) {
          const C y = sm.Ys[(size_t)a * (nb + 1) + bb];
          if constexpr (sizeof(R) == 4) {
            // complex64: Horner-form D-dagger term (gather_horner); padded j >= r1 are never stored
            gather_horner<RB>(x[s], sm.W1s[a], static_cast<R>(a - pl.mt1) * (R(1) / R(pl.p1)), y);
          } else {
#pragma unroll
            for (int j = 0; j < RB; ++j)
              if (j < r1) cmacc(x[s][j], __ldg(sm.W1s + j * M1 + a), y);
          }
        }
      }
    }
    fft_dif<S1, RB>(x, pl.p1, P1, lig, sm.tw1s, +1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S1; ++s) {
      const int k1 = bitrev(s * P1 + lig, pl.lp1);
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (j < r1) sm.Gs[((size_t)j * nb + bb) * (pl.p1 + 1) + k1] = x[s][j];
    }
  }
}

// Single-column strips (nb == 1: one ePIE position spread over >= 64 CTAs).
// The column's r1 transforms are spread over the CTA's lane groups (one j1
// per group, in place in Gs) instead of one lane group carrying all r1, and
// the band rows / D-dagger gathers run one thread per row / per u1.
template <class R, int S1, int RB>
__device__ __forceinline__ void cols_forward_j1(const PftDev<R>& pl, ColsSmem<R>& sm) {
  using C = typename CT<R>::C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P1 = pl.p1 < 32 ? pl.p1 : 32;
  const int gpw = 32 / P1;
  const int lig = lane & (P1 - 1), grp = warp * gpw + lane / P1, ngrp = nwarps * gpw;
  const int ld = pl.p1 + 1, M1 = pl.M1, r1 = pl.r1;
  // warp-uniform loop: the lane-group FFT shuffles over the full warp
  for (int base = warp * gpw; base < r1; base += ngrp) {
    const int j = base + (grp - warp * gpw);
    const bool valid = j < r1;
    C x[S1][1];
#pragma unroll
    for (int s = 0; s < S1; ++s) x[s][0] = valid ? sm.Gs[(size_t)j * ld + s * P1 + lig] : czero<C>();
    fft_dif<S1, 1>(x, pl.p1, P1, lig, sm.tw1s, -1);
    if (valid) {
#pragma unroll
      for (int s = 0; s < S1; ++s) sm.Gs[(size_t)j * ld + bitrev(s * P1 + lig, pl.lp1)] = x[s][0];  // X[j][u1]
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < M1; a += blockDim.x) {
    const int u1 = mod_nonneg(a - pl.mt1, pl.p1);
    C acc = czero<C>();
    if constexpr (sizeof(R) == 4) {
      const R base = static_cast<R>(a - pl.mt1) * (R(1) / R(pl.p1));
      acc = sm.Gs[(size_t)(r1 - 1) * ld + u1];
      for (int j = r1 - 2; j >= 0; --j) acc = cfmar(acc, base, sm.Gs[(size_t)j * ld + u1]);
      acc = cmul(sm.W1s[a], acc);
    } else {
      for (int j = 0; j < r1; ++j) cmac(acc, __ldg(sm.W1s + j * M1 + a), sm.Gs[(size_t)j * ld + u1]);
    }
    sm.Ys[(size_t)a * 2] = acc;  // Ys stride nb + 1 = 2
  }
}

template <class R, int S1, int RB>
__device__ __forceinline__ void cols_adjoint_j1(const PftDev<R>& pl, ColsSmem<R>& sm) {
  using C = typename CT<R>::C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P1 = pl.p1 < 32 ? pl.p1 : 32;
  const int gpw = 32 / P1;
  const int lig = lane & (P1 - 1), grp = warp * gpw + lane / P1, ngrp = nwarps * gpw;
  const int ld = pl.p1 + 1, M1 = pl.M1, r1 = pl.r1;
  for (int u1 = threadIdx.x; u1 < pl.p1; u1 += blockDim.x) {
    C x[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) x[j] = czero<C>();
    for (int a = mod_nonneg(u1 + pl.mt1, pl.p1); a < M1; a += pl.p1) {
      const C y = sm.Ys[(size_t)a * 2];
      if constexpr (sizeof(R) == 4) {
        gather_horner<RB>(x, sm.W1s[a], static_cast<R>(a - pl.mt1) * (R(1) / R(pl.p1)), y);
      } else {
#pragma unroll
        for (int j = 0; j < RB; ++j)
          if (j < r1) cmacc(x[j], __ldg(sm.W1s + j * M1 + a), y);
      }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j)
      if (j < r1) sm.Gs[(size_t)j * ld + u1] = x[j];
  }
  __syncthreads();
  for (int base = warp * gpw; base < r1; base += ngrp) {  // warp-uniform (full-warp shuffles)
    const int j = base + (grp - warp * gpw);
    const bool valid = j < r1;
    C x[S1][1];
#pragma unroll
    for (int s = 0; s < S1; ++s) x[s][0] = valid ? sm.Gs[(size_t)j * ld + s * P1 + lig] : czero<C>();
    fft_dif<S1, 1>(x, pl.p1, P1, lig, sm.tw1s, +1);
    if (valid) {
#pragma unroll
      for (int s = 0; s < S1; ++s) sm.Gs[(size_t)j * ld + bitrev(s * P1 + lig, pl.lp1)] = x[s][0];  // Gs[j][k1]
    }
  }
}

template <class R>
__device__ __forceinline__ void cols_store_g(const PftDev<R>& pl, ColsSmem<R>& sm,
                                             typename CT<R>::C* Gf, int b0, int nb, int nbv) {
  using C = typename CT<R>::C;
  const int rows = pl.p1 * pl.r1;
  const int ld = pl.p1 + 1;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const int k1 = t & (pl.p1 - 1), j1 = t >> pl.lp1;
    C* dst = Gf + ((size_t)k1 * pl.r1 + j1) * pl.M2 + b0;
    const C* src = sm.Gs + (size_t)j1 * nb * ld + k1;
#pragma unroll
    for (int bb = 0; bb < 16; ++bb)
      if (bb < nbv) dst[bb] = src[(size_t)bb * ld];
  }
}

// Band projection residual in place on the strip (solver.cpp:61-69 with
// phase_unit solver.cpp:21-24): y <- y - d * y/|y|  (|y| == 0 -> phase 1).
// Optionally accumulates sum (|y| - d)^2 into *acc (evaluator).
// Visit every (a, bb) of an M1 x nb strip; one division per thread, not per element.
template <class F>
__device__ __forceinline__ void strip_for(int M1, int nb, F&& f) {
  const int step = blockDim.x / nb;
  if ((int)threadIdx.x >= step * nb) return;
  const int bb = threadIdx.x % nb;
  for (int a = threadIdx.x / nb; a < M1; a += step) f(a, bb);
}

template <class R>
__device__ __forceinline__ void project_strip(const PftDev<R>& pl, ColsSmem<R>& sm, int nb, int nbv,
                                              const R* dc, int b0, bool residual, double* acc) {
  double local = 0.0;
  strip_for(pl.M1, nb, [&](int a, int bb) {
    if (bb >= nbv) return;
    auto& y = sm.Ys[(size_t)a * (nb + 1) + bb];
    const R d = dc[(size_t)a * pl.M2 + b0 + bb];
    const R mag = hypot(y.x, y.y);
    if (acc) {
      const double e = (double)mag - (double)d;
      local += e * e;
    }
    if (residual) {
      if (mag > R(0)) {
        const R ux = y.x / mag, uy = y.y / mag;  // phase_unit = v / |v|
        y.x -= d * ux;
        y.y -= d * uy;
      } else {
        y.x -= d;
      }
    }
  });
  if (acc) *acc += local;
}

// Block-wide sum of a double into out[slot] (deterministic order).
__device__ __forceinline__ void block_sum_store(double v, double* scratch, double* out) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += scratch[w];
    *out = s;
  }
}

// MODE 0: forward cols -> band.
// MODE 1: forward cols -> band residual vs dcrop -> adjoint cols -> Gout.
// MODE 2: forward cols -> sum (|band| - dcrop)^2 per CTA into partial.
// grid = (ceil(M2/nb), batch).
// NT = 320: single-column strips (one ePIE position) run one warp per j1 for
// r1 <= 10, so each lane-group FFT phase is one round instead of two.
// Body of one (strip bx, field f) work item of a grid with gx strips per field
// (also the cols phase of the persistent band sweep, band_sweep.cuh).
template <class R, int S1, int RB, int MODE>
__device__ __forceinline__ void k_fwd_cols_body(const PftDev<R>& pl, const typename CT<R>::C* __restrict__ G,
                                                typename CT<R>::C* __restrict__ band,
                                                const R* __restrict__ dcrop, long long dstride,
                                                typename CT<R>::C* __restrict__ Gout,
                                                double* __restrict__ partial, int bx, int f, int gx,
                                                unsigned char* smem_raw) {
  using C = typename CT<R>::C;
  const int nb = pl.nb;
  ColsSmem<R> sm(smem_raw, pl, nb);
  const int b0 = bx * nb;
  const int nbv = min(nb, pl.M2 - b0);
  cols_load_tables(pl, sm);
  const C* Gf = G + (size_t)f * pl.p1 * pl.r1 * pl.M2;
  cols_load_g(pl, sm, Gf, b0, nb, nbv);
  __syncthreads();
  if (nb == 1) cols_forward_j1<R, S1, RB>(pl, sm);
  else cols_forward<R, S1, RB>(pl, sm, nb);
  __syncthreads();
  if (band) {
    C* bf = band + (size_t)f * pl.M1 * pl.M2;
    strip_for(pl.M1, nb, [&](int a, int bb) {
      if (bb < nbv) bf[(size_t)a * pl.M2 + b0 + bb] = sm.Ys[(size_t)a * (nb + 1) + bb];
    });
  }
  if (MODE == 0) return;
  const R* dc = dcrop + (size_t)f * dstride;
  if (MODE == 2) {
    double acc = 0.0;
    project_strip(pl, sm, nb, nbv, dc, b0, false, &acc);
    block_sum_store(acc, sm.red, partial + (size_t)f * gx + bx);
    return;
  }
  project_strip(pl, sm, nb, nbv, dc, b0, true, nullptr);
  __syncthreads();
  if (nb == 1) cols_adjoint_j1<R, S1, RB>(pl, sm);
  else cols_adjoint<R, S1, RB>(pl, sm, nb);
  __syncthreads();
  cols_store_g(pl, sm, Gout + (size_t)f * pl.p1 * pl.r1 * pl.M2, b0, nb, nbv);
  __syncthreads();  // shared memory free for the caller's next work item
}

template <class R, int S1, int RB, int MODE, int NT = 256>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 2) k_fwd_cols(PftDev<R> pl, const typename CT<R>::C* __restrict__ G,
                                                  typename CT<R>::C* __restrict__ band,
                                                  const R* __restrict__ dcrop, long long dstride,
                                                  typename CT<R>::C* __restrict__ Gout,
                                                  double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  k_fwd_cols_body<R, S1, RB, MODE>(pl, G, band, dcrop, dstride, Gout, partial, blockIdx.x, blockIdx.y, gridDim.x,
                                   smem_raw);
}

// Adjoint cols: band -> Gt. grid = (ceil(M2/nb), batch).
template <class R, int S1, int RB>
__global__ void __launch_bounds__(256, 3) k_adj_cols(PftDev<R> pl, const typename CT<R>::C* __restrict__ band,
                                                  typename CT<R>::C* __restrict__ Gt) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = pl.nb;
  ColsSmem<R> sm(smem_raw, pl, nb);
  const int f = blockIdx.y, b0 = blockIdx.x * nb;
  const int nbv = min(nb, pl.M2 - b0);
  cols_load_tables(pl, sm);
  griddep_launch_dependents();
  griddep_wait();  // PDL (API path): the band is the previous kernel's output
  const C* bf = band + (size_t)f * pl.M1 * pl.M2;
  strip_for(pl.M1, nb, [&](int a, int bb) {
    sm.Ys[(size_t)a * (nb + 1) + bb] = bb < nbv ? bf[(size_t)a * pl.M2 + b0 + bb] : czero<C>();
  });
  __syncthreads();
  if (nb == 1) cols_adjoint_j1<R, S1, RB>(pl, sm);
  else cols_adjoint<R, S1, RB>(pl, sm, nb);
  __syncthreads();
  cols_store_g(pl, sm, Gt + (size_t)f * pl.p1 * pl.r1 * pl.M2, b0, nb, nbv);
}

// ------------------------------------------------------- adjoint rows pass
// Per (field, k1): D^dagger along axis 2 (gather over the b's of each u2),
// backward FFT over u2 -> k2, B2^dagger expansion into T, then A^dagger
// (z[l1][c] = sum_j1 conj(B1[l1][j1]) T[j1][c]) with an epilogue:
//   EPI 0: out[f] <- z                                  (pft_adjoint_2d)
//   EPI 1: object window -= beta * conj(probe) * z      (solver.cpp:244-245)
//          and, if G2 != nullptr, the forward rows pass of the new exit wave
//          probe .* object (solver.cpp:247) fused in the same CTA -> G2.
//   EPI 2: probe -= gamma * conj(object window) * z     (solver.cpp:249-250)
struct EpiArgs {
  void* out;               // EPI 0: [batch][n1][n2]
  void* obj;               // EPI 1/2: object window base (frame)
  long long obj_ld;
  long long obj_off;       // element offset of the window's (0,0)
  void* probe;             // [n1][n2]
  double step;             // beta_pft or gamma_pft
  void* G2;                // EPI 1: fused forward output of the new exit wave P z' (may be null);
                           // EPI 2: fused forward output of the NEXT position's exit wave
                           //        P' z[obj_off2] (cross-position fusion; may be null)
  long long obj_off2;      // EPI 2 with G2: element offset of the next position's window
  int vec_ok;              // host-verified 16-byte alignment of out / obj window / probe rows
  int dbg;                 // profiling build only (PFTG_DEBUG_ADJ): skip P1 (1) / fused stage B (2) / epilogue (4)
};

template <class R, int S2, int RB, int EPI>
__global__ void __launch_bounds__(sizeof(R) == 4 ? 512 : 256) k_adj_rows(PftDev<R> pl, const typename CT<R>::C* __restrict__ Gt,
                                                  EpiArgs ep) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RowsSmem<R> sm(smem_raw, pl);
  const int k1 = blockIdx.x, f = blockIdx.y;
  rows_load_tables(pl, sm.Bv1s, sm.Bv2s, sm.W2s, sm.tw2s);
  // this row block's r1 x M2 slice of the adjoint intermediate; each element is
  // read by exactly one lane (coalesced across the lanes' consecutive b)
  const C* Gblk = Gt + ((size_t)f * pl.p1 + k1) * pl.r1 * pl.M2;
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int P2 = pl.p2 < 32 ? pl.p2 : 32;
  const int gpw = 32 / P2;
  const int lig = lane & (P2 - 1), giw = lane / P2;
  const int ldT = ldT_of(pl.n2, pl.q2), q2 = pl.q2, r2 = pl.r2, M2 = pl.M2;
  for (int base = warp * gpw; base < pl.r1; base += nwarps * gpw) {
    const int j1 = base + giw;
    const bool valid = j1 < pl.r1;
    C x[S2][RB];
#pragma unroll
    for (int s = 0; s < S2; ++s) {
#pragma unroll
      for (int j = 0; j < RB; ++j) x[s][j] = czero<C>();
      if (valid) {
        const int u2 = s * P2 + lig;
        for (int b = mod_nonneg(u2 + pl.mt2, pl.p2); b < M2; b += pl.p2) {
          const C g = Gblk[(size_t)j1 * M2 + b];
#pragma unroll
          for (int j = 0; j < RB; ++j)
            if (j < r2) cmacc(x[s][j], sm.W2s[j * M2 + b], g);
        }
      }
    }
    fft_dif<S2, RB>(x, pl.p2, P2, lig, sm.tw2s, +1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S2; ++s) {
      const int k2 = bitrev(s * P2 + lig, pl.lp2);
      C* trow = sm.T + (size_t)j1 * ldT + (size_t)k2 * (q2 + 1);
      for (int l2 = 0; l2 < q2; ++l2) {
        const R* bv = sm.Bv2s + l2 * r2;
        C t = czero<C>();
#pragma unroll
        for (int j = 0; j < RB; ++j)
          if (j < r2) bmacc(t, bv[j], x[s][j], (j & 1) != 0);
        trow[l2] = t;
      }
    }
  }
  __syncthreads();

  // A^dagger + epilogue, one column per thread.
  const int q1 = pl.q1, r1 = pl.r1, n2 = pl.n2;
  const bool fuse_fwd = (EPI >= 1) && ep.G2 != nullptr;
  for (int c = threadIdx.x; c < n2; c += blockDim.x) {
    const int tc = c + c / q2;
    C tv[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) tv[j] = j < r1 ? sm.T[(size_t)j * ldT + tc] : czero<C>();
    C acc2[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc2[j] = czero<C>();
    for (int l1 = 0; l1 < q1; ++l1) {
      const R* bv = sm.Bv1s + l1 * r1;
      C z = czero<C>();
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (j < r1) bmacc(z, bv[j], tv[j], (j & 1) != 0);
      const long long row = (long long)k1 * q1 + l1;
      if (EPI == 0) {
        C* out = reinterpret_cast<C*>(ep.out) + (size_t)f * pl.n1 * n2;
        out[row * n2 + c] = z;
      } else if (EPI == 1) {
        C* obj = reinterpret_cast<C*>(ep.obj) + ep.obj_off;
        const C* pr = reinterpret_cast<const C*>(ep.probe);
        const C pv = pr[row * n2 + c];
        C o = obj[row * ep.obj_ld + c];
        const C g = cmulc(pv, z);  // conj(P) * resid
        o.x -= (R)ep.step * g.x;
        o.y -= (R)ep.step * g.y;
        obj[row * ep.obj_ld + c] = o;
        if (fuse_fwd) {
          const C e = cmul(pv, o);  // new exit wave
#pragma unroll
          for (int j = 0; j < RB; ++j)
            if (j < r1) bmac(acc2[j], bv[j], e, (j & 1) != 0);
        }
      } else {
        const C* obj = reinterpret_cast<const C*>(ep.obj) + ep.obj_off;
        C* pr = reinterpret_cast<C*>(ep.probe);
        const C o = obj[row * ep.obj_ld + c];
        C pv = pr[row * n2 + c];
        const C g = cmulc(o, z);  // conj(z_j) * resid2
        pv.x -= (R)ep.step * g.x;
        pv.y -= (R)ep.step * g.y;
        pr[row * n2 + c] = pv;
        if (fuse_fwd) {  // next position's exit wave from this thread's own new probe element
          const C on = reinterpret_cast<const C*>(ep.obj)[ep.obj_off2 + row * ep.obj_ld + c];
          const C e = cmul(pv, on);
#pragma unroll
          for (int j = 0; j < RB; ++j)
            if (j < r1) bmac(acc2[j], bv[j], e, (j & 1) != 0);
        }
      }
    }
    if (fuse_fwd) {
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (j < r1) sm.T[(size_t)j * ldT + tc] = acc2[j];
    }
  }
  if (fuse_fwd) {
    __syncthreads();
    C* G2blk = reinterpret_cast<C*>(ep.G2) + ((size_t)f * pl.p1 + k1) * pl.r1 * pl.M2;
    rows_stage_b_to_g<R, S2, RB>(pl, sm.T, sm.Bv2s, sm.W2s, sm.tw2s, G2blk);
  }
}

}  // namespace pftg
