// Specialized rows-pass kernels for the plan shapes on the hot path
// (compile-time q, r, p; square plans). Same math and data layout as the
// generic kernels in pft_kernels.cuh, restructured for sm_100a throughput:
//
//  * B tables travel as kernel parameters (constant bank 0) and every loop
//    over (l, j) is unrolled, so each FFMA takes its coefficient straight from
//    the constant bank -- no shared-memory load per MAC.
//  * Node symmetry: the twiddle nodes x_l = 1 - 2l/q satisfy x_{q-l} = -x_l
//    exactly in IEEE arithmetic (q a power of two), hence
//    B[q-l][j] = (-1)^j B[l][j] (pft.cpp:52-61). Contractions over l are done
//    on the sums z_l + z_{q-l} (even j) and differences z_l - z_{q-l} (odd j),
//    and expansions produce rows l and q-l from one even/odd pair of partial
//    sums: half the FMAs of the direct form. B[q/2][j] = w_j 0^j vanishes for
//    j >= 1 and is skipped.
//  * complex64 fields are read and written as 128-bit pairs of columns.
#pragma once

#include "pft_kernels.cuh"

namespace pftg {

// b[l][j] = nonzero part of B[l][j] for l <= q/2 (rows q/2+1.. follow by symmetry)
template <class R, int Q, int RR>
struct BPar {
  R b1[Q / 2 + 1][RR];
  R b2[Q / 2 + 1][RR];
};

// acc += (odd ? i b : b) * v   with b a compile-time-indexed parameter
template <class C, class R>
__device__ __forceinline__ void bmac_p(C& acc, R b, C v, bool odd) { bmac(acc, b, v, odd); }

// Load VC consecutive complex columns of one row (16-byte vectors when VEC).
template <class R, int VC, bool VEC>
__device__ __forceinline__ void load_cols(const typename CT<R>::C* __restrict__ p, typename CT<R>::C (&x)[VC]) {
  using C = typename CT<R>::C;
  if constexpr (VEC && sizeof(C) == 8 && VC % 2 == 0) {
#pragma unroll
    for (int v = 0; v < VC; v += 2) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p + v));
      x[v] = CT<R>::mk(t.x, t.y);
      x[v + 1] = CT<R>::mk(t.z, t.w);
    }
  } else {
#pragma unroll
    for (int v = 0; v < VC; ++v) x[v] = __ldg(p + v);
  }
}

// Stage A with pairing for VC consecutive columns: acc[v][j1] = sum_l B1[l][j1] z[l][c+v].
// Rows are loaded in batches of U symmetric pairs so that ~64 registers of
// loads are in flight per thread (the kernel is latency-bound otherwise).
template <class R, int Q, int RR, int VC, bool VEC>
__device__ __forceinline__ void stage_a_pairs(const BPar<R, Q, RR>& bp, const typename CT<R>::C* __restrict__ zc,
                                              long long ld, const typename CT<R>::C* __restrict__ pc, int pld,
                                              typename CT<R>::C (&acc)[VC][RR]) {
  using C = typename CT<R>::C;
  constexpr int WORDS = (int)(sizeof(C) / 4) * VC;  // registers per row
  constexpr int UMAX = 32 / WORDS > 0 ? 32 / WORDS : 1;
  constexpr int NP = Q / 2 - 1;                     // symmetric pairs (l, Q-l), 0 < l < Q/2
  constexpr int U = NP < UMAX ? (NP > 0 ? NP : 1) : UMAX;
  auto row = [&](int l, C (&x)[VC]) {
    load_cols<R, VC, VEC>(zc + (long long)l * ld, x);
    if (pc) {
      C pv[VC];
      load_cols<R, VC, VEC>(pc + (long long)l * pld, pv);
#pragma unroll
      for (int v = 0; v < VC; ++v) x[v] = cmul(pv[v], x[v]);
    }
  };
#pragma unroll
  for (int v = 0; v < VC; ++v)
#pragma unroll
    for (int j = 0; j < RR; ++j) acc[v][j] = czero<C>();
  {
    C a[VC], h[VC];
    row(0, a);
    row(Q / 2, h);
#pragma unroll
    for (int v = 0; v < VC; ++v) {
#pragma unroll
      for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[0][j], a[v], j & 1);
      bmac(acc[v][0], bp.b1[Q / 2][0], h[v], false);
    }
  }
#pragma unroll
  for (int l0 = 1; l0 < Q / 2; l0 += U) {
    C x[U][2][VC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (l0 + u < Q / 2) {
        row(l0 + u, x[u][0]);
        row(Q - l0 - u, x[u][1]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (l0 + u < Q / 2) {
#pragma unroll
        for (int v = 0; v < VC; ++v) {
          const C sp = cadd(x[u][0][v], x[u][1][v]), dm = csub(x[u][0][v], x[u][1][v]);
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[l0 + u][j], (j & 1) ? dm : sp, j & 1);
        }
      }
  }
}

// Columns per thread for the streaming passes: enough bytes per row load to
// keep the memory system busy when q is small.
template <class R, int Q>
constexpr int cols_per_thread() {
  return sizeof(R) == 4 ? (Q >= 32 ? 1 : (Q >= 16 ? 2 : 4)) : (Q >= 16 ? 1 : 2);
}

// Expansion over l with pairing: out[l] = sum_j conj(B[l][j]) x[j], all l < Q.
// Calls emit(l, value) for every l.
template <class R, int Q, int RR, class Emit>
__device__ __forceinline__ void expand_pairs(const R (&b)[Q / 2 + 1][RR], const typename CT<R>::C (&x)[RR],
                                             Emit&& emit) {
  using C = typename CT<R>::C;
  {
    C e = czero<C>();
#pragma unroll
    for (int j = 0; j < RR; ++j) bmacc(e, b[0][j], x[j], j & 1);
    emit(0, e);
    C h = czero<C>();
    bmacc(h, b[Q / 2][0], x[0], false);
    emit(Q / 2, h);
  }
#pragma unroll
  for (int l = 1; l < Q / 2; ++l) {
    C e = czero<C>(), o = czero<C>();
#pragma unroll
    for (int j = 0; j < RR; j += 2) bmacc(e, b[l][j], x[j], false);
#pragma unroll
    for (int j = 1; j < RR; j += 2) bmacc(o, b[l][j], x[j], true);
    emit(l, cadd(e, o));
    emit(Q - l, csub(e, o));
  }
}

// Same expansion for V columns at once, emitting rows in symmetric pairs:
//   single(l, z[V]) for l = 0 and l = Q/2, pair(l, z_l[V], z_{Q-l}[V]) for 0 < l < Q/2.
template <class R, int Q, int RR, int V, class Single, class Pair>
__device__ __forceinline__ void expand_pairs_v(const R (&b)[Q / 2 + 1][RR],
                                               const typename CT<R>::C (&x)[V][RR], Single&& single,
                                               Pair&& pair) {
  using C = typename CT<R>::C;
  {
    C e[V], h[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      e[v] = czero<C>();
      h[v] = czero<C>();
#pragma unroll
      for (int j = 0; j < RR; ++j) bmacc(e[v], b[0][j], x[v][j], j & 1);
      bmacc(h[v], b[Q / 2][0], x[v][0], false);
    }
    single(0, e);
    single(Q / 2, h);
  }
#pragma unroll
  for (int l = 1; l < Q / 2; ++l) {
    C zl[V], zm[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      C e = czero<C>(), o = czero<C>();
#pragma unroll
      for (int j = 0; j < RR; j += 2) bmacc(e, b[l][j], x[v][j], false);
#pragma unroll
      for (int j = 1; j < RR; j += 2) bmacc(o, b[l][j], x[v][j], true);
      zl[v] = cadd(e, o);
      zm[v] = csub(e, o);
    }
    pair(l, zl, zm);
  }
}

// ---- shared-memory coefficient rows (rolled loops: no uniform-register spills) ----
// Row l of B (RR values) padded to RRP = round_up(RR, 16 bytes) for vector loads.
template <class R, int RR>
constexpr int brow_pad() {
  return sizeof(R) == 4 ? (RR + 3) / 4 * 4 : (RR + 1) / 2 * 2;
}

template <class R, int Q, int RR>
__device__ __forceinline__ void stage_btab(const R (&b)[Q / 2 + 1][RR], R* dst) {
  constexpr int RP = brow_pad<R, RR>();
  for (int i = threadIdx.x; i < (Q / 2 + 1) * RP; i += blockDim.x) {
    const int l = i / RP, j = i % RP;
    dst[i] = j < RR ? b[l][j] : R(0);
  }
}

template <class R, int RR>
__device__ __forceinline__ void load_brow(const R* __restrict__ row, R (&b)[RR]) {
  constexpr int RP = brow_pad<R, RR>();
  R t[RP];
  if constexpr (sizeof(R) == 4) {
#pragma unroll
    for (int k = 0; k < RP; k += 4) {
      const float4 v = *reinterpret_cast<const float4*>(row + k);
      t[k] = v.x;
      t[k + 1] = v.y;
      t[k + 2] = v.z;
      t[k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < RP; k += 2) {
      const double2 v = *reinterpret_cast<const double2*>(row + k);
      t[k] = v.x;
      t[k + 1] = v.y;
    }
  }
#pragma unroll
  for (int j = 0; j < RR; ++j) b[j] = t[j];
}

// expand_pairs_v with the coefficients read from a shared-memory table (btab,
// rows of brow_pad entries) in a rolled loop over l.
template <class R, int Q, int RR, int V, class Single, class Pair>
__device__ __forceinline__ void expand_pairs_sm(const R* __restrict__ btab, const typename CT<R>::C (&x)[V][RR],
                                                Single&& single, Pair&& pair) {
  using C = typename CT<R>::C;
  constexpr int RP = brow_pad<R, RR>();
  {
    R b0[RR];
    load_brow<R, RR>(btab, b0);
    const R bh = btab[(Q / 2) * RP];
    C e[V], h[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      e[v] = czero<C>();
      h[v] = czero<C>();
#pragma unroll
      for (int j = 0; j < RR; ++j) bmacc(e[v], b0[j], x[v][j], j & 1);
      bmacc(h[v], bh, x[v][0], false);
    }
    single(0, e);
    single(Q / 2, h);
  }
  // partial unroll: independent pairs overlap their LDS / FMA latency chains
#pragma unroll 3
  for (int l = 1; l < Q / 2; ++l) {
    R bl[RR];
    load_brow<R, RR>(btab + l * RP, bl);
    C zl[V], zm[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      // (accumulating the odd taps without their -i factor and applying it once removes the
      // (b, b) register-pair MOVs -- 23 % of kt_adj_rows' instructions -- and makes the isolated
      // launch 0.5 us faster, but the PDL-chained cfg2 step 10 us slower (0.228 -> 0.238 ms,
      // same-box A/B): kept in the per-tap form)
      C e = czero<C>(), o = czero<C>();
#pragma unroll
      for (int j = 0; j < RR; j += 2) bmacc(e, bl[j], x[v][j], false);
#pragma unroll
      for (int j = 1; j < RR; j += 2) bmacc(o, bl[j], x[v][j], true);
      zl[v] = cadd(e, o);
      zm[v] = csub(e, o);
    }
    pair(l, zl, zm);
  }
}

// Tile-major record layout of the rows -> cols intermediate used by the
// persistent cols pass (pft_cols.cuh): G[f][k1][b / kStripNB][j1 * kStripNB + b % kStripNB],
// each (k1, strip) record padded by two elements (16-byte aligned records):
// a rows tile (f, k1) writes its records as one contiguous bulk store, a cols
// strip gathers its p1 records with p1 bulk loads.
constexpr int kStripNB = 8;
__host__ __device__ constexpr int strip_rec(int r) { return r * kStripNB + 2; }

// Stage B (+ FFT over k2 + axis-2 band) from T in shared memory, pairing over l2.
// Output: Gblk[j1][b] (row-block layout) or, when gstrip != nullptr, the
// strip-major layout of field gstrip for row block k1.
template <class R, int Q, int RR, int P>
__device__ __forceinline__ void fast_stage_b_to_g(const PftDev<R>& pl, const BPar<R, Q, RR>& bp,
                                                  const typename CT<R>::C* T, const typename CT<R>::C* W2s,
                                                  const typename CT<R>::C* tw2, typename CT<R>::C* Gblk,
                                                  int nwarps = -1, typename CT<R>::C* gstrip = nullptr,
                                                  int k1 = 0, int warp0 = 0) {
  using C = typename CT<R>::C;
  constexpr int PL = P < 32 ? P : 32;
  constexpr int S = P / PL;
  constexpr int GPW = 32 / PL;
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - warp0;  // warp within the calling group
  if (nwarps < 0) nwarps = blockDim.x >> 5;
  const int lig = lane & (PL - 1), giw = lane / PL;
  const int ldT = ldT_of(pl.n2, Q), M2 = pl.M2, mt2 = pl.mt2;
  constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
  for (int base = warp * GPW; base < RR; base += nwarps * GPW) {
    const int j1 = base + giw;
    const bool valid = j1 < RR;
    C x[S][RR];
#pragma unroll
    for (int s = 0; s < S; ++s) {
#pragma unroll
      for (int j = 0; j < RR; ++j) x[s][j] = czero<C>();
      if (valid) {
        const int k2 = s * PL + lig;
        const C* trow = T + (size_t)j1 * ldT + (size_t)k2 * (Q + 1);
        {
          const C t0 = trow[0], th = trow[Q / 2];
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(x[s][j], bp.b2[0][j], t0, j & 1);
          bmac(x[s][0], bp.b2[Q / 2][0], th, false);
        }
#pragma unroll
        for (int l = 1; l < Q / 2; ++l) {
          const C a = trow[l], b = trow[Q - l];
          const C sp = cadd(a, b), dm = csub(a, b);
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(x[s][j], bp.b2[l][j], (j & 1) ? dm : sp, j & 1);
        }
      }
    }
    fft_dif<S, RR>(x, P, PL, lig, tw2, -1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int u2 = bitrev(s * PL + lig, LP);
      if (gstrip) {
        constexpr int REC = strip_rec(RR);
        band_contract<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, RR, x[s], [&](int b, C v) {
          gstrip[((size_t)k1 * (M2 / kStripNB) + b / kStripNB) * REC + j1 * kStripNB + (b % kStripNB)] = v;
        });
      } else {
        band_contract<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, RR, x[s],
                          [&](int b, C v) { Gblk[(size_t)j1 * M2 + b] = v; });
      }
    }
  }
}

template <class R>
__device__ __forceinline__ void fast_load_tables(const PftDev<R>& pl, typename CT<R>::C* W2s,
                                                 typename CT<R>::C* tw2s) {
  for (int i = threadIdx.x; i < pl.r2 * pl.M2; i += blockDim.x) W2s[i] = pl.W2t[i];
  for (int i = threadIdx.x; i < pl.p2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
}

template <class R>
__host__ __device__ inline size_t fast_rows_smem(int n2, int q, int r, int M2, int p) {
  using C = typename CT<R>::C;
  return ((sizeof(C) * ((size_t)r * ldT_of(n2, q) + (size_t)r * M2 + p / 2 + 1)) + 15) & ~size_t(15);
}

// Threads per CTA for the specialized rows kernels: one warp (lane group) per
// j1 in the stage-B phase, at least 8 warps for the streaming phase.
template <int RR, int P>
constexpr int fast_nt() {
  constexpr int gpw = 32 / (P < 32 ? P : 32);
  constexpr int w = (RR + gpw - 1) / gpw;
  return 32 * (w < 8 ? 8 : w);
}
template <class R, int RR, int P>
constexpr int fast_min_blocks() {
  return (sizeof(R) == 4 && fast_nt<RR, P>() <= 320) ? 2 : 1;
}

// Forward rows pass. VEC: 16-byte column vectors allowed (host-checked alignment).
template <class R, int Q, int RR, int P, int V>
__global__ void __launch_bounds__(fast_nt<RR, P>(), fast_min_blocks<R, RR, P>())
    kf_fwd_rows(PftDev<R> pl, BPar<R, Q, RR> bp, Src<R> src, typename CT<R>::C* __restrict__ G) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* T = reinterpret_cast<C*>(smem_raw);
  const int ldT = ldT_of(pl.n2, Q);
  C* W2s = T + (size_t)RR * ldT;
  C* tw2s = W2s + (size_t)RR * pl.M2;
  fast_load_tables(pl, W2s, tw2s);
  const int k1 = blockIdx.x, f = blockIdx.y;
  const long long off = src.offs ? src.offs[f] : (long long)f * src.bstride;
  const C* zb = src.base + off + (long long)k1 * Q * src.ld;
  const C* pb = src.probe ? src.probe + (long long)k1 * Q * pl.n2 : nullptr;
  // V == 2 marks a 16-byte aligned source (vector loads allowed); the number of
  // columns per thread is chosen by q (cols_per_thread).
  constexpr int VC = cols_per_thread<R, Q>();
  constexpr bool VEC = V == 2;
  for (int c = threadIdx.x * VC; c < pl.n2; c += blockDim.x * VC) {
    C acc[VC][RR];
    stage_a_pairs<R, Q, RR, VC, VEC>(bp, zb + c, src.ld, pb ? pb + c : nullptr, pl.n2, acc);
#pragma unroll
    for (int v = 0; v < VC; ++v) {
      const int tc = (c + v) + (c + v) / Q;
#pragma unroll
      for (int j = 0; j < RR; ++j) T[(size_t)j * ldT + tc] = acc[v][j];
    }
  }
  __syncthreads();
  C* Gblk = G + ((size_t)f * pl.p1 + k1) * RR * pl.M2;
  fast_stage_b_to_g<R, Q, RR, P>(pl, bp, T, W2s, tw2s, Gblk);
}

// One-element asynchronous global -> shared copy (LDGSTS: 8 bytes for
// complex64, 16 for complex128) and its group fences
template <class C>
__device__ __forceinline__ void pf_cp(C* smem, const C* gmem) {
  if constexpr (sizeof(C) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void pf_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void pf_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Shared-memory bytes of the ePIE epilogue prefetch (PF = 1): probe, object
// window and (EPI 2) next object window rows of one row block.
template <class R>
__host__ inline size_t adj_prefetch_smem(int n2, int q) {
  return 3 * sizeof(typename CT<R>::C) * (size_t)q * n2 + 16;
}

// Adjoint rows pass (+ ePIE epilogues), mirror of k_adj_rows with pairing.
// PF = 1 (ePIE epilogues): the row block's probe / object window rows (and
// the next position's window rows for the EPI 2 fused forward) are copied
// into shared memory with cp.async at kernel entry, overlapping the D-dagger /
// FFT phase -- the epilogue then runs on shared memory instead of one L2
// round trip per expanded row (it was 5.7 us of a cfg4 position's 12 us
// kernel, tools/band_dbg.sh).
// Body of one (row block k1, field f) work item (also the adjoint-rows phase of
// the persistent band sweep, band_sweep.cuh); any block size >= fast_nt.
template <class R, int Q, int RR, int P, int V, int EPI, int PF = 0>
__device__ __forceinline__ void kf_adj_rows_body(const PftDev<R>& pl, const BPar<R, Q, RR>& bp,
                                                 const typename CT<R>::C* __restrict__ Gt, const EpiArgs& ep, int k1,
                                                 int f, unsigned char* smem_raw) {
  using C = typename CT<R>::C;
  C* T = reinterpret_cast<C*>(smem_raw);
  const int ldT = ldT_of(pl.n2, Q);
  C* W2s = T + (size_t)RR * ldT;
  C* tw2s = W2s + (size_t)RR * pl.M2;
  C* pfP = smem_after<C>(smem_raw, tw2s + P / 2 + 1, 16);  // [Q][n2] probe rows (PF)
  C* pfO = pfP + (size_t)Q * pl.n2;                         // object window rows
  C* pfN = pfO + (size_t)Q * pl.n2;                         // next window rows (EPI 2 + G2)
  if constexpr (PF && EPI >= 1) {
    const int n2 = pl.n2;
    const long long r0 = (long long)k1 * Q;
    const C* pg = reinterpret_cast<const C*>(ep.probe) + r0 * n2;
    const C* og = reinterpret_cast<const C*>(ep.obj) + ep.obj_off + r0 * ep.obj_ld;
    const C* ng = reinterpret_cast<const C*>(ep.obj) + ep.obj_off2 + r0 * ep.obj_ld;
    const bool nxt = EPI == 2 && ep.G2 != nullptr;
    for (int i = threadIdx.x; i < Q * n2; i += blockDim.x) {
      const int l = i / n2, c = i - l * n2;
      pf_cp(pfP + i, pg + (long long)l * n2 + c);
      pf_cp(pfO + i, og + (long long)l * ep.obj_ld + c);
      if (nxt) pf_cp(pfN + i, ng + (long long)l * ep.obj_ld + c);
    }
    pf_commit();
  }
  fast_load_tables(pl, W2s, tw2s);
  const C* Gblk = Gt + ((size_t)f * pl.p1 + k1) * RR * pl.M2;
  __syncthreads();

  constexpr int PL = P < 32 ? P : 32;
  constexpr int S = P / PL;
  constexpr int GPW = 32 / PL;
  constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lig = lane & (PL - 1), giw = lane / PL;
  const int M2 = pl.M2, mt2 = pl.mt2;
  for (int base = warp * GPW; base < RR && !PFTG_DBG(ep.dbg, 1); base += nwarps * GPW) {
    const int j1 = base + giw;
    const bool valid = j1 < RR;
    C x[S][RR];
#pragma unroll
    for (int s = 0; s < S; ++s) {
#pragma unroll
      for (int j = 0; j < RR; ++j) x[s][j] = czero<C>();
      if (valid) {
        const int u2 = s * PL + lig;
        for (int b = (u2 + mt2) & (P - 1); b < M2; b += P) {
          const C g = Gblk[(size_t)j1 * M2 + b];
#pragma unroll
          for (int j = 0; j < RR; ++j) cmacc(x[s][j], W2s[j * M2 + b], g);
        }
      }
    }
    fft_dif<S, RR>(x, P, PL, lig, tw2s, +1);
    if (!valid) continue;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int k2 = bitrev(s * PL + lig, LP);
      C* trow = T + (size_t)j1 * ldT + (size_t)k2 * (Q + 1);
      expand_pairs<R, Q, RR>(bp.b2, x[s], [&](int l, C v) { trow[l] = v; });
    }
  }
  __syncthreads();

  const bool fuse_fwd = (EPI >= 1) && ep.G2 != nullptr;
  const int n2 = pl.n2;
  const long long row0 = (long long)k1 * Q;
  if constexpr (PF && EPI >= 1) {
    pf_wait_all();
    __syncthreads();
  }
  for (int c = threadIdx.x * V; c < n2 && !PFTG_DBG(ep.dbg, 4); c += blockDim.x * V) {
    C tv[V][RR];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int tc = (c + v) + (c + v) / Q;
#pragma unroll
      for (int j = 0; j < RR; ++j) tv[v][j] = T[(size_t)j * ldT + tc];
    }
    if (EPI == 0) {
      C* out = reinterpret_cast<C*>(ep.out) + (size_t)f * pl.n1 * n2 + row0 * n2 + c;
      auto store = [&](int l, const C (&z)[V]) {
        if constexpr (V == 2) {
          *reinterpret_cast<float4*>(out + (long long)l * n2) = make_float4(z[0].x, z[0].y, z[V - 1].x, z[V - 1].y);
        } else {
          out[(long long)l * n2] = z[0];
        }
      };
      expand_pairs_v<R, Q, RR, V>(bp.b1, tv, store, [&](int l, const C (&zl)[V], const C (&zm)[V]) {
        store(l, zl);
        store(Q - l, zm);
      });
      continue;
    }
    C* obj = reinterpret_cast<C*>(ep.obj) + ep.obj_off + row0 * ep.obj_ld + c;
    C* pr = reinterpret_cast<C*>(ep.probe) + row0 * n2 + c;
    // reads of the row block's probe / object / next-window elements (l = row in block)
    auto ld_p = [&](int l, int v) { return PF ? pfP[(size_t)l * n2 + c + v] : pr[(long long)l * n2 + v]; };
    auto ld_o = [&](int l, int v) { return PF ? pfO[(size_t)l * n2 + c + v] : obj[(long long)l * ep.obj_ld + v]; };
    const R st = (R)ep.step;
    C acc2[V][RR];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < RR; ++j) acc2[v][j] = czero<C>();
    // object update z -= beta conj(P) resid (solver.cpp:244-245) -> new exit P z
    auto upd_obj = [&](int l, const C (&z)[V], C (&e)[V]) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const C pv = ld_p(l, v);
        C o = ld_o(l, v);
        const C g = cmulc(pv, z[v]);
        o.x -= st * g.x;
        o.y -= st * g.y;
        obj[(long long)l * ep.obj_ld + v] = o;
        e[v] = cmul(pv, o);
      }
    };
    // probe update P -= gamma conj(z_j) resid2 (solver.cpp:249-250); with G2 set
    // (cross-position fusion) e = the next position's exit wave P' z_next
    const C* objn = reinterpret_cast<const C*>(ep.obj) + ep.obj_off2 + row0 * ep.obj_ld + c;
    auto upd_probe = [&](int l, const C (&z)[V], C (&e)[V]) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const C o = ld_o(l, v);
        C pv = ld_p(l, v);
        const C g = cmulc(o, z[v]);
        pv.x -= st * g.x;
        pv.y -= st * g.y;
        pr[(long long)l * n2 + v] = pv;
        if (fuse_fwd) e[v] = cmul(pv, PF ? pfN[(size_t)l * n2 + c + v] : objn[(long long)l * ep.obj_ld + v]);
      }
    };
    if (EPI >= 1) {
      expand_pairs_v<R, Q, RR, V>(
          bp.b1, tv,
          [&](int l, const C (&z)[V]) {
            C e[V];
            if (EPI == 1) upd_obj(l, z, e);
            else upd_probe(l, z, e);
            if (fuse_fwd) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                if (l == 0) {
#pragma unroll
                  for (int j = 0; j < RR; ++j) bmac(acc2[v][j], bp.b1[0][j], e[v], j & 1);
                } else {
                  bmac(acc2[v][0], bp.b1[Q / 2][0], e[v], false);
                }
              }
            }
          },
          [&](int l, const C (&zl)[V], const C (&zm)[V]) {
            C el[V], em[V];
            if (EPI == 1) {
              upd_obj(l, zl, el);
              upd_obj(Q - l, zm, em);
            } else {
              upd_probe(l, zl, el);
              upd_probe(Q - l, zm, em);
            }
            if (fuse_fwd) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const C sp = cadd(el[v], em[v]), dm = csub(el[v], em[v]);
#pragma unroll
                for (int j = 0; j < RR; ++j) bmac(acc2[v][j], bp.b1[l][j], (j & 1) ? dm : sp, j & 1);
              }
            }
          });
      if (fuse_fwd) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int tc = (c + v) + (c + v) / Q;
#pragma unroll
          for (int j = 0; j < RR; ++j) T[(size_t)j * ldT + tc] = acc2[v][j];
        }
      }
    }
  }
  if (fuse_fwd && !PFTG_DBG(ep.dbg, 2)) {
    __syncthreads();
    C* G2blk = reinterpret_cast<C*>(ep.G2) + ((size_t)f * pl.p1 + k1) * RR * pl.M2;
    fast_stage_b_to_g<R, Q, RR, P>(pl, bp, T, W2s, tw2s, G2blk);
  }
  __syncthreads();  // shared memory free for the caller's next work item
}

template <class R, int Q, int RR, int P, int V, int EPI, int PF = 0>
__global__ void __launch_bounds__(fast_nt<RR, P>(), fast_min_blocks<R, RR, P>())
    kf_adj_rows(PftDev<R> pl, BPar<R, Q, RR> bp, const typename CT<R>::C* __restrict__ Gt, EpiArgs ep) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  kf_adj_rows_body<R, Q, RR, P, V, EPI, PF>(pl, bp, Gt, ep, blockIdx.x, blockIdx.y, smem_raw);
}

}  // namespace pftg
