// Tile path of the 2-D PFT for small batches (BASELINE configs[0]: one 512^2
// complex128 field, p = 16, q = 32): the persistent rows kernels schedule one
// CTA per (field, k1) row block, i.e. 16 CTAs on 148 SMs for a single cfg1
// field, and are latency-bound there. Here every stage is spread over
// >= p1 * p2 CTAs (256 for cfg1) instead:
//
//  forward  (pft.cpp:119-172)
//   kq_fwd_ab   CTA per (k1, k2) tile of q1 x q2 input elements: stage A
//               T[j1][l2] = sum_l1 B1[l1][j1] z[k1 q1 + l1][k2 q2 + l2] and stage B
//               C[k1][k2][j1][j2] = sum_l2 T[j1][l2] B2[l2][j2]   (the field is
//               read exactly once, one coalesced tile per CTA)
//   kq_fft2     CTA per (j1, j2) slice: 2-D radix-2 DFT over (k1, k2) in shared
//               memory (SliceBatchFft2::forward, fft.cpp:259-291)
//   kq_band     CTA per (u1, u2): E[j1][b] = sum_j2 C^[u1][u2][j1][j2] W2[b][j2]
//               for the band columns b with (b - mt2) mod p2 = u2, then
//               out[a][b] = sum_j1 W1[a][j1] E[j1][b] for the rows a of u1 --
//               exactly the reference's inner / outer sums (E is its `inner`)
//  adjoint  (pft.cpp:174-226)
//   kq_adj_band CTA per (u1, u2): C[u1][u2][j1][j2] = sum over the (a, b) of
//               (u1, u2), a-major, of (conj(W1[a][j1]) y[a][b]) conj(W2[b][j2])
//               -- the reference's scatter-add order, as a gather (no atomics)
//   kq_fft2     backward (unnormalized)
//   kq_adj_ab   CTA per (k1, k2): T[j1][l2] = sum_j2 C[j1][j2] conj(B2[l2][j2]),
//               z[l1][l2] = sum_j1 conj(B1[l1][j1]) T[j1][l2], one coalesced tile
//
// The intermediate C (p1 p2 r1 r2 complex per field: 590 KB for cfg1) stays in
// L2. The six kernels launch in plain stream order (programmatic dependent
// launch measured slower here); in a CUDA graph a forward + adjoint pair of a
// cfg1 field takes ~37 us against ~51 us on the persistent rows kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "internal.hpp"
#include "tma.cuh"

namespace pftg {

namespace {

template <class R>
using Cx = typename CT<R>::C;

template <class... KA, class... A>
void launch_tile(void (*kernel)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // Programmatic dependent launch, also inside graph capture. Every tile kernel releases
  // its dependents right after its own griddepcontrol.wait, so only the next kernel's launch
  // and table prologue overlap the running one (releasing at entry let three or four
  // short kernels pile up on the SMs: 52.6 vs 47.1 us per forward + adjoint).
  (void)capturing;
  at[0].val.programmaticStreamSerializationAllowed = knobs().no_pdl ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PFTG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

// Cooperative gather of n elements into shared memory, U loads in flight per
// thread before their stores (a plain strided loop would serialize one global
// round trip per element: the cold tile load dominated kq_fwd_ab, ncu r8 t8).
template <int U, class C, class F>
__device__ __forceinline__ void gather_smem(C* dst, int n, F&& src) {
  for (int base = threadIdx.x; base < n; base += U * blockDim.x) {
    C v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x;
      if (i < n) v[u] = src(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// a in [0, M) with (a - mt) mod p == u: a0 = (u + mt) mod p, then every p-th
__device__ __forceinline__ int band_first(int u, int mt, int p) { return (u + mt) % p; }

// QC / RC: compile-time q and r of a specialized square plan (0 = runtime)
template <class R, int QC = 0, int RC = 0>
__global__ void __launch_bounds__(256) kq_fwd_ab(PftDev<R> pd, const Cx<R>* __restrict__ z, long long bstride,
                                                 Cx<R>* __restrict__ Cg) {
  using C = Cx<R>;
  extern __shared__ __align__(16) unsigned char sm[];
  const int k2 = blockIdx.x, k1 = blockIdx.y, f = blockIdx.z;
  const int q1 = QC ? QC : pd.q1, q2 = QC ? QC : pd.q2, r1 = RC ? RC : pd.r1, r2 = RC ? RC : pd.r2, n2 = pd.n2;
  C* tile = reinterpret_cast<C*>(sm);
  C* T = tile + q1 * q2;
  R* b1 = reinterpret_cast<R*>(T + r1 * q2);
  R* b2 = b1 + q1 * r1;
  for (int i = threadIdx.x; i < q1 * r1; i += blockDim.x) b1[i] = pd.Bv1[i];
  for (int i = threadIdx.x; i < q2 * r2; i += blockDim.x) b2[i] = pd.Bv2[i];
  griddep_wait();  // z may be the previous kernel's output
  griddep_launch_dependents();  // after the wait: one kernel of look-ahead, never two
  const C* src = z + f * bstride + (long long)k1 * q1 * n2 + (long long)k2 * q2;
  gather_smem<8>(tile, q1 * q2, [&](int i) {
    const int l1 = i / q2, l2 = i - l1 * q2;
    return src[(long long)l1 * n2 + l2];
  });
  __syncthreads();
  for (int o = threadIdx.x; o < r1 * q2; o += blockDim.x) {
    const int j1 = o / q2, l2 = o - j1 * q2;
    C acc = czero<C>();
#pragma unroll 8
    for (int l1 = 0; l1 < q1; ++l1) bmac(acc, b1[l1 * r1 + j1], tile[l1 * q2 + l2], (j1 & 1) != 0);
    T[o] = acc;
  }
  __syncthreads();
  C* dst = Cg + ((size_t)(f * pd.p1 + k1) * pd.p2 + k2) * (size_t)(r1 * r2);
  for (int o = threadIdx.x; o < r1 * r2; o += blockDim.x) {
    const int j1 = o / r2, j2 = o - j1 * r2;
    C acc = czero<C>();
#pragma unroll 8
    for (int l2 = 0; l2 < q2; ++l2) bmac(acc, b2[l2 * r2 + j2], T[j1 * q2 + l2], (j2 & 1) != 0);
    dst[o] = acc;
  }
}

// 2-D unnormalized DFT over (k1, k2) of slice s = blockIdx.x of field blockIdx.y,
// sign SIGN (-1 forward, +1 backward); iterative radix-2 DIT, rows then columns.
template <class R, int SIGN, int PC = 0, int RC = 0>
__global__ void __launch_bounds__(256) kq_fft2(PftDev<R> pd, Cx<R>* __restrict__ Cg) {
  using C = Cx<R>;
  extern __shared__ __align__(16) unsigned char sm[];
  const int p1 = PC ? PC : pd.p1, p2 = PC ? PC : pd.p2, lp1 = PC ? ilog2c(PC) : pd.lp1, lp2 = PC ? ilog2c(PC) : pd.lp2;
  const int rr = RC ? RC * RC : pd.r1 * pd.r2;
  C* s = reinterpret_cast<C*>(sm);
  C* tw1 = s + p1 * p2;
  C* tw2 = tw1 + p1 / 2;
  for (int i = threadIdx.x; i < p1 / 2; i += blockDim.x) tw1[i] = pd.tw1[i];
  for (int i = threadIdx.x; i < p2 / 2; i += blockDim.x) tw2[i] = pd.tw2[i];
  griddep_wait();
  griddep_launch_dependents();  // after the wait: one kernel of look-ahead, never two
  C* g = Cg + (size_t)blockIdx.y * p1 * p2 * rr + blockIdx.x;
  {
    constexpr int U = 4;
    for (int base = threadIdx.x; base < p1 * p2; base += U * blockDim.x) {
      C v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * blockDim.x;
        if (i < p1 * p2) v[u] = g[(size_t)i * rr];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * blockDim.x;
        if (i < p1 * p2) {
          const int k1 = i >> lp2, k2 = i & (p2 - 1);
          const int b1 = lp1 ? (int)(__brev((unsigned)k1) >> (32 - lp1)) : 0;
          const int b2 = lp2 ? (int)(__brev((unsigned)k2) >> (32 - lp2)) : 0;
          s[(b1 << lp2) | b2] = v[u];
        }
      }
    }
  }
  __syncthreads();
  // along k2 (within rows)
  for (int half = 1; half < p2; half <<= 1) {
    const int tstride = p2 / (2 * half);
    for (int t = threadIdx.x; t < p1 * (p2 / 2); t += blockDim.x) {
      const int row = t / (p2 / 2), tt = t - row * (p2 / 2);
      const int pos = tt & (half - 1);
      const int i0 = row * p2 + ((tt - pos) << 1) + pos, i1 = i0 + half;
      C w = tw2[pos * tstride];
      if (SIGN > 0) w.y = -w.y;
      const C a = s[i0], b = cmul(s[i1], w);
      s[i0] = cadd(a, b);
      s[i1] = csub(a, b);
    }
    __syncthreads();
  }
  // along k1 (across rows)
  for (int half = 1; half < p1; half <<= 1) {
    const int tstride = p1 / (2 * half);
    for (int t = threadIdx.x; t < (p1 / 2) * p2; t += blockDim.x) {
      const int col = t % p2, tt = t / p2;
      const int pos = tt & (half - 1);
      const int r0 = ((tt - pos) << 1) + pos;
      const int i0 = r0 * p2 + col, i1 = i0 + half * p2;
      C w = tw1[pos * tstride];
      if (SIGN > 0) w.y = -w.y;
      const C a = s[i0], b = cmul(s[i1], w);
      s[i0] = cadd(a, b);
      s[i1] = csub(a, b);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < p1 * p2; i += blockDim.x) g[(size_t)i * rr] = s[i];
}

template <class R, int RC = 0>
__global__ void __launch_bounds__(128) kq_band(PftDev<R> pd, const Cx<R>* __restrict__ Cg, Cx<R>* __restrict__ out) {
  using C = Cx<R>;
  extern __shared__ __align__(16) unsigned char sm[];
  const int u2 = blockIdx.x, u1 = blockIdx.y, f = blockIdx.z;
  const int r1 = RC ? RC : pd.r1, r2 = RC ? RC : pd.r2, M1 = pd.M1, M2 = pd.M2, p1 = pd.p1, p2 = pd.p2;
  const int a0 = band_first(u1, pd.mt1, p1), b0 = band_first(u2, pd.mt2, p2);
  const int na = a0 < M1 ? (M1 - 1 - a0) / p1 + 1 : 0;
  const int nb = b0 < M2 ? (M2 - 1 - b0) / p2 + 1 : 0;
  if (na == 0 || nb == 0) return;
  C* S = reinterpret_cast<C*>(sm);  // [r1][r2]
  C* E = S + r1 * r2;               // [r1][nb]
  C* w1 = E + r1 * nb;              // [na][r1]  W1[a][j1] of this CTA's rows
  C* w2 = w1 + na * r1;             // [nb][r2]  W2[b][j2] of its columns
  // plan tables first (independent of the previous kernel), one parallel round trip
  for (int i = threadIdx.x; i < na * r1; i += blockDim.x) {
    const int ai = i / r1, j1 = i - ai * r1;
    w1[i] = pd.W1t[(size_t)j1 * M1 + a0 + ai * p1];
  }
  for (int i = threadIdx.x; i < nb * r2; i += blockDim.x) {
    const int bi = i / r2, j2 = i - bi * r2;
    w2[i] = pd.W2t[(size_t)j2 * M2 + b0 + bi * p2];
  }
  griddep_wait();
  griddep_launch_dependents();  // after the wait: one kernel of look-ahead, never two
  const C* slice = Cg + ((size_t)(f * p1 + u1) * p2 + u2) * (size_t)(r1 * r2);
  gather_smem<4>(S, r1 * r2, [&](int i) { return slice[i]; });
  __syncthreads();
  // inner (pft.cpp:163-166): sum_j2 row[j2] w2[j2], ascending j2
  for (int o = threadIdx.x; o < r1 * nb; o += blockDim.x) {
    const int j1 = o / nb, bi = o - j1 * nb;
    C inner = czero<C>();
#pragma unroll 4
    for (int j2 = 0; j2 < r2; ++j2) inner = cadd(inner, cmul(S[j1 * r2 + j2], w2[bi * r2 + j2]));
    E[o] = inner;
  }
  __syncthreads();
  C* of = out + (size_t)f * M1 * M2;
  for (int o = threadIdx.x; o < na * nb; o += blockDim.x) {
    const int ai = o / nb, bi = o - ai * nb, a = a0 + ai * p1, b = b0 + bi * p2;
    C acc = czero<C>();
#pragma unroll 4
    for (int j1 = 0; j1 < r1; ++j1) acc = cadd(acc, cmul(w1[ai * r1 + j1], E[j1 * nb + bi]));
    of[(size_t)a * M2 + b] = acc;
  }
}

template <class R, int RC = 0>
__global__ void __launch_bounds__(256) kq_adj_band(PftDev<R> pd, const Cx<R>* __restrict__ band,
                                                   Cx<R>* __restrict__ Cg) {
  using C = Cx<R>;
  extern __shared__ __align__(16) unsigned char sm[];
  const int u2 = blockIdx.x, u1 = blockIdx.y, f = blockIdx.z;
  const int r1 = RC ? RC : pd.r1, r2 = RC ? RC : pd.r2, M1 = pd.M1, M2 = pd.M2, p1 = pd.p1, p2 = pd.p2;
  const int a0 = band_first(u1, pd.mt1, p1), b0 = band_first(u2, pd.mt2, p2);
  const int na = a0 < M1 ? (M1 - 1 - a0) / p1 + 1 : 0;
  const int nb = b0 < M2 ? (M2 - 1 - b0) / p2 + 1 : 0;
  C* Y = reinterpret_cast<C*>(sm);  // [na][nb]
  C* w1 = Y + na * nb;              // [na][r1] conj(W1[a][j1])
  C* w2 = w1 + na * r1;             // [nb][r2] conj(W2[b][j2])
  C* F = w2 + nb * r2;              // [na][r1][nb] conj(W1[a][j1]) y[a][b]
  for (int i = threadIdx.x; i < na * r1; i += blockDim.x) {
    const int ai = i / r1, j1 = i - ai * r1;
    C w = pd.W1t[(size_t)j1 * M1 + a0 + ai * p1];
    w.y = -w.y;
    w1[i] = w;
  }
  for (int i = threadIdx.x; i < nb * r2; i += blockDim.x) {
    const int bi = i / r2, j2 = i - bi * r2;
    C w = pd.W2t[(size_t)j2 * M2 + b0 + bi * p2];
    w.y = -w.y;
    w2[i] = w;
  }
  griddep_wait();
  griddep_launch_dependents();  // after the wait: one kernel of look-ahead, never two
  const C* yf = band + (size_t)f * M1 * M2;
  for (int i = threadIdx.x; i < na * nb; i += blockDim.x) {
    const int ai = i / nb, bi = i - ai * nb;
    Y[i] = yf[(size_t)(a0 + ai * p1) * M2 + b0 + bi * p2];
  }
  __syncthreads();
  C* dst = Cg + ((size_t)(f * p1 + u1) * p2 + u2) * (size_t)(r1 * r2);
  // the reference's scatter order (pft.cpp:188-201): a ascending, then b, term
  // (conj(w1[j1]) y) conj(w2[j2]) accumulated into C[j1][j2]
  const int o = threadIdx.x;
  const int j1 = o / r2, j2 = o - j1 * r2;
  // every c1 = conj(w1) y first (one barrier), then the accumulation chains
  for (int i = threadIdx.x; i < na * r1 * nb; i += blockDim.x) {
    const int ai = i / (r1 * nb), rem = i - ai * (r1 * nb), jj = rem / nb, bi = rem - jj * nb;
    F[i] = cmul(w1[ai * r1 + jj], Y[ai * nb + bi]);
  }
  __syncthreads();
  C acc = czero<C>();
  if (o < r1 * r2) {
    for (int ai = 0; ai < na; ++ai) {
      const C* Fa = F + (size_t)(ai * r1 + j1) * nb;
#pragma unroll 4
      for (int bi = 0; bi < nb; ++bi) acc = cadd(acc, cmul(Fa[bi], w2[bi * r2 + j2]));
    }
    dst[o] = acc;
  }
}

template <class R, int QC = 0, int RC = 0>
__global__ void __launch_bounds__(256) kq_adj_ab(PftDev<R> pd, const Cx<R>* __restrict__ Cg, Cx<R>* __restrict__ z,
                                                 long long bstride) {
  using C = Cx<R>;
  extern __shared__ __align__(16) unsigned char sm[];
  const int k2 = blockIdx.x, k1 = blockIdx.y, f = blockIdx.z;
  const int q1 = QC ? QC : pd.q1, q2 = QC ? QC : pd.q2, r1 = RC ? RC : pd.r1, r2 = RC ? RC : pd.r2, n2 = pd.n2;
  C* S = reinterpret_cast<C*>(sm);  // [r1][r2]
  C* T = S + r1 * r2;               // [r1][q2]
  R* b1 = reinterpret_cast<R*>(T + r1 * q2);
  R* b2 = b1 + q1 * r1;
  for (int i = threadIdx.x; i < q1 * r1; i += blockDim.x) b1[i] = pd.Bv1[i];
  for (int i = threadIdx.x; i < q2 * r2; i += blockDim.x) b2[i] = pd.Bv2[i];
  griddep_wait();
  griddep_launch_dependents();  // after the wait: one kernel of look-ahead, never two
  const C* slice = Cg + ((size_t)(f * pd.p1 + k1) * pd.p2 + k2) * (size_t)(r1 * r2);
  gather_smem<4>(S, r1 * r2, [&](int i) { return slice[i]; });
  __syncthreads();
  // M = Cslice * B2^H (pft.cpp:213-220)
  for (int o = threadIdx.x; o < r1 * q2; o += blockDim.x) {
    const int j1 = o / q2, l2 = o - j1 * q2;
    C acc = czero<C>();
#pragma unroll 4
    for (int j2 = 0; j2 < r2; ++j2) bmacc(acc, b2[l2 * r2 + j2], S[j1 * r2 + j2], (j2 & 1) != 0);
    T[o] = acc;
  }
  __syncthreads();
  // Zblk = conj(B1) * T (pft.cpp:221-223)
  C* dst = z + f * bstride + (long long)k1 * q1 * n2 + (long long)k2 * q2;
  for (int i = threadIdx.x; i < q1 * q2; i += blockDim.x) {
    const int l1 = i / q2, l2 = i - l1 * q2;
    C acc = czero<C>();
#pragma unroll 4
    for (int j1 = 0; j1 < r1; ++j1) bmacc(acc, b1[l1 * r1 + j1], T[j1 * q2 + l2], (j1 & 1) != 0);
    dst[(long long)l1 * n2 + l2] = acc;
  }
}

template <class K>
void smem_optin(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) PFTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  // one shared-memory carveout for the whole chain: no L1 / shared
  // reconfiguration of the SMs between consecutive kernels
  PFTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}

template <class R>
size_t ab_smem(const PftDev<R>& pd) {
  return sizeof(Cx<R>) * ((size_t)pd.q1 * pd.q2 + (size_t)pd.r1 * pd.q2) + sizeof(R) * ((size_t)pd.q1 * pd.r1 + (size_t)pd.q2 * pd.r2);
}
template <class R>
size_t adj_ab_smem(const PftDev<R>& pd) {
  return sizeof(Cx<R>) * ((size_t)pd.r1 * pd.r2 + (size_t)pd.r1 * pd.q2) + sizeof(R) * ((size_t)pd.q1 * pd.r1 + (size_t)pd.q2 * pd.r2);
}
template <class R>
size_t fft2_smem(const PftDev<R>& pd) {
  return sizeof(Cx<R>) * ((size_t)pd.p1 * pd.p2 + pd.p1 / 2 + pd.p2 / 2 + 2);
}
// the literal BASELINE configs[0] plan (q = 32, r = 12 on both axes): compile-time loop bounds
template <class R>
bool spec12(const PftDev<R>& pd) {
  return pd.q1 == 32 && pd.q2 == 32 && pd.r1 == 12 && pd.r2 == 12;
}

template <class R>
size_t adj_band_smem(const PftDev<R>& pd) {
  const size_t na = (pd.M1 + pd.p1 - 1) / pd.p1, nb = (pd.M2 + pd.p2 - 1) / pd.p2;
  return sizeof(Cx<R>) * (na * nb + na * pd.r1 + nb * pd.r2 + na * pd.r1 * nb);
}

template <class R>
int band_rows(int M, int p) {
  return (M + p - 1) / p;
}

}  // namespace

template <class R>
bool tile_path_ok(const PftDev<R>& pd, std::size_t batch) {
  if (knobs().no_tile) return false;
  const bool fits = ab_smem(pd) <= 200 * 1024 && adj_ab_smem(pd) <= 200 * 1024 && fft2_smem(pd) <= 200 * 1024 &&
                    adj_band_smem(pd) <= 200 * 1024 && (size_t)pd.r1 * pd.r2 <= 256 && batch <= 65535;
  if (!fits) return false;
  if (knobs().force_tile) return true;
  // the persistent rows kernels run one CTA per (field, k1): use the tile path
  // when that leaves most SMs idle
  return (long long)batch * pd.p1 < 148 / 2;
}

template <class R>
void tile_apply(const PftDev<R>& pd, const void* z, long long bstride, void* band, int batch, cudaStream_t st) {
  const size_t cn = (size_t)pd.p1 * pd.p2 * pd.r1 * pd.r2;
  Scratch Cg(sizeof(Cx<R>) * cn * batch, st);
  const dim3 tiles(pd.p2, pd.p1, batch);
  {
    ProfScope prof(st, K_FWD_ROWS);
    auto k = spec12(pd) ? kq_fwd_ab<R, 32, 12> : kq_fwd_ab<R>;
    smem_optin(k, ab_smem(pd));
    launch_tile(k, tiles, dim3(256), ab_smem(pd), st, pd, static_cast<const Cx<R>*>(z), bstride, Cg.as<Cx<R>>());
  }
  {
    ProfScope prof(st, K_FWD_COLS);
    auto k = (spec12(pd) && pd.p1 == 16 && pd.p2 == 16) ? kq_fft2<R, -1, 16, 12> : kq_fft2<R, -1>;
    smem_optin(k, fft2_smem(pd));
    launch_tile(k, dim3(pd.r1 * pd.r2, batch), dim3(256), fft2_smem(pd), st, pd, Cg.as<Cx<R>>());
  }
  {
    ProfScope prof(st, K_FWD_COLS);
    const size_t na = band_rows<R>(pd.M1, pd.p1), nb = band_rows<R>(pd.M2, pd.p2);
    const size_t sm = sizeof(Cx<R>) * ((size_t)pd.r1 * pd.r2 + pd.r1 * nb + na * pd.r1 + nb * pd.r2);
    auto k = spec12(pd) ? kq_band<R, 12> : kq_band<R>;
    smem_optin(k, sm);
    launch_tile(k, tiles, dim3(128), sm, st, pd, (const Cx<R>*)Cg.as<Cx<R>>(), static_cast<Cx<R>*>(band));
  }
}

template <class R>
void tile_adjoint(const PftDev<R>& pd, const void* band, void* z, long long bstride, int batch, cudaStream_t st) {
  const size_t cn = (size_t)pd.p1 * pd.p2 * pd.r1 * pd.r2;
  Scratch Cg(sizeof(Cx<R>) * cn * batch, st);
  const dim3 tiles(pd.p2, pd.p1, batch);
  {
    ProfScope prof(st, K_ADJ_COLS);
    const size_t na = band_rows<R>(pd.M1, pd.p1), nb = band_rows<R>(pd.M2, pd.p2);
    const size_t sm = sizeof(Cx<R>) * (na * nb + na * pd.r1 + nb * pd.r2 + na * pd.r1 * nb);
    auto k = spec12(pd) ? kq_adj_band<R, 12> : kq_adj_band<R>;
    smem_optin(k, sm);
    launch_tile(k, tiles, dim3(256), sm, st, pd, static_cast<const Cx<R>*>(band), Cg.as<Cx<R>>());
  }
  {
    ProfScope prof(st, K_ADJ_COLS);
    auto k = (spec12(pd) && pd.p1 == 16 && pd.p2 == 16) ? kq_fft2<R, 1, 16, 12> : kq_fft2<R, 1>;
    smem_optin(k, fft2_smem(pd));
    launch_tile(k, dim3(pd.r1 * pd.r2, batch), dim3(256), fft2_smem(pd), st, pd, Cg.as<Cx<R>>());
  }
  {
    ProfScope prof(st, K_ADJ_ROWS);
    auto k = spec12(pd) ? kq_adj_ab<R, 32, 12> : kq_adj_ab<R>;
    smem_optin(k, adj_ab_smem(pd));
    launch_tile(k, tiles, dim3(256), adj_ab_smem(pd), st, pd, (const Cx<R>*)Cg.as<Cx<R>>(), static_cast<Cx<R>*>(z),
                bstride);
  }
}

template bool tile_path_ok<float>(const PftDev<float>&, std::size_t);
template bool tile_path_ok<double>(const PftDev<double>&, std::size_t);
template void tile_apply<float>(const PftDev<float>&, const void*, long long, void*, int, cudaStream_t);
template void tile_apply<double>(const PftDev<double>&, const void*, long long, void*, int, cudaStream_t);
template void tile_adjoint<float>(const PftDev<float>&, const void*, void*, long long, int, cudaStream_t);
template void tile_adjoint<double>(const PftDev<double>&, const void*, void*, long long, int, cudaStream_t);

}  // namespace pftg
