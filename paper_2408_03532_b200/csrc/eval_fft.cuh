// Full-FFT residual of the forward-model evaluator for 512 x 512 complex64
// windows (BASELINE configs[4]): Phi_j = (1/n) sum_k (|FFT2(P .* z_j)_k| - d_jk)^2
// (objective_value, /root/reference/proj/core/src/solver.cpp:89-102, in its
// Parseval form; fast_fft2 forward unnormalized, fft.cpp:92-104).
//
// Each 512-point DFT is three radix-8 passes held in registers (Stockham
// order, 512 = 8 x 8 x 8): a thread owns 8 points, runs an 8-point DFT
// (24 complex adds), applies the inter-pass twiddles, and exchanges through
// shared memory; the output comes out in natural order. Compared with the
// lane-group radix-2 kernels (fft_kernels.cuh: 9 stages, 5 of them shuffle
// stages) this is ~5x fewer instructions per point.
//   pass 1: y[t][m]  = DFT8_k x[t + 64k] * W512^(t m)          (t < 64)
//   pass 2: z[m][t1][j2] = DFT8_t2 y[t1 + 8 t2][m] * W64^(t1 j2)
//   pass 3: X[m + 8 j2 + 64 j1] = DFT8_t1 z[m][t1][j2]
// Shared-memory layouts S1[m * 66 + t] and S2[t1 * 72 + j2 * 8 + m] keep
// every 16-lane phase of the exchanges on distinct banks.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace pftg {

constexpr int kE512Ld1 = 66, kE512Ld2 = 72, kE512Buf = 8 * kE512Ld2;

// 8-point forward DFT (sign -1), natural in / natural out.
__device__ __forceinline__ void dft8_fwd(float2 (&a)[8]) {
  constexpr float r = 0.70710678118654752440f;
  const float2 b0 = cadd(a[0], a[4]), b1 = cadd(a[1], a[5]), b2 = cadd(a[2], a[6]), b3 = cadd(a[3], a[7]);
  const float2 d4 = csub(a[0], a[4]), d5 = csub(a[1], a[5]), d6 = csub(a[2], a[6]), d7 = csub(a[3], a[7]);
  // odd half twiddles: W8^1 = r(1 - i), W8^2 = -i, W8^3 = -r(1 + i)
  const float2 b5 = f2mul(make_float2(d5.x + d5.y, d5.y - d5.x), make_float2(r, r));
  const float2 b6 = make_float2(d6.y, -d6.x);
  const float2 b7 = f2mul(make_float2(d7.y - d7.x, -(d7.x + d7.y)), make_float2(r, r));
  const float2 c0 = cadd(b0, b2), c2 = csub(b0, b2), c1 = cadd(b1, b3), e3 = csub(b1, b3);
  const float2 c3 = make_float2(e3.y, -e3.x);
  const float2 c4 = cadd(d4, b6), c6 = csub(d4, b6), c5 = cadd(b5, b7), e7 = csub(b5, b7);
  const float2 c7 = make_float2(e7.y, -e7.x);
  a[0] = cadd(c0, c1);
  a[4] = csub(c0, c1);
  a[2] = cadd(c2, c3);
  a[6] = csub(c2, c3);
  a[1] = cadd(c4, c5);
  a[5] = csub(c4, c5);
  a[3] = cadd(c6, c7);
  a[7] = csub(c6, c7);
}

// W512^e for e in [0, 512) from the half table tw[k] = W512^k, k < 256.
__device__ __forceinline__ float2 w512(const float2* tw, int e) {
  const float2 w = tw[e & 255];
  return (e & 256) ? make_float2(-w.x, -w.y) : w;
}

__device__ __forceinline__ float2 cswapri(float2 v) { return make_float2(v.y, v.x); }

// 8-point DFT of either sign: the +1 transform is swap(DFT_-1(swap(x))), swap(a + ib) = b + ia.
template <int SIGN>
__device__ __forceinline__ void dft8(float2 (&a)[8]) {
  if constexpr (SIGN < 0) {
    dft8_fwd(a);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cswapri(a[k]);
    dft8_fwd(a);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cswapri(a[k]);
  }
}

template <int SIGN>
__device__ __forceinline__ float2 w512s(const float2* tw, int e) {
  float2 w = w512(tw, e);
  if (SIGN > 0) w.y = -w.y;
  return w;
}

// One unnormalized 512-point DFT (sign SIGN) held by a group of 64 threads,
// thread role l in [0, 64): in a[k] = x[l + 64 k], out a[j] = X[l + 64 j]
// (natural order on both sides, so a forward and an inverse transform chain
// without an exchange). S: >= kE512Buf complex of shared memory private to the
// group; sync(): barrier over the group. The caller syncs before reusing S.
template <int SIGN, class Sync>
__device__ __forceinline__ void fft512(float2 (&a)[8], float2* S, const float2* tws, int l, Sync&& sync) {
  const int m = l & 7, hi = l >> 3;
  dft8<SIGN>(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512s<SIGN>(tws, l * k));
#pragma unroll
  for (int k = 0; k < 8; ++k) S[k * kE512Ld1 + l] = a[k];
  sync();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = S[m * kE512Ld1 + hi + 8 * k];
  dft8<SIGN>(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512s<SIGN>(tws, 8 * hi * k));
  sync();
#pragma unroll
  for (int k = 0; k < 8; ++k) S[hi * kE512Ld2 + k * 8 + m] = a[k];
  sync();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = S[k * kE512Ld2 + hi * 8 + m];
  dft8<SIGN>(a);
}

// ---- full-FFT ePIE stage for 512 x 512 complex64 windows (solver.cpp:237-262) ----
// Same operator sequence as the lane-group kernels (fft_kernels.cuh): rows
// forward -> cols forward + modulus projection + inverse -> rows inverse x 1/n
// with the object update (+ the forward row transform of the new exit wave,
// blind mode) -> cols -> rows inverse with the probe update; the spectrum is
// in natural order, so the projection reads the measured magnitudes d as is.
enum { E512_FWD = 0, E512_OBJ = 1, E512_PROBE = 2 };

// grid 128, block 256 (four 64-thread groups, one window row each).
// frame + *off: the window (row stride ld); X: rows in, X2: fused forward out (E512_OBJ).
template <int MODE>
__global__ void __launch_bounds__(256) ke_rows512_epie(const float2* __restrict__ tw, float2* frame, long long ld,
                                                       long long off, float2* probe,
                                                       float2* X, float2* X2, float scale, float step, int fuse,
                                                       long long off_next) {
  // window offsets by value (graph node parameters) and the row loads issued
  // before the twiddle-table barrier: one L2 round trip before the first pass
  __shared__ float2 tws[256];
  __shared__ __align__(16) float2 sbuf[4][kE512Buf];
  const int g = threadIdx.x >> 6, l = threadIdx.x & 63;
  const int r = blockIdx.x * 4 + g;
  float2* S = sbuf[g];
  auto gsync = [&]() { named_sync(1 + g, 64); };
  float2* orow = frame + off + (long long)r * ld;
  float2* prow = probe + (size_t)r * 512;
  float2 a[8];
  // Programmatic dependent launch (per-position graphs): the epilogue's operands
  // (probe / object rows, next window) were last written at least two kernels back,
  // so they are requested before the wait; X / X2 (the previous kernel's output)
  // after it. The dependents are released only after this kernel's own wait.
  float2 pvv[8], ovv[8], nvv[8];
  if (MODE != E512_FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      pvv[k] = prow[l + 64 * k];
      ovv[k] = orow[l + 64 * k];
    }
    if (MODE == E512_PROBE && fuse) {
      const float2* nrow = frame + off_next + (long long)r * ld;
#pragma unroll
      for (int k = 0; k < 8; ++k) nvv[k] = nrow[l + 64 * k];
    }
  }
  griddep_wait();
  griddep_launch_dependents();
  if (MODE == E512_FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(prow[l + 64 * k], orow[l + 64 * k]);
  } else {
    const float2* xin = (MODE == E512_OBJ ? X : X2) + (size_t)r * 512;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = xin[l + 64 * k];
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  if (MODE == E512_FWD) {
    fft512<-1>(a, S, tws, l, gsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * 512 + l + 64 * k] = a[k];
    return;
  }
  fft512<+1>(a, S, tws, l, gsync);
  if (MODE == E512_OBJ) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = l + 64 * k;
      float2 proj = a[k];
      proj.x *= scale;
      proj.y *= scale;
      const float2 pv = pvv[k];
      float2 o = ovv[k];
      const float2 resid = csub(cmul(pv, o), proj);  // probe*z - projected
      const float2 gr = cmulc(pv, resid);
      o.x -= step * gr.x;
      o.y -= step * gr.y;
      orow[c] = o;
      a[k] = cmul(pv, o);  // new exit wave (solver.cpp:256)
    }
    if (fuse) {
      gsync();  // S free
      fft512<-1>(a, S, tws, l, gsync);
#pragma unroll
      for (int k = 0; k < 8; ++k) X2[(size_t)r * 512 + l + 64 * k] = a[k];
    }
    return;
  }
  // E512_PROBE
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = l + 64 * k;
    float2 proj = a[k];
    proj.x *= scale;
    proj.y *= scale;
    float2 pv = pvv[k];
    const float2 o = ovv[k];
    const float2 resid = csub(cmul(pv, o), proj);
    const float2 gr = cmulc(o, resid);
    pv.x -= step * gr.x;
    pv.y -= step * gr.y;
    prow[c] = pv;
    a[k] = pv;
  }
  if (fuse) {
    // the next scan position's forward row transform (E512_FWD of position
    // j+1) from the probe row just updated here: its object rows were final
    // after the object-update kernel, and this group owns probe row r
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(a[k], nvv[k]);
    gsync();  // S free
    fft512<-1>(a, S, tws, l, gsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * 512 + l + 64 * k] = a[k];
  }
}

// Columns: forward DFT, modulus projection X <- d X/|X| (|X| = 0 -> d;
// solver.cpp:35-42) against the natural-order magnitudes, inverse DFT
// (unnormalized; the row pass scales), in place. grid 512 / NCOL, block 64 NCOL.
template <int NCOL>
__global__ void __launch_bounds__(64 * NCOL) ke_cols512_proj(float2* X, const float* __restrict__ d,
                                                             const float2* __restrict__ tw) {
  constexpr int CS = kE512Buf + 2;
  __shared__ float2 tws[256];
  __shared__ __align__(16) float2 sbuf[NCOL * CS];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tws[i] = tw[i];
  const int c = threadIdx.x % NCOL, t = threadIdx.x / NCOL;
  const int col = blockIdx.x * NCOL + c;
  float2 a[8];
  float dv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) dv[k] = d[(size_t)(t + 64 * k) * 512 + col];
  griddep_wait();  // PDL: the measured magnitudes and the twiddles do not depend on the previous kernel, X does
  griddep_launch_dependents();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = X[(size_t)(t + 64 * k) * 512 + col];
  __syncthreads();  // tws ready
  float2* S = sbuf + c * CS;
  auto bsync = []() { __syncthreads(); };
  fft512<-1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float mag = hypotf(a[k].x, a[k].y);
    a[k] = mag > 0.f ? make_float2(dv[k] * (a[k].x / mag), dv[k] * (a[k].y / mag)) : make_float2(dv[k], 0.f);
  }
  __syncthreads();  // S free
  fft512<+1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) X[(size_t)(t + 64 * k) * 512 + col] = a[k];
}

// ---- 256-point variant (BASELINE configs[2] windows) ----
// 256 = 8 x (8 x 4): a group of 32 threads (one warp) holds one transform,
// thread l owns x[l + 32 k]. pass 1: DFT8 over k, twiddle W256^(l m);
// pass 2: thread (m, t1) = (l & 7, l >> 3) runs DFT8 over t2 of y[t1 + 4 t2][m],
// twiddle W32^(t1 j2); pass 3: thread l runs two DFT4s over t1 for
// (m, j2) = (l & 7, (l >> 3) + 4 h), h = 0, 1, and ends holding X[l + 32 k]
// (K = m + 8 j2 + 64 j1 = l + 32 (h + 2 j1)): natural order in and out.
constexpr int kE256Ld1 = 33, kE256Ld2 = 9, kE256Buf = 32 * kE256Ld2;

__device__ __forceinline__ void dft4_fwd(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3), e3 = csub(a1, a3);
  const float2 b3 = make_float2(e3.y, -e3.x);  // * (-i)
  a0 = cadd(b0, b2);
  a2 = csub(b0, b2);
  a1 = cadd(b1, b3);
  a3 = csub(b1, b3);
}

template <int SIGN>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  if constexpr (SIGN < 0) {
    dft4_fwd(a0, a1, a2, a3);
  } else {
    a0 = cswapri(a0); a1 = cswapri(a1); a2 = cswapri(a2); a3 = cswapri(a3);
    dft4_fwd(a0, a1, a2, a3);
    a0 = cswapri(a0); a1 = cswapri(a1); a2 = cswapri(a2); a3 = cswapri(a3);
  }
}

// W256^e for e in [0, 256) from the half table tw[k] = W256^k, k < 128.
template <int SIGN>
__device__ __forceinline__ float2 w256s(const float2* tw, int e) {
  float2 w = tw[e & 127];
  if (e & 128) w = make_float2(-w.x, -w.y);
  if (SIGN > 0) w.y = -w.y;
  return w;
}

template <int SIGN, class Sync>
__device__ __forceinline__ void fft256(float2 (&a)[8], float2* S, const float2* tws, int l, Sync&& sync) {
  const int m = l & 7, hi = l >> 3;  // hi in [0, 4)
  dft8<SIGN>(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w256s<SIGN>(tws, l * k));
#pragma unroll
  for (int k = 0; k < 8; ++k) S[k * kE256Ld1 + l] = a[k];
  sync();
  // pass 2: (m, t1 = hi), t = t1 + 4 t2
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = S[m * kE256Ld1 + hi + 4 * k];
  dft8<SIGN>(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w256s<SIGN>(tws, 8 * hi * k));
  sync();
#pragma unroll
  for (int k = 0; k < 8; ++k) S[(m * 4 + hi) * kE256Ld2 + k] = a[k];  // z[m][t1][j2]
  sync();
  // pass 3: (m, j2 = hi + 4 h), DFT4 over t1 -> X[m + 8 j2 + 64 j1] = X[l + 32 (h + 2 j1)]
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j2 = hi + 4 * h;
    float2 v0 = S[(m * 4 + 0) * kE256Ld2 + j2], v1 = S[(m * 4 + 1) * kE256Ld2 + j2];
    float2 v2 = S[(m * 4 + 2) * kE256Ld2 + j2], v3 = S[(m * 4 + 3) * kE256Ld2 + j2];
    dft4<SIGN>(v0, v1, v2, v3);
    a[h] = v0;
    a[h + 2] = v1;
    a[h + 4] = v2;
    a[h + 6] = v3;
  }
}

// ePIE full-FFT stage rows for 256 x 256 windows: grid 64, block 128 (four
// warps, one window row each; the group barrier is a warp barrier).
template <int MODE>
__global__ void __launch_bounds__(128) ke_rows256_epie(const float2* __restrict__ tw, float2* frame, long long ld,
                                                       long long off, float2* probe,
                                                       float2* X, float2* X2, float scale, float step, int fuse,
                                                       long long off_next) {
  __shared__ float2 tws[128];
  __shared__ __align__(16) float2 sbuf[4][kE256Buf];
  const int g = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + g;  // one row per warp: 4 (grid 64) or 2 (grid 128) rows per CTA
  float2* S = sbuf[g];
  auto wsync = []() { __syncwarp(); };
  float2* orow = frame + off + (long long)r * ld;
  float2* prow = probe + (size_t)r * 256;
  float2 a[8];
  // Programmatic dependent launch (per-position graphs): the epilogue's operands
  // (probe / object rows, next window) were last written at least two kernels back,
  // so they are requested before the wait; X / X2 (the previous kernel's output)
  // after it. The dependents are released only after this kernel's own wait.
  float2 pvv[8], ovv[8], nvv[8];
  if (MODE != E512_FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      pvv[k] = prow[l + 32 * k];
      ovv[k] = orow[l + 32 * k];
    }
    if (MODE == E512_PROBE && fuse) {
      const float2* nrow = frame + off_next + (long long)r * ld;
#pragma unroll
      for (int k = 0; k < 8; ++k) nvv[k] = nrow[l + 32 * k];
    }
  }
  griddep_wait();
  griddep_launch_dependents();
  if (MODE == E512_FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(prow[l + 32 * k], orow[l + 32 * k]);
  } else {
    const float2* xin = (MODE == E512_OBJ ? X : X2) + (size_t)r * 256;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = xin[l + 32 * k];
  }
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  if (MODE == E512_FWD) {
    fft256<-1>(a, S, tws, l, wsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * 256 + l + 32 * k] = a[k];
    return;
  }
  fft256<+1>(a, S, tws, l, wsync);
  if (MODE == E512_OBJ) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = l + 32 * k;
      float2 proj = a[k];
      proj.x *= scale;
      proj.y *= scale;
      const float2 pv = pvv[k];
      float2 o = ovv[k];
      const float2 resid = csub(cmul(pv, o), proj);
      const float2 gr = cmulc(pv, resid);
      o.x -= step * gr.x;
      o.y -= step * gr.y;
      orow[c] = o;
      a[k] = cmul(pv, o);
    }
    if (fuse) {
      __syncwarp();
      fft256<-1>(a, S, tws, l, wsync);
#pragma unroll
      for (int k = 0; k < 8; ++k) X2[(size_t)r * 256 + l + 32 * k] = a[k];
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = l + 32 * k;
    float2 proj = a[k];
    proj.x *= scale;
    proj.y *= scale;
    float2 pv = pvv[k];
    const float2 o = ovv[k];
    const float2 resid = csub(cmul(pv, o), proj);
    const float2 gr = cmulc(o, resid);
    pv.x -= step * gr.x;
    pv.y -= step * gr.y;
    prow[c] = pv;
    a[k] = pv;
  }
  if (fuse) {  // next position's forward row transform (see ke_rows512_epie)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(a[k], nvv[k]);
    __syncwarp();
    fft256<-1>(a, S, tws, l, wsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * 256 + l + 32 * k] = a[k];
  }
}

// Columns for 256 x 256: forward, projection, inverse, in place. grid 256 / NCOL, block 32 NCOL.
template <int NCOL>
__global__ void __launch_bounds__(32 * NCOL) ke_cols256_proj(float2* X, const float* __restrict__ d,
                                                             const float2* __restrict__ tw) {
  constexpr int CS = kE256Buf + 1;
  __shared__ float2 tws[128];
  __shared__ __align__(16) float2 sbuf[NCOL * CS];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tws[i] = tw[i];
  const int c = threadIdx.x % NCOL, t = threadIdx.x / NCOL;
  const int col = blockIdx.x * NCOL + c;
  float2 a[8];
  float dv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) dv[k] = d[(size_t)(t + 32 * k) * 256 + col];
  griddep_wait();  // PDL: see ke_cols512_proj
  griddep_launch_dependents();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = X[(size_t)(t + 32 * k) * 256 + col];
  __syncthreads();
  float2* S = sbuf + c * CS;
  auto bsync = []() { __syncthreads(); };
  fft256<-1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float mag = hypotf(a[k].x, a[k].y);
    a[k] = mag > 0.f ? make_float2(dv[k] * (a[k].x / mag), dv[k] * (a[k].y / mag)) : make_float2(dv[k], 0.f);
  }
  __syncthreads();
  fft256<+1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) X[(size_t)(t + 32 * k) * 256 + col] = a[k];
}

// Rows: x[r][c] = probe[r][c] * frame[offs[f] + r * ld + c]; X[f][r][:] =
// DFT_512 of the row, natural order. grid (512 / (4 * RPG), positions), block
// 256 = four 64-thread groups, each transforming RPG rows.
template <int RPG>
__global__ void __launch_bounds__(256, 2) ke_rows512(const float2* __restrict__ frame, long long ld,
                                                  const long long* __restrict__ offs,
                                                  const float2* __restrict__ probe, const float2* __restrict__ tw,
                                                  float2* __restrict__ X) {
  __shared__ float2 tws[256];
  __shared__ __align__(16) float2 sbuf[4][kE512Buf];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  const int g = threadIdx.x >> 6, l = threadIdx.x & 63;
  const int f = blockIdx.y;
  const int m = l & 7, hi = l >> 3;
  float2* S = sbuf[g];
  const float2* fr = frame + offs[f];
  float2* Xf = X + (size_t)f * 512 * 512;
  // the next row's window and probe values are loaded while this row is transformed
  float2 nz[8], np[8];
  auto load_row = [&](int rr) {
    const int r = (blockIdx.x * RPG + rr) * 4 + g;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      np[k] = probe[(size_t)r * 512 + l + 64 * k];
      nz[k] = fr[(long long)r * ld + l + 64 * k];
    }
  };
  load_row(0);
  for (int rr = 0; rr < RPG; ++rr) {
    const int r = (blockIdx.x * RPG + rr) * 4 + g;
    float2 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(np[k], nz[k]);
    if (rr + 1 < RPG) load_row(rr + 1);
    dft8_fwd(a);
#pragma unroll
    for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512(tws, l * k));  // pass 1: W512^(t m), t = l
#pragma unroll
    for (int k = 0; k < 8; ++k) S[k * kE512Ld1 + l] = a[k];
    named_sync(1 + g, 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = S[m * kE512Ld1 + hi + 8 * k];
    dft8_fwd(a);
#pragma unroll
    for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512(tws, 8 * hi * k));  // pass 2: W64^(t1 j2)
    named_sync(1 + g, 64);  // S1 fully read
#pragma unroll
    for (int k = 0; k < 8; ++k) S[hi * kE512Ld2 + k * 8 + m] = a[k];
    named_sync(1 + g, 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = S[k * kE512Ld2 + hi * 8 + m];
    dft8_fwd(a);
    float2* xr = Xf + (size_t)r * 512;
#pragma unroll
    for (int k = 0; k < 8; ++k) xr[l + 64 * k] = a[k];
    named_sync(1 + g, 64);  // S2 fully read before the next row
  }
}

// Columns + residual: a CTA owns 8 adjacent columns of one position (512
// threads: column c = tid & 7, t = tid >> 3), transforms them and accumulates
// sum (|X| - d)^2 (d natural, float) into partial[f * 64 + blockIdx.x].
static __global__ void __launch_bounds__(512) ke_cols512_eval(const float2* __restrict__ X, const float* __restrict__ d,
                                                      const float2* __restrict__ tw, double* __restrict__ partial) {
  constexpr int CS = kE512Buf + 2;  // per-column buffer stride (== 2 mod 16 banks of 8-byte words)
  __shared__ float2 tws[256];
  __shared__ __align__(16) float2 sbuf[8 * CS];
  __shared__ double red[16];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tws[i] = tw[i];
  const int c = threadIdx.x & 7, t = threadIdx.x >> 3;
  const int m = t & 7, hi = t >> 3;
  const int f = blockIdx.y, c0 = blockIdx.x * 8;
  const float2* Xf = X + (size_t)f * 512 * 512 + c0 + c;
  const float* df = d + (size_t)f * 512 * 512 + c0 + c;
  float2 a[8];
  float dv[8];  // measured magnitudes of this thread's outputs, loaded up front
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = Xf[(size_t)(t + 64 * k) * 512];
    dv[k] = df[(size_t)(t + 64 * k) * 512];
  }
  __syncthreads();  // tws ready
  dft8_fwd(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512(tws, t * k));
  float2* S = sbuf + c * CS;
#pragma unroll
  for (int k = 0; k < 8; ++k) S[k * kE512Ld1 + t] = a[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = S[m * kE512Ld1 + hi + 8 * k];
  dft8_fwd(a);
#pragma unroll
  for (int k = 1; k < 8; ++k) a[k] = cmul(a[k], w512(tws, 8 * hi * k));
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k) S[hi * kE512Ld2 + k * 8 + m] = a[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = S[k * kE512Ld2 + hi * 8 + m];
  dft8_fwd(a);
  // output k1 = m + 8 hi + 64 j1 = t + 64 j1 (natural row index of the spectrum)
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    // |X| as sqrt(x^2 + y^2): the spectra are far from float overflow / underflow, and hypotf's
    // scaling costs ~3 x the instructions (evaluator step 4.56 -> see DESIGN)
    const double e = (double)sqrtf(fmaf(a[k].x, a[k].x, a[k].y * a[k].y)) - (double)dv[k];
    acc += e * e;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 16; ++w) s += red[w];
    partial[(size_t)f * 64 + blockIdx.x] = s;
  }
}

}  // namespace pftg
