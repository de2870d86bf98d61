// Persistent cols passes for the specialized plan shapes (batched PFT).
//
// The cols pass of the forward PFT (FFT over k1 + axis-1 band contraction,
// the k1 half of pft.cpp:147-170) and of the adjoint (the D-dagger gather over
// a + backward FFT over u1, pft.cpp:184-205) touch only ~16 % of a field's
// bytes but were latency-bound as one-shot CTAs. Here each CTA loops over
// band strips of kStripNB columns and double-buffers its input:
//  * forward: the rows pass writes G strip-major (pft_fast.cuh), so a strip is
//    one contiguous 1-D bulk copy (cp.async.bulk) issued one iteration ahead;
//  * adjoint: the band strip (kStripNB columns of every row) is prefetched into
//    registers one iteration ahead and parked in shared memory.
#pragma once

#include "pft_fast.cuh"
#include "tma.cuh"

namespace pftg {

constexpr int kColsThreads = 256;

// Elements per field of the strip-major G layout.
template <class R>
__host__ inline long long strip_field_elems(const PftDev<R>& pd) {
  return (long long)(pd.M2 / kStripNB) * pd.p1 * strip_rec(pd.r1);
}

template <class R>
__host__ __device__ inline size_t cols_fwd_smem(int p1, int r, int M1) {
  using C = typename CT<R>::C;
  size_t b = sizeof(C) * (2 * (size_t)p1 * strip_rec(r) + (size_t)M1 * (kStripNB + 1) + p1 / 2 + 1);
  return ((b + 15) & ~size_t(15)) + 128 + 2 * sizeof(uint64_t);
}

template <class R, int RR, int P>
__global__ void __launch_bounds__(kColsThreads, 2)
    kc_fwd_cols(PftDev<R> pl, const typename CT<R>::C* __restrict__ G, long long gstride,
                typename CT<R>::C* __restrict__ band, int nstrips_field, int ntotal) {
  using C = typename CT<R>::C;
  constexpr int REC = strip_rec(RR);
  constexpr int PL = P < 32 ? P : 32;
  constexpr int S = P / PL;
  constexpr int GPW = 32 / PL;
  constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  const int sbytes_e = P * REC;  // elements per strip
  C* buf = reinterpret_cast<C*>(smem_raw);  // [2][P * REC]
  C* Ys = buf + 2 * (size_t)sbytes_e;       // [M1][kStripNB + 1]
  C* tw1s = Ys + (size_t)M1 * (kStripNB + 1);
  uint64_t* full = smem_after<uint64_t>(smem_raw, tw1s + P / 2 + 1, 16);
  const uint32_t strip_bytes = (uint32_t)(sbytes_e * sizeof(C));
  for (int i = threadIdx.x; i < P / 2; i += blockDim.x) tw1s[i] = pl.tw1[i];
  // strip sg = (field, st): record k1 of the strip sits at G[f][k1][st] (tile-major
  // layout written by the rows pass); P record copies land as buf[k1][REC]
  auto load_strip = [&](int sg, C* dst, uint64_t* bar) {
    const int f = sg / nstrips_field, st = sg % nstrips_field;
    const C* src = G + (size_t)f * gstride + (size_t)st * REC;
    mbar_arrive_expect_tx(bar, strip_bytes);
    for (int k1 = 0; k1 < P; ++k1)
      bulk_g2s(dst + (size_t)k1 * REC, src + (size_t)k1 * nstrips_field * REC, (uint32_t)(REC * sizeof(C)), bar);
  };
  griddep_launch_dependents();
  griddep_wait();  // PDL: G is the previous kernel's output
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_fence_init();
    for (int s = 0; s < 2; ++s) {
      const int sg = blockIdx.x + s * gridDim.x;
      if (sg < ntotal) {
        load_strip(sg, buf + (size_t)s * sbytes_e, &full[s]);
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lig = lane & (PL - 1), giw = lane / PL;
  const int bb = warp * GPW + giw;  // band column within the strip (kColsThreads/32*GPW >= kStripNB)
  const bool valid = bb < kStripNB;
  uint32_t i = 0;
  for (int sg = blockIdx.x; sg < ntotal; sg += gridDim.x, ++i) {
    const int s = i & 1;
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    const C* sb = buf + (size_t)s * sbytes_e;
    mbar_wait(&full[s], (i >> 1) & 1);
    C x[S][RR];
#pragma unroll
    for (int ss = 0; ss < S; ++ss) {
      const int k1 = ss * PL + lig;
#pragma unroll
      for (int j = 0; j < RR; ++j) x[ss][j] = valid ? sb[(size_t)k1 * REC + j * kStripNB + bb] : czero<C>();
    }
    fft_dif<S, RR>(x, P, PL, lig, tw1s, -1);
    if (valid) {
#pragma unroll
      for (int ss = 0; ss < S; ++ss) {
        const int u1 = bitrev(ss * PL + lig, LP);
        band_contract<RR>(pl.W1t, M1, (u1 + mt1) & (P - 1), P, RR, x[ss],
                          [&](int a, C v) { Ys[(size_t)a * (kStripNB + 1) + bb] = v; });
      }
    }
    __syncthreads();  // strip buffer s consumed, Ys complete
    if (threadIdx.x == 0 && sg + 2 * (int)gridDim.x < ntotal) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      load_strip(sg + 2 * gridDim.x, buf + (size_t)s * sbytes_e, &full[s]);
    }
    // band rows a, columns b0 .. b0+7: 4 threads x 2 columns per row (64-byte segments)
    C* bf = band + (size_t)f * M1 * M2 + b0;
    for (int e = threadIdx.x; e < M1 * (kStripNB / 2); e += blockDim.x) {
      const int a = e / (kStripNB / 2), cc = (e % (kStripNB / 2)) * 2;
      const C v0 = Ys[(size_t)a * (kStripNB + 1) + cc], v1 = Ys[(size_t)a * (kStripNB + 1) + cc + 1];
      if constexpr (sizeof(C) == 8) {
        *reinterpret_cast<float4*>(bf + (size_t)a * M2 + cc) = make_float4(v0.x, v0.y, v1.x, v1.y);
      } else {
        bf[(size_t)a * M2 + cc] = v0;
        bf[(size_t)a * M2 + cc + 1] = v1;
      }
    }
    __syncthreads();  // Ys free for the next strip
  }
}

template <class R>
__host__ __device__ inline size_t cols_adj_smem(int p1, int r, int M1) {
  using C = typename CT<R>::C;
  size_t b = sizeof(C) * ((size_t)M1 * (kStripNB + 1) + (size_t)p1 * (r * kStripNB + 1) + p1 / 2 + 1);
  return ((b + 15) & ~size_t(15)) + 128;
}

// Adjoint cols pass: band strip -> Gt[f][k1][j1][b] (row-block layout read by
// the adjoint rows pass). The next strip's band values are loaded into
// registers while the current strip is transformed.
template <class R, int RR, int P>
__global__ void __launch_bounds__(kColsThreads, 2)
    kc_adj_cols(PftDev<R> pl, const typename CT<R>::C* __restrict__ band, typename CT<R>::C* __restrict__ Gt,
                int nstrips_field, int ntotal) {
  using C = typename CT<R>::C;
  constexpr int PL = P < 32 ? P : 32;
  constexpr int S = P / PL;
  constexpr int GPW = 32 / PL;
  constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
  constexpr int LDY = kStripNB + 1;
  constexpr int GREC = RR * kStripNB + 1;  // padded per-k1 record: conflict-free k1-strided writes
  // per-thread share of a strip: M1 rows x kStripNB columns, 2 columns per item
  constexpr int MAXIT = 8;  // supports M1 * kStripNB / 2 <= kColsThreads * MAXIT
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  C* Ys = reinterpret_cast<C*>(smem_raw);  // [M1][LDY]
  C* Gs = Ys + (size_t)M1 * LDY;           // [P][GREC]
  C* tw1s = Gs + (size_t)P * GREC;
  for (int i = threadIdx.x; i < P / 2; i += blockDim.x) tw1s[i] = pl.tw1[i];
  const int items = M1 * (kStripNB / 2);
  C pre[MAXIT][2];
  auto prefetch = [&](int sg) {
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    const C* bf = band + (size_t)f * M1 * M2 + b0;
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int e = threadIdx.x + it * kColsThreads;
      if (e < items) {
        const int a = e / (kStripNB / 2), cc = (e % (kStripNB / 2)) * 2;
        if constexpr (sizeof(C) == 8) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(bf + (size_t)a * M2 + cc));
          pre[it][0] = CT<R>::mk(v.x, v.y);
          pre[it][1] = CT<R>::mk(v.z, v.w);
        } else {
          pre[it][0] = __ldg(bf + (size_t)a * M2 + cc);
          pre[it][1] = __ldg(bf + (size_t)a * M2 + cc + 1);
        }
      }
    }
  };
  auto park = [&]() {
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int e = threadIdx.x + it * kColsThreads;
      if (e < items) {
        const int a = e / (kStripNB / 2), cc = (e % (kStripNB / 2)) * 2;
        Ys[(size_t)a * LDY + cc] = pre[it][0];
        Ys[(size_t)a * LDY + cc + 1] = pre[it][1];
      }
    }
  };
  griddep_launch_dependents();
  griddep_wait();  // PDL: the band is the previous kernel's output
  if ((int)blockIdx.x < ntotal) {
    prefetch(blockIdx.x);
    park();
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lig = lane & (PL - 1), giw = lane / PL;
  const int bb = warp * GPW + giw;
  const bool valid = bb < kStripNB;
  for (int sg = blockIdx.x; sg < ntotal; sg += gridDim.x) {
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    const bool more = sg + (int)gridDim.x < ntotal;
    if (more) prefetch(sg + gridDim.x);  // in flight during the transform below
    C x[S][RR];
#pragma unroll
    for (int ss = 0; ss < S; ++ss) {
#pragma unroll
      for (int j = 0; j < RR; ++j) x[ss][j] = czero<C>();
      if (valid) {
        const int u1 = ss * PL + lig;
        for (int a = (u1 + mt1) & (P - 1); a < M1; a += P) {
          const C y = Ys[(size_t)a * LDY + bb];
#pragma unroll
          for (int j = 0; j < RR; ++j) cmacc(x[ss][j], __ldg(pl.W1t + j * M1 + a), y);
        }
      }
    }
    fft_dif<S, RR>(x, P, PL, lig, tw1s, +1);
    if (valid) {
#pragma unroll
      for (int ss = 0; ss < S; ++ss) {
        const int k1 = bitrev(ss * PL + lig, LP);
#pragma unroll
        for (int j = 0; j < RR; ++j) Gs[(size_t)k1 * GREC + j * kStripNB + bb] = x[ss][j];
      }
    }
    __syncthreads();  // Ys consumed, Gs complete
    // Gt[f][k1][j1][b0 .. b0+7]: 64-byte segments, 2 columns per item
    C* gf = Gt + (size_t)f * P * RR * M2 + b0;
    for (int e = threadIdx.x; e < P * RR * (kStripNB / 2); e += blockDim.x) {
      const int kj = e / (kStripNB / 2), cc = (e % (kStripNB / 2)) * 2;
      const int k1 = kj / RR, j = kj % RR;
      const C v0 = Gs[(size_t)k1 * GREC + j * kStripNB + cc], v1 = Gs[(size_t)k1 * GREC + j * kStripNB + cc + 1];
      if constexpr (sizeof(C) == 8) {
        *reinterpret_cast<float4*>(gf + (size_t)kj * M2 + cc) = make_float4(v0.x, v0.y, v1.x, v1.y);
      } else {
        gf[(size_t)kj * M2 + cc] = v0;
        gf[(size_t)kj * M2 + cc + 1] = v1;
      }
    }
    if (more) park();
    __syncthreads();  // Ys refilled, Gs drained
  }
}

// ---------------------------------------------------------------------------
// Lane-local variants for p1 = 32 (complex64): one thread runs a whole 32-point
// FFT in registers (the radix-2 DIF of common.cuh with the same twiddle table
// and operation order, so results are bit-identical to the lane-group FFT),
// instead of one lane group per sequence with 5 shuffle stages. The band
// contraction is then done per band row a by one thread: the r1 W1[j][a]
// coefficients stay in its registers for the CTA's lifetime and the kStripNB
// outputs of a row are stored as one 64-byte segment.

// Radix-2 DIF over N values held by one thread: natural in, bit-reversed out.
// Twiddle index 0 (w = 1 exactly) skips the multiply: bit-identical for finite
// values. W: register array or shared-memory pointer of the N/2 twiddles.
template <int N, class C, class W>
__device__ __forceinline__ void fft_dif_local(C (&x)[N], const W& w, int sign) {
#pragma unroll
  for (int h = N / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & h) == 0) {
        const int ti = (i & (h - 1)) * (N / (2 * h));
        const C a = x[i], c = x[i + h];
        x[i] = cadd(a, c);
        if (ti == 0) {
          x[i + h] = csub(a, c);
        } else {
          C tw = w[ti];
          if (sign > 0) tw.y = -tw.y;
          x[i + h] = cmul(csub(a, c), tw);
        }
      }
    }
  }
}

constexpr int kLocalP = 32;

// Forward: warp-specialized. Warps 0..2 (one thread per (j1, bb) sequence)
// run the FFTs of strip i into Xs[i & 1] while warps 3..6 run the band
// contraction of strip i-1; mbarriers hand the spectrum buffers back and
// forth, so neither group idles at a block barrier. A band thread owns the
// rows a and a + 128 (same u1 = (a - mt1) mod 32): every spectrum value it
// reads from shared memory feeds two rows (M1 <= 256), each evaluated by
// Horner's rule (band_horner, pft_fast.cuh).
// FFT warps = one warpgroup (80 of its 128 threads own a sequence), band
// warps = two warpgroups (one band row each); setmaxnreg moves registers from
// the band warps (56) to the FFT warps (128: a whole 32-point transform + 16
// twiddles per thread) at 2 CTAs per SM (80 registers at launch).
constexpr int kFftWarps = 4, kBandWarps = 8;
constexpr int kColsRegLaunch = 80, kColsRegFft = 128, kColsRegBand = 56;
static_assert(32 * kFftWarps * (kColsRegFft - kColsRegLaunch) <= 32 * kBandWarps * (kColsRegLaunch - kColsRegBand),
              "register hand-over must balance");
constexpr int kStripBufs = 2;  // strips in flight (G is L2-resident between the passes)
constexpr int kBandLd = 10;    // staged band rows: 80-byte stride, 16-byte aligned, conflict-light
constexpr int kAdjLdy = 10;    // adjoint cols band strip rows: 80-byte stride (16-byte cp.async targets)

template <class R>
__host__ __device__ inline size_t cols_fwd_local_smem(int r, int M1) {
  using C = typename CT<R>::C;
  const size_t b =
      sizeof(C) * (kStripBufs * (size_t)kLocalP * strip_rec(r) + 2 * (size_t)kLocalP * (r * kStripNB + 1) +
                   (size_t)M1 * kBandLd);
  return ((b + 15) & ~size_t(15)) + 128 + (kStripBufs + 4) * sizeof(uint64_t);
}

template <class R, int RR>
__global__ void __launch_bounds__(32 * (kFftWarps + kBandWarps), 2)
    kc_fwd_cols_local(PftDev<R> pl, const typename CT<R>::C* __restrict__ G, long long gstride,
                      typename CT<R>::C* __restrict__ band, int nstrips_field, int ntotal, int dbg) {
  using C = typename CT<R>::C;
  static_assert(sizeof(R) == 4, "lane-local cols pass: complex64");
  constexpr int P = kLocalP;
  constexpr int REC = strip_rec(RR);
  constexpr int NSEQ = RR * kStripNB;  // (j1, bb) sequences per strip
  static_assert(NSEQ <= 32 * kFftWarps, "one FFT thread per sequence");
  constexpr int LDX = NSEQ + 1;        // Xs[u][j1 * 8 + bb], padded
  constexpr int FT = 32 * kFftWarps, BT = 32 * kBandWarps;
  static_assert(BT % P == 0, "rows a and a + BT share u1");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  const int sbytes_e = P * REC;
  C* buf = reinterpret_cast<C*>(smem_raw);        // [kStripBufs][P * REC]
  C* Xs = buf + kStripBufs * (size_t)sbytes_e;    // [2][P][LDX]
  C* Bs = Xs + 2 * (size_t)P * LDX;               // [M1][kBandLd]: the strip's band rows, staged
  uint64_t* bars = smem_after<uint64_t>(smem_raw, Bs + (size_t)M1 * kBandLd, 16);
  uint64_t* full = bars;                 // TMA -> FFT warps
  uint64_t* xready = bars + kStripBufs;  // FFT -> band warps
  uint64_t* xfree = xready + 2;          // band -> FFT warps
  const uint32_t strip_bytes = (uint32_t)(sbytes_e * sizeof(C));
  // strip sg = (field, st): record k1 of the strip sits at G[f][k1][st] (tile-major
  // layout written by the rows pass); P record copies land as buf[k1][REC]
  auto load_strip = [&](int sg, C* dst, uint64_t* bar) {
    const int f = sg / nstrips_field, st = sg % nstrips_field;
    const C* src = G + (size_t)f * gstride + (size_t)st * REC;
    mbar_arrive_expect_tx(bar, strip_bytes);
    for (int k1 = 0; k1 < P; ++k1)
      bulk_g2s(dst + (size_t)k1 * REC, src + (size_t)k1 * nstrips_field * REC, (uint32_t)(REC * sizeof(C)), bar);
  };
  griddep_launch_dependents();
  griddep_wait();  // PDL: G is the previous kernel's output
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStripBufs; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xready[s], 1);
      mbar_init(&xfree[s], 1);
    }
    mbar_fence_init();
    for (int s = 0; s < kStripBufs; ++s) {
      const int sg = blockIdx.x + s * gridDim.x;
      if (sg < ntotal) {
        load_strip(sg, buf + (size_t)s * sbytes_e, &full[s]);
      }
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < FT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kColsRegFft));
  else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kColsRegBand));
  if (t < FT) {
    // ---------------- FFT warps ----------------
    C w[P / 2];  // twiddles, in registers for the CTA's lifetime
#pragma unroll
    for (int k = 0; k < P / 2; ++k) w[k] = pl.tw1[k];
    uint32_t i = 0;
    for (int sg = blockIdx.x; sg < ntotal; sg += gridDim.x, ++i) {
      const int s = i & 1, sbi = (int)(i % kStripBufs);
      const C* sb = buf + (size_t)sbi * sbytes_e;
      C* X = Xs + (size_t)s * P * LDX;
      if (!PFTG_DBG(dbg, 4) || i < kStripBufs) mbar_wait(&full[sbi], (i / kStripBufs) & 1);
      if (i >= 2) mbar_wait(&xfree[s], ((i >> 1) - 1) & 1);
      if (t < NSEQ && !PFTG_DBG(dbg, 1)) {
        // sequence (j1, bb) = (t / 8, t % 8): FFT over k1, spectrum to X[u][t]
        C x[P];
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) x[k1] = sb[(size_t)k1 * REC + t];
        fft_dif_local<P>(x, w, -1);
#pragma unroll
        for (int pos = 0; pos < P; ++pos) X[(size_t)((__brev((unsigned)pos) >> 27) & (P - 1)) * LDX + t] = x[pos];
      }
      named_sync(1, FT);  // strip buffer sbi consumed, X complete
      if (t == 0) {
        mbar_arrive(&xready[s]);
        if (!PFTG_DBG(dbg, 4) && sg + kStripBufs * (int)gridDim.x < ntotal) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          load_strip(sg + kStripBufs * gridDim.x, buf + (size_t)sbi * sbytes_e, &full[sbi]);
        }
      }
    }
    return;
  }
  // ---------------- band warps ----------------
  // thread (u1, column) = (tb / 8, tb % 8): reads its r1 spectrum values once and
  // evaluates the M1 / p1 band rows a = u1 + mt1 (mod p1) of that column by
  // Horner (one shared-memory read per value instead of one per (row, value))
  static_assert(BT == P * kStripNB, "one band thread per (u1, column)");
  const int tb = t - FT;
  const int ub = tb / kStripNB, bbt = tb % kStripNB;
  uint32_t i = 0;
  for (int sg = blockIdx.x; sg < ntotal; sg += gridDim.x, ++i) {
    const int s = i & 1;
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    mbar_wait(&xready[s], (i >> 1) & 1);
    if (!PFTG_DBG(dbg, 2)) {
      const C* xr = Xs + (size_t)s * P * LDX + (size_t)ub * LDX;
      C xv[RR];
#pragma unroll
      for (int j = 0; j < RR; ++j) xv[j] = xr[j * kStripNB + bbt];
      for (int a = (ub + mt1) & (P - 1); a < M1; a += P) {
        const R base = static_cast<R>(a - mt1) * (R(1) / R(P));
        C acc = xv[RR - 1];
#pragma unroll
        for (int j = RR - 2; j >= 0; --j) acc = cfmar(acc, base, xv[j]);
        Bs[(size_t)a * kBandLd + bbt] = cmul(__ldg(pl.W1t + a), acc);
      }
    }
    named_sync(2, BT);  // X[s] fully read, Bs complete
    if (tb == 0) mbar_arrive(&xfree[s]);
    C* bdst = band + (size_t)f * M1 * M2 + b0;
    for (int k = tb; k < M1 * (kStripNB / 2); k += BT) {
      const int row = k / (kStripNB / 2), q = k % (kStripNB / 2);
      *reinterpret_cast<float4*>(bdst + (size_t)row * M2 + 2 * q) =
          *reinterpret_cast<const float4*>(Bs + (size_t)row * kBandLd + 2 * q);
    }
    named_sync(2, BT);  // Bs drained
  }
}

template <class R>
__host__ __device__ inline size_t cols_adj_local_smem(int r, int M1) {
  using C = typename CT<R>::C;
  const size_t b = sizeof(C) * (2 * (size_t)M1 * kAdjLdy + (size_t)r * kStripNB * (kLocalP + 1));
  return ((b + 15) & ~size_t(15)) + 128;
}

// 16-byte global -> shared asynchronous copy (LDGSTS), bypassing registers.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Adjoint: gather over the band rows of each u1 (thread (u1, bb)), then one
// thread per (j1, bb) runs the inverse 32-point FFT and stores its 32 values
// straight to Gt (row-block layout; per k1 a warp writes 4 j1 x 64-byte
// segments). The band strip of the next iteration streams into the other Ys
// buffer with cp.async while this one is transformed (no register staging).
template <class R, int RR>
__global__ void __launch_bounds__(kColsThreads, 2)
    kc_adj_cols_local(PftDev<R> pl, const typename CT<R>::C* __restrict__ band, typename CT<R>::C* __restrict__ Gt,
                      int nstrips_field, int ntotal, int dbg) {
  using C = typename CT<R>::C;
  constexpr int P = kLocalP;
  constexpr int LDY = kAdjLdy;             // Ys[a][bb], 80-byte rows (16-byte aligned pairs)
  constexpr int NSEQ = RR * kStripNB;
  constexpr int LDS_ = P + 1;              // Xs[(j1, bb)][u]
  static_assert(sizeof(R) == 4, "lane-local cols pass: complex64");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  C* Ys0 = reinterpret_cast<C*>(smem_raw);  // [2][M1][LDY]
  C* Xs = Ys0 + 2 * (size_t)M1 * LDY;       // [NSEQ][LDS_]
  C w[P / 2];
#pragma unroll
  for (int k = 0; k < P / 2; ++k) w[k] = pl.tw1[k];
  const int items = M1 * (kStripNB / 2);  // 16-byte pairs per strip
  auto fetch = [&](int sg, C* Ys) {
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    const C* bf = band + (size_t)f * M1 * M2 + b0;
    for (int e = threadIdx.x; e < items; e += blockDim.x) {
      const int aa = e / (kStripNB / 2), cc = (e % (kStripNB / 2)) * 2;
      cp_async16(Ys + (size_t)aa * LDY + cc, bf + (size_t)aa * M2 + cc);
    }
    cp_async_commit();
  };
  griddep_launch_dependents();
  griddep_wait();  // PDL: the band is the previous kernel's output
  if ((int)blockIdx.x < ntotal) fetch(blockIdx.x, Ys0);
  const int t = threadIdx.x;
  const int gu = t >> 3, gbb = t & 7;  // gather thread (u1, bb), t < P * kStripNB
  uint32_t i = 0;
  for (int sg = blockIdx.x; sg < ntotal; sg += gridDim.x, ++i) {
    const int f = sg / nstrips_field, b0 = (sg % nstrips_field) * kStripNB;
    C* Ys = Ys0 + (size_t)(i & 1) * M1 * LDY;
    cp_async_wait_all();
    __syncthreads();  // Ys[i & 1] landed for every thread; Xs free (previous FFT done)
    if (sg + (int)gridDim.x < ntotal && !PFTG_DBG(dbg, 8)) fetch(sg + gridDim.x, Ys0 + (size_t)((i + 1) & 1) * M1 * LDY);
    if (t < P * kStripNB && !PFTG_DBG(dbg, 1)) {  // dbg 1: profiling switch, no gather
      C x[RR];
#pragma unroll
      for (int j = 0; j < RR; ++j) x[j] = czero<C>();
      for (int aa = (gu + mt1) & (P - 1); aa < M1; aa += P)
        gather_horner<RR>(x, __ldg(pl.W1t + aa), static_cast<R>(aa - mt1) * (R(1) / R(P)), Ys[(size_t)aa * LDY + gbb]);
#pragma unroll
      for (int j = 0; j < RR; ++j) Xs[(size_t)(j * kStripNB + gbb) * LDS_ + gu] = x[j];
    }
    __syncthreads();  // Xs complete
    if (t < NSEQ && !PFTG_DBG(dbg, 2)) {  // dbg 2: no FFT
      C x[P];
#pragma unroll
      for (int uu = 0; uu < P; ++uu) x[uu] = Xs[(size_t)t * LDS_ + uu];
      fft_dif_local<P>(x, w, +1);
      // sequence t = (j1, bb): Gt[f][k1][j1][b0 + bb]
      C* gcol = Gt + (size_t)f * P * RR * M2 + (size_t)(t / kStripNB) * M2 + b0 + (t % kStripNB);
      if (!PFTG_DBG(dbg, 4)) {  // dbg 4: no stores
#pragma unroll
        for (int pos = 0; pos < P; ++pos) {
          constexpr int LP = 5;
          const int k1 = (__brev((unsigned)pos) >> (32 - LP)) & (P - 1);
          gcol[(size_t)k1 * RR * M2] = x[pos];
        }
      }
    }
  }
  cp_async_wait_all();
}

}  // namespace pftg
