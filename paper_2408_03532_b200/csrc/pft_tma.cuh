// Persistent, TMA-fed forward rows pass for the batched PFT (the hot kernel of
// BASELINE configs[1]): one CTA per SM loops over (field, k1) row blocks.
//
//  * A producer warp streams the row block through a ring of NS shared-memory
//    slots with 1-D bulk copies (cp.async.bulk -> UBLKCP). Each slot holds the
//    symmetric row pair (l, q-l) (or (0, q/2)), so the node-symmetry pairing of
//    stage A (pft_fast.cuh) needs no register staging. The producer runs ahead
//    across block boundaries: while the consumers do stage B / FFT / band of
//    block t, the first NS pairs of block t+1 are already in flight, so HBM
//    never idles behind the compute phase.
//  * 512 consumer threads own 512*VC columns each for the whole block
//    (accumulators stay in registers across all q rows), then write T to
//    shared memory and run the same stage-B/FFT/band code as kf_fwd_rows.
// Math identical to kf_fwd_rows / pft.cpp:119-172 (see pft_kernels.cuh).
#pragma once

#include "pft_fast.cuh"
#include "tma.cuh"

namespace pftg {

constexpr int kTmaConsumers = 512;

template <class R>
__host__ __device__ inline size_t tma_rows_smem(int n2, int q, int r, int M2, int p, int ns) {
  using C = typename CT<R>::C;
  size_t b = sizeof(C) * ((size_t)ns * 2 * n2 + (size_t)r * ldT_of(n2, q) + (size_t)r * M2 + p / 2 + 1);
  b = (b + 15) & ~size_t(15);
  return b + 2 * ns * sizeof(uint64_t);
}

template <class R, int Q, int RR, int P, int VC>
__global__ void __launch_bounds__(kTmaConsumers + 32, 1)
    kt_fwd_rows(PftDev<R> pl, BPar<R, Q, RR> bp, const typename CT<R>::C* __restrict__ z, long long ld,
                long long bstride, int ntiles, int NS, typename CT<R>::C* __restrict__ G, int dbg,
                long long gstride) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n2 = pl.n2;
  C* ring = reinterpret_cast<C*>(smem_raw);
  C* T = ring + (size_t)NS * 2 * n2;
  const int ldT = ldT_of(n2, Q);
  C* W2s = T + (size_t)RR * ldT;
  C* tw2s = W2s + (size_t)RR * pl.M2;
  uint64_t* bars = smem_after<uint64_t>(smem_raw, tw2s + P / 2 + 1, 16);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;

  fast_load_tables(pl, W2s, tw2s);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const uint32_t row_bytes = (uint32_t)(n2 * sizeof(C));
  if (threadIdx.x >= kTmaConsumers) {
    // ---------------- producer warp ----------------
    if (threadIdx.x != kTmaConsumers) return;
    uint32_t seq = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int f = t / pl.p1, k1 = t % pl.p1;
      const C* base = z + (long long)f * bstride + (long long)k1 * Q * ld;
      // (an L2 bulk prefetch of the next row block was measured slower: 93 -> 101 us)
      for (int pi = 0; pi < Q / 2; ++pi, ++seq) {
        const int s = seq % NS;
        if (seq >= NS) mbar_wait(&empty[s], ((seq / NS) - 1) & 1);
        const int la = pi == 0 ? 0 : pi, lb = pi == 0 ? Q / 2 : Q - pi;
        mbar_arrive_expect_tx(&full[s], 2 * row_bytes);
        C* slot = ring + (size_t)s * 2 * n2;
        bulk_g2s(slot, base + (long long)la * ld, row_bytes, &full[s]);
        bulk_g2s(slot + n2, base + (long long)lb * ld, row_bytes, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int lane = threadIdx.x & 31;
  const int c0 = threadIdx.x * VC;
  uint32_t seq = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int f = t / pl.p1, k1 = t % pl.p1;
    C acc[VC][RR];
#pragma unroll
    for (int v = 0; v < VC; ++v)
#pragma unroll
      for (int j = 0; j < RR; ++j) acc[v][j] = czero<C>();
#pragma unroll
    for (int pi = 0; pi < Q / 2; ++pi, ++seq) {
      const int s = seq % NS;
      mbar_wait(&full[s], (seq / NS) & 1);
      const C* slot = ring + (size_t)s * 2 * n2;
      C a[VC], b[VC];
      if constexpr (VC == 2 && sizeof(C) == 8) {
        const float4 ta = *reinterpret_cast<const float4*>(slot + c0);
        const float4 tb = *reinterpret_cast<const float4*>(slot + n2 + c0);
        a[0] = CT<R>::mk(ta.x, ta.y);
        a[VC - 1] = CT<R>::mk(ta.z, ta.w);
        b[0] = CT<R>::mk(tb.x, tb.y);
        b[VC - 1] = CT<R>::mk(tb.z, tb.w);
      } else {
#pragma unroll
        for (int v = 0; v < VC; ++v) {
          a[v] = slot[c0 + v];
          b[v] = slot[n2 + c0 + v];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if PFTG_DBG(dbg, 2) {  // profiling experiment: pure streaming (keep the loads alive)
        if (a[0].x == 1234.5f && b[0].y == -1234.5f) acc[0][0].x += 1;
        continue;
      }
#pragma unroll
      for (int v = 0; v < VC; ++v) {
        if (pi == 0) {
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[0][j], a[v], j & 1);
          bmac(acc[v][0], bp.b1[Q / 2][0], b[v], false);
        } else {
          const C sp = cadd(a[v], b[v]), dm = csub(a[v], b[v]);
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[pi][j], (j & 1) ? dm : sp, j & 1);
        }
      }
    }
    // all consumers are past stage B of the previous block: T may be overwritten
    named_sync(1, kTmaConsumers);
#pragma unroll
    for (int v = 0; v < VC; ++v) {
      const int c = c0 + v;
      const int tc = c + c / Q;
#pragma unroll
      for (int j = 0; j < RR; ++j) T[(size_t)j * ldT + tc] = acc[v][j];
    }
    named_sync(1, kTmaConsumers);
    if PFTG_DBG(dbg, 1) continue;  // profiling experiment: streaming + stage A only
    C* Gblk = G + ((size_t)f * pl.p1 + k1) * RR * pl.M2;
    // gstride > 0: strip-major layout for the persistent cols pass (field stride gstride)
    fast_stage_b_to_g<R, Q, RR, P>(pl, bp, T, W2s, tw2s, Gblk, kTmaConsumers / 32,
                                   gstride > 0 ? G + (size_t)f * gstride : nullptr, k1);
  }
}

// ---------------------------------------------------------------------------
// Warp-specialized variant of kt_fwd_rows: group A (16 warps) streams row
// pairs from the TMA ring and accumulates stage A in registers; group B (one
// warp per j1) runs stage B / FFT / band of the previous block concurrently, so
// HBM streaming never stops for the compute phase. T is single-buffered: group
// B holds it only for stage B (its results stay in registers for the FFT and
// band), while group A needs it again only after a whole block of streaming,
// so the shared memory a second T would take goes to the TMA ring instead
// (8 x 16 KB in flight per SM instead of 3). W2 is read through L1.
template <int RR, int P>
constexpr int fwd_b_warps() {
  constexpr int gpw = 32 / (P < 32 ? P : 32);
  return (RR + gpw - 1) / gpw;
}

template <class R>
__host__ __device__ inline size_t tma2_rows_smem(int n2, int q, int r, int M2, int p, int ns, bool probe = false) {
  using C = typename CT<R>::C;
  const size_t slot = 2 * (size_t)(n2 + 2) + (probe ? 2 * (size_t)n2 : 0);  // row pair (+2: alignment shift) + probe rows
  // complex64: W2 row 0 (Horner band) + a strip-major staging block of the tile's G;
  // complex128: the full W2 table (direct band contraction)
  const size_t wtab = sizeof(R) == 4 ? (size_t)M2 + (size_t)(M2 / kStripNB) * strip_rec(r) : (size_t)r * M2;
  size_t b = sizeof(C) * ((size_t)ns * slot + (size_t)r * ldT_of(n2, q) + wtab + p / 2 + 1);
  b = (b + 15) & ~size_t(15);
  return b + (2 * ns + 2) * sizeof(uint64_t);
}

// offs != nullptr: field f starts at z + offs[f] (scan windows); probe != nullptr:
// the exit wave probe .* window is transformed (the probe rows ride in the same
// ring slot as the window rows, both by bulk copy).
//
// AT = group-A threads. AT = 512 (VC = 2 / 1 columns per thread) is the
// general layout. AT = 256 with VC = 4 (complex64, n2 = 1024) halves the
// per-slot overhead (barrier wait / arrive / addressing) per element: each
// thread owns two column pairs half a row apart (conflict-free LDS.128), and
// the warpgroups hand registers over with setmaxnreg: group A grows to RA, the
// group-B + producer warpgroups shrink to RB (the block is padded to whole
// warpgroups). RA = 0: no register redistribution.
// SPL = 2 (p2 = 64, two slots per lane): two group-B warps per j1, each
// keeping one half of the 64-point transform after its first (in-thread)
// stage -- halves the per-tile FFT + band chain of the q = 8 plans (scan
// windows of the ePIE band stage and the evaluator). The register hand-over
// then runs the other way: group A (one column per thread) shrinks to RA,
// group B grows to RB.
template <int AT, int RR, int P, int SPL = 1>
constexpr int fwd_rows_threads(bool wg_aligned) {
  const int n = AT + 32 * fwd_b_warps<RR, P>() * SPL + 32;
  return wg_aligned ? (n + 127) / 128 * 128 : n;
}

template <class R, int Q, int RR, int P, int VC, int AT = kTmaConsumers, int RA = 0, int RB = 0, int SPL = 1>
__global__ void __launch_bounds__(fwd_rows_threads<AT, RR, P, SPL>(RA > 0), 1)
    kt2_fwd_rows(PftDev<R> pl, BPar<R, Q, RR> bp, const typename CT<R>::C* __restrict__ z, long long ld,
                 long long bstride, int ntiles, int NS, typename CT<R>::C* __restrict__ G, long long gstride,
                 int dbg, const long long* __restrict__ offs, const typename CT<R>::C* __restrict__ probe) {
  using C = typename CT<R>::C;
  constexpr int NBW = fwd_b_warps<RR, P>() * SPL;
  constexpr int BT = 32 * NBW;
  static_assert(VC != 4 || sizeof(R) == 4, "VC = 4: complex64 only");
  static_assert(SPL == 1 || (SPL == 2 && P == 64 && sizeof(R) == 4), "slot split: complex64, p2 = 64 only");
  static_assert(RA == 0 || AT % 128 == 0, "setmaxnreg needs warpgroup-aligned roles");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n2 = pl.n2;
  const int ldT = ldT_of(n2, Q);
  // slot: [row a (n2 + 2)][row b (n2 + 2)][probe row a][probe row b]; a window
  // that starts 8 bytes past a 16-byte boundary (odd complex64 offset) is copied
  // from one element earlier and read with shift 1 (one column per consumer)
  const int lds = n2 + 2;
  const size_t slot_e = 2 * (size_t)lds + (probe ? 2 * (size_t)n2 : 0);
  C* ring = reinterpret_cast<C*>(smem_raw);
  C* T = ring + (size_t)NS * slot_e;  // [RR][ldT]
  constexpr bool HORNER = sizeof(R) == 4;
  constexpr int REC = strip_rec(RR);
  C* W2s = T + (size_t)RR * ldT;  // complex64: [M2] (row 0) then Gst [M2 / 8][REC]; complex128: [RR][M2]
  C* Gst = W2s + pl.M2;
  C* tw2s = W2s + (HORNER ? (size_t)pl.M2 + (size_t)(pl.M2 / kStripNB) * REC : (size_t)RR * pl.M2);
  uint64_t* bars = smem_after<uint64_t>(smem_raw, tw2s + P / 2 + 1, 16);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* tready = bars + 2 * NS;
  uint64_t* tfree = tready + 1;
  if constexpr (HORNER) {
    for (int i = threadIdx.x; i < pl.M2; i += blockDim.x) W2s[i] = pl.W2t[i];
    for (int i = threadIdx.x; i < pl.p2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
  } else {
    fast_load_tables(pl, W2s, tw2s);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], AT);
    }
    mbar_init(tready, 1);
    mbar_init(tfree, 1);
    mbar_fence_init();
  }
  __syncthreads();
  griddep_launch_dependents();
  griddep_wait();  // PDL: the previous kernel's writes (and reads of our outputs) are complete
  const uint32_t row_bytes = (uint32_t)(n2 * sizeof(C));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (RA > 0 && RA >= RB) {
    if (threadIdx.x < AT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RA));
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RB));
  } else if constexpr (RA > 0) {
    if (threadIdx.x < AT) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RA));
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RB));
  }

  if (threadIdx.x >= AT + BT) {
    // ---------------- producer ----------------
    if (threadIdx.x != AT + BT) return;
    const uint64_t pol = l2_evict_first_policy();
    const bool hint = !offs && !PFTG_DBG(dbg, 16);  // scan windows overlap (L2 reuse): no hint; dbg 16: profiling switch
    uint32_t seq = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int f = t / pl.p1, k1 = t % pl.p1;
      const C* base = z + (offs ? offs[f] : (long long)f * bstride) + (long long)k1 * Q * ld;
      const int sh = (int)((reinterpret_cast<uintptr_t>(base) & 15) / sizeof(C));
      const uint32_t wbytes = row_bytes + (sh ? 16u : 0u);
      base -= sh;
      const C* pbase = probe ? probe + (size_t)k1 * Q * n2 : nullptr;
      for (int pi = 0; pi < Q / 2; ++pi, ++seq) {
        const int s = seq % NS;
        if (seq >= NS) mbar_wait(&empty[s], ((seq / NS) - 1) & 1);
        const int la = pi == 0 ? 0 : pi, lb = pi == 0 ? Q / 2 : Q - pi;
        mbar_arrive_expect_tx(&full[s], 2 * wbytes + (pbase ? 2 * row_bytes : 0u));
        C* slot = ring + (size_t)s * slot_e;
        if (hint) {
          bulk_g2s_hint(slot, base + (long long)la * ld, wbytes, &full[s], pol);
          bulk_g2s_hint(slot + lds, base + (long long)lb * ld, wbytes, &full[s], pol);
        } else {
          bulk_g2s(slot, base + (long long)la * ld, wbytes, &full[s]);
          bulk_g2s(slot + lds, base + (long long)lb * ld, wbytes, &full[s]);
        }
        if (pbase) {
          bulk_g2s(slot + 2 * lds, pbase + (size_t)la * n2, row_bytes, &full[s]);
          bulk_g2s(slot + 2 * lds + n2, pbase + (size_t)lb * n2, row_bytes, &full[s]);
        }
      }
    }
    return;
  }

  if (threadIdx.x >= AT) {
    // ---------------- group B: stage B (releases T) + FFT + band ----------------
    constexpr int PL = P < 32 ? P : 32;
    constexpr int S = P / PL;
    constexpr int GPW = 32 / PL;
    constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
    const int lig = lane & (PL - 1), giw = lane / PL;
    const int wb = warp - AT / 32;
    const int half = wb % SPL;                      // SPL = 2: which slot this warp keeps
    const int j1 = (wb / SPL) * GPW + giw;  // NBW * GPW >= RR * SPL: one j1 per lane group (pair)
    const bool valid = j1 < RR;
    const int M2 = pl.M2, mt2 = pl.mt2;
    uint32_t i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int f = t / pl.p1, k1 = t % pl.p1;
      mbar_wait(tready, i & 1);
      if PFTG_DBG(dbg, 1) {  // profiling experiment: group B only hands T back
        named_sync(2, BT);
        if (threadIdx.x == AT) mbar_arrive(tfree);
        continue;
      }
      C x[S][RR];
#pragma unroll
      for (int ss = 0; ss < S; ++ss) {
#pragma unroll
        for (int j = 0; j < RR; ++j) x[ss][j] = czero<C>();
        if (valid) {
          const int k2 = ss * PL + lig;
          const C* trow = T + (size_t)j1 * ldT + (size_t)k2 * (Q + 1);
          {
            const C t0 = trow[0], th = trow[Q / 2];
#pragma unroll
            for (int j = 0; j < RR; ++j) bmac(x[ss][j], bp.b2[0][j], t0, j & 1);
            bmac(x[ss][0], bp.b2[Q / 2][0], th, false);
          }
#pragma unroll
          for (int l = 1; l < Q / 2; ++l) {
            const C a = trow[l], b = trow[Q - l];
            const C sp = cadd(a, b), dm = csub(a, b);
#pragma unroll
            for (int j = 0; j < RR; ++j) bmac(x[ss][j], bp.b2[l][j], (j & 1) ? dm : sp, j & 1);
          }
        }
      }
      // the previous tile's G records (bulk stores below) have left the staging block
      if (HORNER && gstride > 0 && threadIdx.x == AT) bulk_wait_read();
      named_sync(2, BT);  // group B is done reading T: group A may overwrite it
      if (threadIdx.x == AT) mbar_arrive(tfree);
      if PFTG_DBG(dbg, 8) {  // profiling experiment: stage B only
        if (x[0][0].x == 1234.5f) G[0] = x[0][1];
        continue;
      }
      if constexpr (SPL == 2) {
        // first DIF stage (slot pair, h = 32) in-thread, then this warp keeps one slot:
        // the remaining cross-lane stages use the same twiddles as the S = 2 transform
        C xh[1][RR];
        const C w = twiddle(tw2s, lig, -1);
#pragma unroll
        for (int j = 0; j < RR; ++j) xh[0][j] = half ? cmul(csub(x[0][j], x[1][j]), w) : cadd(x[0][j], x[1][j]);
        fft_dif<1, RR>(xh, P, PL, lig, tw2s, -1);
        if PFTG_DBG(dbg, 4) {  // profiling experiment: stage B + FFT, no band
          if (xh[0][0].x == 1234.5f) G[0] = xh[0][1];
          continue;
        }
        if (valid) {
          const int u2 = bitrev(half * PL + lig, LP);
          band_horner<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, mt2, R(1) / R(P), xh[0], [&](int b, C v) {
            Gst[(size_t)(b / kStripNB) * REC + j1 * kStripNB + (b % kStripNB)] = v;
          });
        }
      } else {
        fft_dif<S, RR>(x, P, PL, lig, tw2s, -1);
        if PFTG_DBG(dbg, 4) {  // profiling experiment: stage B + FFT, no band
          if (x[0][0].x == 1234.5f) G[0] = x[0][1];
          continue;
        }
      }
      if constexpr (HORNER) {
        // band by Horner into the staging block, then coalesced record copies:
        // this tile owns record (strip, k1) = 80 contiguous elements of every strip
        if (SPL == 1 && valid) {
#pragma unroll
          for (int ss = 0; ss < S; ++ss) {
            const int u2 = bitrev(ss * PL + lig, LP);
            band_horner<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, mt2, R(1) / R(P), x[ss], [&](int b, C v) {
              Gst[(size_t)(b / kStripNB) * REC + j1 * kStripNB + (b % kStripNB)] = v;
            });
          }
        }
        named_sync(2, BT);  // staging block complete
        const int tb = threadIdx.x - AT;
        constexpr int NREC = RR * kStripNB;
        const int nrec = M2 / kStripNB;
        if PFTG_DBG(dbg, 32) continue;  // profiling experiment: band staged, no G stores
        if (gstride > 0) {
          // one 1-D bulk store per (strip, k1) record (16-byte aligned: strip_rec); the
          // staging block is reused after bulk_wait_read() at the next tile's stage B
          if (threadIdx.x == AT) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // tile-major layout G[f][k1][strip][REC]: the tile's records are one contiguous block
            bulk_s2g(G + (size_t)f * gstride + (size_t)k1 * nrec * REC, Gst, (uint32_t)(nrec * REC * sizeof(C)));
            bulk_commit();
          }
        } else {
          C* Gblk = G + ((size_t)f * pl.p1 + k1) * RR * M2;
          for (int e = tb; e < RR * M2; e += BT) {
            const int jj = e / M2, b = e - jj * M2;
            Gblk[e] = Gst[(size_t)(b / kStripNB) * REC + jj * kStripNB + (b % kStripNB)];
          }
        }
      } else {
        if (!valid) continue;
#pragma unroll
        for (int ss = 0; ss < S; ++ss) {
          const int u2 = bitrev(ss * PL + lig, LP);
          if (gstride > 0) {
            C* gstrip = G + (size_t)f * gstride;
            band_contract<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, RR, x[ss], [&](int b, C v) {
              gstrip[((size_t)k1 * (M2 / kStripNB) + b / kStripNB) * REC + j1 * kStripNB + (b % kStripNB)] = v;
            });
          } else {
            C* Gblk = G + ((size_t)f * pl.p1 + k1) * RR * M2;
            band_contract<RR>(W2s, M2, (u2 + mt2) & (P - 1), P, RR, x[ss],
                              [&](int b, C v) { Gblk[(size_t)j1 * M2 + b] = v; });
          }
        }
      }
    }
    if (HORNER && gstride > 0 && threadIdx.x == AT) bulk_wait_all();  // G records written before exit
    return;
  }

  // ---------------- group A: stream + stage A -> T ----------------
  // column of this thread's v-th accumulator
  auto colv = [&](int v) { return VC == 4 ? 2 * (int)threadIdx.x + (v & 1) + (v >> 1) * (n2 >> 1) : (int)threadIdx.x * VC + v; };
  const int c0 = threadIdx.x * VC;
  const bool dbg_stream = VC != 4 && PFTG_DBG(dbg, 2) != 0;
  // shared-memory byte address of this thread's first column in slot 0 (VC = 4)
  const uint32_t abase = smem_u32(ring) + 16u * threadIdx.x;
  const uint32_t slot_bytes = (uint32_t)(slot_e * sizeof(C));
  // ring position (slot, phase) advanced incrementally: no division in the unrolled loop
  int s = 0;
  uint32_t ph = 0;
  uint32_t i = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    // alignment shift of this tile's window rows in the slot (see the producer)
    const int sh = offs ? (int)((reinterpret_cast<uintptr_t>(z + offs[t / pl.p1]) & 15) / sizeof(C)) : 0;
    C acc[VC][RR];
#pragma unroll
    for (int v = 0; v < VC; ++v)
#pragma unroll
      for (int j = 0; j < RR; ++j) acc[v][j] = czero<C>();
#pragma unroll
    for (int pi = 0; pi < Q / 2; ++pi) {
      mbar_wait(&full[s], ph);
      const C* slot = ring + (size_t)s * slot_e;
      C a[VC], b[VC];
      if constexpr (VC == 4) {  // host guarantees n2 == AT * VC, sh == 0 and no probe here
        constexpr uint32_t N2 = AT * VC, ROWB = (N2 + 2) * 8;
        const uint32_t sa = abase + (uint32_t)s * slot_bytes;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float4 ta = lds128(sa + hh * (N2 / 2) * 8);
          const float4 tb = lds128(sa + ROWB + hh * (N2 / 2) * 8);
          a[2 * hh] = CT<R>::mk(ta.x, ta.y);
          a[2 * hh + 1] = CT<R>::mk(ta.z, ta.w);
          b[2 * hh] = CT<R>::mk(tb.x, tb.y);
          b[2 * hh + 1] = CT<R>::mk(tb.z, tb.w);
        }
      } else if constexpr (VC == 2 && sizeof(C) == 8) {
        if (sh == 0) {  // 16-byte phase (plain fields, even window offsets)
          const float4 ta = *reinterpret_cast<const float4*>(slot + c0);
          const float4 tb = *reinterpret_cast<const float4*>(slot + lds + c0);
          a[0] = CT<R>::mk(ta.x, ta.y);
          a[VC - 1] = CT<R>::mk(ta.z, ta.w);
          b[0] = CT<R>::mk(tb.x, tb.y);
          b[VC - 1] = CT<R>::mk(tb.z, tb.w);
        } else {
#pragma unroll
          for (int v = 0; v < VC; ++v) {
            a[v] = slot[sh + c0 + v];
            b[v] = slot[lds + sh + c0 + v];
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < VC; ++v) {
          a[v] = slot[sh + c0 + v];
          b[v] = slot[lds + sh + c0 + v];
        }
      }
      if (VC != 4 && probe) {  // exit wave: probe * window (stage_a_pairs order)
#pragma unroll
        for (int v = 0; v < VC; ++v) {
          a[v] = cmul(slot[2 * lds + c0 + v], a[v]);
          b[v] = cmul(slot[2 * lds + n2 + c0 + v], b[v]);
        }
      }
      mbar_arrive(&empty[s]);  // every consumer thread arrives (count AT): no warp sync needed
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
      if (dbg_stream) {  // profiling experiment: group A only consumes the ring
        acc[0][0].x += a[0].x + b[0].y;
        continue;
      }
#pragma unroll
      for (int v = 0; v < VC; ++v) {
        if (pi == 0) {
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[0][j], a[v], j & 1);
          bmac(acc[v][0], bp.b1[Q / 2][0], b[v], false);
        } else {
          const C sp = cadd(a[v], b[v]), dm = csub(a[v], b[v]);
#pragma unroll
          for (int j = 0; j < RR; ++j) bmac(acc[v][j], bp.b1[pi][j], (j & 1) ? dm : sp, j & 1);
        }
      }
    }
    if (i >= 1) mbar_wait(tfree, (i - 1) & 1);  // group B has finished stage B of the previous block
#pragma unroll
    for (int v = 0; v < VC; ++v) {
      const int c = colv(v);
      const int tc = c + c / Q;
#pragma unroll
      for (int j = 0; j < RR; ++j) T[(size_t)j * ldT + tc] = acc[v][j];
    }
    named_sync(1, AT);
    if (threadIdx.x == 0) mbar_arrive(tready);
  }
}

// ---------------------------------------------------------------------------
// Warp-specialized persistent adjoint rows pass (pft_adjoint_2d second half,
// pft.cpp:205-224). One CTA per SM loops over (field, k1) row blocks:
//   group P1 (one warp per j1): D-dagger gather of the block's r1 x M2 slice
//     (prefetched by a 1-D bulk copy into a double buffer), inverse FFT over
//     k2 in registers, B2-dagger expansion with row-pair symmetry -> T[i & 1];
//   group P2 (10 warps): A-dagger expansion of T[i & 1] with row-pair symmetry
//     and 128-bit streaming stores of the q1 output rows.
// T is double-buffered, so P1 builds block i+1 while P2 writes block i; the two
// groups hand off through mbarriers (tready / tfree). W2 is read through L1.
constexpr int kAdjP2Warps = 10;

template <int RR, int P>
constexpr int adj_p1_warps() {
  constexpr int gpw = 32 / (P < 32 ? P : 32);
  return (RR + gpw - 1) / gpw;
}

template <class R>
__host__ __device__ inline size_t tma_adj_smem(int n2, int q, int r, int M2, int p) {
  using C = typename CT<R>::C;
  size_t b = sizeof(C) * (2 * (size_t)r * ldT_of(n2, q) + p / 2 + 1 + 2 * (size_t)r * M2);
  b = (b + 15) & ~size_t(15);
  return b + 128 + 8 * sizeof(uint64_t) + 4096;  // alignment slack, barriers, coefficient tables
}

//
// Wide variant (RA > 0, complex64, n2 == P2T * VC with VC = 4): P2 is 8 warps
// (256 threads x 4 columns, two column pairs half a row apart, so each row is
// exactly one round of 128-bit stores), placed first so the roles are whole
// warpgroups; setmaxnreg moves registers from P1 (RB) to P2 (RA). The default
// layout (P1 first, 10 P2 warps x 2 columns) needs 1.6 rounds per row.
template <int RR, int P, int P2T>
constexpr int adj_rows_threads(bool wide) {
  const int n = 32 * adj_p1_warps<RR, P>() + P2T;
  return wide ? (n + 127) / 128 * 128 : n;
}

template <class R, int Q, int RR, int P, int VC, int P2T_ = 32 * kAdjP2Warps, int RA = 0, int RB = 0>
__global__ void __launch_bounds__(adj_rows_threads<RR, P, P2T_>(RA > 0), 1)
    kt_adj_rows(PftDev<R> pl, BPar<R, Q, RR> bp, const typename CT<R>::C* __restrict__ Gt,
                typename CT<R>::C* __restrict__ out, int ntiles, int dbg) {
  using C = typename CT<R>::C;
  constexpr int NP1 = adj_p1_warps<RR, P>();
  constexpr int P1T = 32 * NP1, P2T = P2T_;
  constexpr bool WIDE = RA > 0;
  static_assert(!WIDE || (VC == 4 && sizeof(R) == 4 && P2T % 128 == 0), "wide adjoint rows: complex64, VC = 4");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n2 = pl.n2, M2 = pl.M2, mt2 = pl.mt2;
  const int ldT = ldT_of(n2, Q);
  C* Tb = reinterpret_cast<C*>(smem_raw);  // [2][RR][ldT]
  C* tw2s = Tb + 2 * (size_t)RR * ldT;
  constexpr int RP = brow_pad<R, RR>();
  R* btab1 = smem_after<R>(smem_raw, tw2s + P / 2 + 1, 16);
  R* btab2 = btab1 + (Q / 2 + 1) * RP;
  C* gbuf = smem_after<C>(smem_raw, btab2 + (Q / 2 + 1) * RP, 128);  // [2][RR * M2]
  uint64_t* bars = smem_after<uint64_t>(smem_raw, gbuf + 2 * (size_t)RR * M2, 16);
  uint64_t* gfull = bars;       // TMA -> P1
  uint64_t* tready = bars + 2;  // P1 -> P2
  uint64_t* tfree = bars + 4;   // P2 -> P1
  const C* W2g = pl.W2t;        // L1-resident table

  for (int i = threadIdx.x; i < P / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
  stage_btab<R, Q, RR>(bp.b1, btab1);
  stage_btab<R, Q, RR>(bp.b2, btab2);
  const uint32_t blk_bytes = (uint32_t)(RR * M2 * sizeof(C));
  griddep_launch_dependents();
  griddep_wait();  // PDL: Gt is the previous kernel's output
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&gfull[s], 1);
      mbar_init(&tready[s], 1);
      mbar_init(&tfree[s], 1);
    }
    mbar_fence_init();
    for (int s = 0; s < 2; ++s) {  // prefetch the first two blocks
      const int t = blockIdx.x + s * gridDim.x;
      if (t < ntiles) {
        mbar_arrive_expect_tx(&gfull[s], blk_bytes);
        bulk_g2s(gbuf + (size_t)s * RR * M2, Gt + (size_t)t * RR * M2, blk_bytes, &gfull[s]);
      }
    }
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // role layout: default P1 warps [0, NP1) then P2; wide: P2 threads [0, P2T) then P1, then padding
  const int p1w = WIDE ? warp - P2T / 32 : warp;
  if constexpr (WIDE) {
    if ((int)threadIdx.x < P2T) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RA));
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RB));
    if (p1w >= NP1) return;  // padding warps
  }
  if (p1w >= 0 && p1w < NP1) {
    // ---------------- P1: gather + inverse FFT + B2-dagger -> T ----------------
    constexpr int PL = P < 32 ? P : 32;
    constexpr int S = P / PL;
    constexpr int GPW = 32 / PL;
    constexpr int LP = (P >= 128) ? 7 : (P >= 64) ? 6 : (P >= 32) ? 5 : (P >= 16) ? 4 : (P >= 8) ? 3 : (P >= 4) ? 2 : 1;
    const int lig = lane & (PL - 1), giw = lane / PL;
    const int j1 = p1w * GPW + giw;
    const bool valid = j1 < RR;
    const bool leader = p1w == 0 && lane == 0;
    uint32_t i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int s = i & 1;
      const C* Gblk = gbuf + (size_t)s * RR * M2;
      C* T = Tb + (size_t)s * RR * ldT;
      mbar_wait(&gfull[s], (i >> 1) & 1);
      if (i >= 2) mbar_wait(&tfree[s], ((i >> 1) - 1) & 1);
      if (!PFTG_DBG(dbg, 1)) {
        C x[S][RR];
#pragma unroll
        for (int ss = 0; ss < S; ++ss) {
#pragma unroll
          for (int j = 0; j < RR; ++j) x[ss][j] = czero<C>();
          if (valid) {
            const int u2 = ss * PL + lig;
            for (int b = (u2 + mt2) & (P - 1); b < M2; b += P) {
              const C g = Gblk[(size_t)j1 * M2 + b];
              if constexpr (sizeof(R) == 4) {
                gather_horner<RR>(x[ss], __ldg(W2g + b), static_cast<R>(b - mt2) * (R(1) / R(P)), g);
              } else {
#pragma unroll
                for (int j = 0; j < RR; ++j) cmacc(x[ss][j], __ldg(W2g + j * M2 + b), g);
              }
            }
          }
        }
        fft_dif<S, RR>(x, P, PL, lig, tw2s, +1);
        if (valid) {
#pragma unroll
          for (int ss = 0; ss < S; ++ss) {
            const int k2 = bitrev(ss * PL + lig, LP);
            C* trow = T + (size_t)j1 * ldT + (size_t)k2 * (Q + 1);
            C xs[1][RR];
#pragma unroll
            for (int j = 0; j < RR; ++j) xs[0][j] = x[ss][j];
            expand_pairs_sm<R, Q, RR, 1>(
                btab2, xs, [&](int l, const C (&z)[1]) { trow[l] = z[0]; },
                [&](int l, const C (&zl)[1], const C (&zm)[1]) {
                  trow[l] = zl[0];
                  trow[Q - l] = zm[0];
                });
          }
        }
      }
      named_sync(1, P1T);  // all of P1 is done with gbuf[s] and T[s]
      if (leader) {
        mbar_arrive(&tready[s]);
        const int tn = t + 2 * (int)gridDim.x;
        if (tn < ntiles) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(&gfull[s], blk_bytes);
          bulk_g2s(gbuf + (size_t)s * RR * M2, Gt + (size_t)tn * RR * M2, blk_bytes, &gfull[s]);
        }
      }
    }
    return;
  }

  // ---------------- P2: A-dagger expansion + streaming stores ----------------
  const int tid = WIDE ? (int)threadIdx.x : (int)threadIdx.x - P1T;
  uint32_t i = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int s = i & 1;
    const int f = t / pl.p1, k1 = t % pl.p1;
    const C* T = Tb + (size_t)s * RR * ldT;
    mbar_wait(&tready[s], (i >> 1) & 1);
    C* o = out + ((size_t)f * pl.n1 + (size_t)k1 * Q) * n2;
    if (WIDE && PFTG_DBG(dbg, 4)) {
      // profiling experiment: P2 idle (P1 alone)
    } else if constexpr (WIDE) {
      // columns 2 tid + {0, 1} and 2 tid + n2 / 2 + {0, 1}; one pass covers the row
      constexpr int N2 = P2T * VC;
      C tv[VC][RR];
#pragma unroll
      for (int v = 0; v < VC; ++v) {
        const int c = 2 * tid + (v & 1) + (v >> 1) * (N2 / 2);
        const int tc = c + c / Q;
#pragma unroll
        for (int j = 0; j < RR; ++j) tv[v][j] = T[(size_t)j * ldT + tc];
      }
      C* ob = o + 2 * tid;
      auto store = [&](int l, const C (&z)[VC]) {
        // streaming (evict-first) stores: the output is not re-read, Gt should stay in L2
        __stcs(reinterpret_cast<float4*>(ob + (size_t)l * N2), make_float4(z[0].x, z[0].y, z[1].x, z[1].y));
        __stcs(reinterpret_cast<float4*>(ob + (size_t)l * N2 + N2 / 2), make_float4(z[2].x, z[2].y, z[3].x, z[3].y));
      };
      expand_pairs_sm<R, Q, RR, VC>(btab1, tv, store, [&](int l, const C (&zl)[VC], const C (&zm)[VC]) {
        store(l, zl);
        store(Q - l, zm);
      });
    } else if (!PFTG_DBG(dbg, 4)) {
      for (int c = tid * VC; c < n2; c += P2T * VC) {
        C tv[VC][RR];
#pragma unroll
        for (int v = 0; v < VC; ++v) {
          const int tc = (c + v) + (c + v) / Q;
#pragma unroll
          for (int j = 0; j < RR; ++j) tv[v][j] = T[(size_t)j * ldT + tc];
        }
        auto store = [&](int l, const C (&z)[VC]) {
          if constexpr (VC == 2 && sizeof(C) == 8) {
            *reinterpret_cast<float4*>(o + (size_t)l * n2 + c) = make_float4(z[0].x, z[0].y, z[VC - 1].x, z[VC - 1].y);
          } else {
#pragma unroll
            for (int v = 0; v < VC; ++v) o[(size_t)l * n2 + c + v] = z[v];
          }
        };
        expand_pairs_sm<R, Q, RR, VC>(btab1, tv, store, [&](int l, const C (&zl)[VC], const C (&zm)[VC]) {
          store(l, zl);
          store(Q - l, zm);
        });
      }
    }
    named_sync(2, P2T);  // all of P2 is done reading T[s]
    if (tid == 0) mbar_arrive(&tfree[s]);
  }
}

}  // namespace pftg
