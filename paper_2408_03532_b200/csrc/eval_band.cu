// PFT band residual of the forward-model evaluator for the q = 8 plans
// (BASELINE configs[4]: 512 x 512 complex64 windows, p = 64, r = 9, M = 128):
//   band_j = PFT2(P .* z_j),  sum (|band_j| - dcrop_j)^2
// (pft_apply_2d, /root/reference/proj/core/src/pft.cpp:119-172, applied to the
// exit wave of solver.cpp:240; residual as in solver.cpp:61-69 / 89-102).
//
// The 2-D PFT is the tensor product of the two 1-D PFTs, so the axis order is
// free. The batched kernels (pft_tma.cuh) contract axis 1 first, which for the
// q = 32 plans shrinks the streamed rows 32 -> 10 before anything else happens.
// For q = 8, r = 9 that order *expands* the data (8 rows -> 9) at full row
// width and then runs 9 slice transforms per row block. Here axis 2 goes first:
//   kb_rows  one warp per window row: exit wave, stage B (contract l2), 64-point
//            FFT over k2, Horner band -> M2 values per row; then stage A
//            (contract the q1 rows of the block with B1) on the M2-wide band
//            rows instead of the n2-wide window rows -> G[f][k1][j1][b];
//   kb_cols  per 8-column strip: 64-point FFTs over k1 as two radix-8 register
//            passes through shared memory, Horner band over j1, residual sum.
// 8 instead of 9 slice transforms per row block, stage A on a quarter of the
// columns, and ordinary multi-CTA occupancy instead of one persistent CTA per
// SM (the window rows come from L2, there is no HBM stream to keep busy).
#include <cstdlib>

#include "eval_fft.cuh"
#include "internal.hpp"
#include "pft_fast.cuh"

namespace pftg {
namespace {

// 16-byte chunk j (two complex64) of the 8-element group g of a staged row,
// XOR-swizzled so that both the coalesced 8-byte writes (lane = element) and
// the 16-byte reads (lane = group) are bank-conflict-free.
__device__ __forceinline__ int eb_chunk(int g, int j) { return g * 4 + (j ^ ((g >> 1) & 3)); }

template <int RR>
struct EbPar {
  float b1[5][RR];
  float b2[5][RR];
};

// x[j] = sum_l B[l][j] t[l] over the 8 nodes with the pair symmetry
// B[8 - l][j] = (-1)^j B[l][j] (minimax.cpp:326-330); b[l][j] for l <= 4.
template <int RR>
__device__ __forceinline__ void eb_contract8(const float (&b)[5][RR], const float2 (&t)[8], float2 (&x)[RR]) {
#pragma unroll
  for (int j = 0; j < RR; ++j) x[j] = czero<float2>();
#pragma unroll
  for (int j = 0; j < RR; ++j) bmac(x[j], b[0][j], t[0], j & 1);
  bmac(x[0], b[4][0], t[4], false);
#pragma unroll
  for (int l = 1; l < 4; ++l) {
    const float2 sp = cadd(t[l], t[8 - l]), dm = csub(t[l], t[8 - l]);
#pragma unroll
    for (int j = 0; j < RR; ++j) bmac(x[j], b[l][j], (j & 1) ? dm : sp, j & 1);
  }
}

// Stage A on the q1 = 8 band rows of a row block (rows[l * ld + pos(b)], even b
// first then odd b): G[j1][b] = sum_l B1[l][j1] rows[l][b]. Thread (m = tid & 63, group g)
// owns columns 2m, 2m + 1 and j1 = g (mod 4); the four groups may sit in one CTA
// (g = tid >> 6) or in the two CTAs of a cluster pair.
template <int RR>
__device__ __forceinline__ void eb_stage_a(const EbPar<RR>& bp, const float2* rows, int ld, int M2, float2* Gt,
                                           int g) {
  const int hM = M2 >> 1;
  for (int m = threadIdx.x & 63; m < hM; m += 64) {
    float2 te[8], to[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      te[l] = rows[l * ld + m];
      to[l] = rows[l * ld + hM + m];
    }
    const float2 spe[3] = {cadd(te[1], te[7]), cadd(te[2], te[6]), cadd(te[3], te[5])};
    const float2 dme[3] = {csub(te[1], te[7]), csub(te[2], te[6]), csub(te[3], te[5])};
    const float2 spo[3] = {cadd(to[1], to[7]), cadd(to[2], to[6]), cadd(to[3], to[5])};
    const float2 dmo[3] = {csub(to[1], to[7]), csub(to[2], to[6]), csub(to[3], to[5])};
#pragma unroll
    for (int j = 0; j < RR; ++j) {
      if ((j & 3) != g) continue;  // warp-uniform
      float2 ae = czero<float2>(), ao = czero<float2>();
      bmac(ae, bp.b1[0][j], te[0], j & 1);
      bmac(ao, bp.b1[0][j], to[0], j & 1);
      if (j == 0) {
        bmac(ae, bp.b1[4][0], te[4], false);
        bmac(ao, bp.b1[4][0], to[4], false);
      }
#pragma unroll
      for (int l = 1; l < 4; ++l) {
        bmac(ae, bp.b1[l][j], (j & 1) ? dme[l - 1] : spe[l - 1], j & 1);
        bmac(ao, bp.b1[l][j], (j & 1) ? dmo[l - 1] : spo[l - 1], j & 1);
      }
      *reinterpret_cast<float4*>(Gt + (size_t)j * M2 + 2 * m) = make_float4(ae.x, ae.y, ao.x, ao.y);
    }
  }
}

// out[l] = sum_j conj(B[l][j]) x[j] for the 8 nodes (adjoint of eb_contract8).
template <int RR>
__device__ __forceinline__ void eb_expand8(const float (&b)[5][RR], const float2 (&x)[RR], float2 (&out)[8]) {
  float2 e0 = czero<float2>(), h = czero<float2>();
#pragma unroll
  for (int j = 0; j < RR; ++j) bmacc(e0, b[0][j], x[j], j & 1);
  bmacc(h, b[4][0], x[0], false);
  out[0] = e0;
  out[4] = h;
#pragma unroll
  for (int l = 1; l < 4; ++l) {
    float2 e = czero<float2>(), o = czero<float2>();
#pragma unroll
    for (int j = 0; j < RR; j += 2) bmacc(e, b[l][j], x[j], false);
#pragma unroll
    for (int j = 1; j < RR; j += 2) bmacc(o, b[l][j], x[j], false);  // conj(i b) = -i b applied once
    out[l] = cadd_mi(e, o);
    out[8 - l] = csub_mi(e, o);
  }
}

// 8 consecutive complex64 (one k2 group of a row); vec: 16-byte aligned.
__device__ __forceinline__ void eb_load8(const float2* p, bool vec, float2 (&v)[8]) {
  if (vec) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 q = *reinterpret_cast<const float4*>(p + 2 * j);
      v[2 * j] = make_float2(q.x, q.y);
      v[2 * j + 1] = make_float2(q.z, q.w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = p[j];
  }
}
__device__ __forceinline__ void eb_store8(float2* p, bool vec, const float2 (&v)[8]) {
  if (vec) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(p + 2 * j) = make_float4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = v[j];
  }
}

// grid (p1, batch), 256 threads: warp w <-> row k1 * 8 + w of the window.
template <int RR, int P2>
__global__ void __launch_bounds__(256, 3)
    kb_rows(PftDev<float> pl, EbPar<RR> bp, const float2* __restrict__ frame, long long ld, long long bstride,
            const long long* __restrict__ offs, const float2* __restrict__ probe, float2* __restrict__ G) {
  constexpr int S = P2 / 32;  // k2 slots per lane
  constexpr int N2 = P2 * 8;  // row length
  constexpr int LP = P2 == 64 ? 6 : 5;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* stage = reinterpret_cast<float2*>(smem_raw);  // [8][N2]: exit-wave rows, then band rows
  float2* W2s = stage + 8 * N2;                         // [M2] row 0 of W2 (Horner band)
  float2* tw2s = W2s + pl.M2;                           // [P2 / 2]
  const int k1 = blockIdx.x, f = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M2 = pl.M2, mt2 = pl.mt2;
  float2* st = stage + warp * N2;
  {
    // field row (scan window: frame + offs[f]; batched fields: frame + f * bstride), times the
    // probe row when there is one (exit wave), coalesced: element c = 32 m + lane
    const float2* zrow = frame + (offs ? offs[f] : (long long)f * bstride) + (long long)(k1 * 8 + warp) * ld;
    float2 v[N2 / 32];
#pragma unroll
    for (int m = 0; m < N2 / 32; ++m) v[m] = __ldg(zrow + 32 * m + lane);
    if (probe) {
      const float2* prow = probe + (size_t)(k1 * 8 + warp) * N2;
      float2 pv[N2 / 32];
#pragma unroll
      for (int m = 0; m < N2 / 32; ++m) pv[m] = __ldg(prow + 32 * m + lane);
#pragma unroll
      for (int m = 0; m < N2 / 32; ++m) v[m] = cmul(pv[m], v[m]);
    }
    for (int i = threadIdx.x; i < M2; i += blockDim.x) W2s[i] = pl.W2t[i];
    for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
#pragma unroll
    for (int m = 0; m < N2 / 32; ++m) {
      const int c = 32 * m + lane, g = c >> 3, e = c & 7;
      st[eb_chunk(g, e >> 1) * 2 + (e & 1)] = v[m];
    }
  }
  __syncthreads();
  float2 x[S][RR];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int k2 = s * 32 + lane;
    float2 t[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 q = *reinterpret_cast<const float4*>(st + eb_chunk(k2, j) * 2);
      t[2 * j] = make_float2(q.x, q.y);
      t[2 * j + 1] = make_float2(q.z, q.w);
    }
    eb_contract8<RR>(bp.b2, t, x[s]);
  }
  __syncwarp();  // the row is consumed: its staging block takes the band row
  fft_dif<S, RR>(x, P2, 32, lane, tw2s, -1);
  // band row, even b first then odd b (the stores of one slot share a parity)
  const int hM = M2 >> 1;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int u2 = bitrev(s * 32 + lane, LP);
    band_horner<RR>(W2s, M2, (u2 + mt2) & (P2 - 1), P2, mt2, 1.0f / P2, x[s],
                    [&](int b, float2 v) { st[(b & 1) * hM + (b >> 1)] = v; });
  }
  __syncthreads();
  eb_stage_a<RR>(bp, stage, N2, M2, G + ((size_t)f * pl.p1 + k1) * RR * M2, threadIdx.x >> 6);
}

// Adjoint rows pass of the q = 8 plans with the ePIE epilogues, axis 1 first
// (the mirror image of kb_rows; pft_adjoint_2d second half, pft.cpp:205-224):
// grid (p1, batch), 256 threads, warp w <-> output row k1 * 8 + w.
//   A-dagger on the band-limited side: R[b] = sum_j1 conj(B1[w][j1]) Gt[k1][j1][b]
//   for exactly the band columns this lane's D-dagger gather needs; inverse FFT
//   over u2; B2-dagger expansion -> 8 consecutive row elements per (lane, slot):
//   the whole output row without a shared-memory intermediate.
//   EPI 0: out[f] row; EPI 1: object window -= beta conj(P) z (solver.cpp:244-245)
//   and, with G2, the forward rows pass of the new exit wave P z' (solver.cpp:247);
//   EPI 2: probe -= gamma conj(window) z (solver.cpp:249-250) and, with G2, the
//   forward rows pass of the NEXT position's exit wave P' z[obj_off2].
// The fused forward continues in the same registers: stage B on the lane's own
// k2 groups (k2 bit-reversed), DIT FFT -> natural u2, Horner band, stage A.
// CL = 2: a cluster pair of 128-thread CTAs per row block (4 rows each, on two
// SMs): every warp also writes its band row into the partner's shared memory
// (DSMEM), and each CTA runs stage A for two of the four j1 groups.
template <int RR, int P2, int EPI, int CL>
__global__ void __launch_bounds__(256 / CL, 1)
    kb_adj_rows(PftDev<float> pl, EbPar<RR> bp, const float2* __restrict__ Gt, EpiArgs ep) {
  constexpr int S = P2 / 32, N2 = P2 * 8;
  constexpr int LP = P2 == 64 ? 6 : 5;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M2 = pl.M2, mt2 = pl.mt2;
  float2* rb = reinterpret_cast<float2*>(smem_raw);  // [8][M2] band rows of the fused forward
  float2* W2s = rb + 8 * M2;                         // [M2] row 0 of W2
  float2* tw2s = W2s + M2;                           // [P2 / 2]
  const int k1 = blockIdx.x / CL, half = blockIdx.x % CL, f = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) + half * (8 / CL);  // row of the block
  const long long row = (long long)k1 * 8 + warp;
  const bool fuse = EPI >= 1 && ep.G2 != nullptr;
  const float st = (float)ep.step;
  for (int i = threadIdx.x; i < M2; i += blockDim.x) W2s[i] = pl.W2t[i];
  for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
  float b1r[RR];
#pragma unroll
  for (int j = 0; j < RR; ++j) b1r[j] = __ldg(pl.Bv1 + warp * RR + j);
  int k2s[S];
#pragma unroll
  for (int s = 0; s < S; ++s) k2s[s] = bitrev(s * 32 + lane, LP);
  // the epilogue's operands, requested before the transform chain
  float2 pv[S][8], ov[S][8], on[S][8];
  float2* orow = nullptr;
  float2* prow = nullptr;
  bool vec_o = false;
  if (EPI >= 1) {
    orow = reinterpret_cast<float2*>(ep.obj) + ep.obj_off + row * ep.obj_ld;
    prow = reinterpret_cast<float2*>(ep.probe) + row * N2;
    vec_o = (reinterpret_cast<uintptr_t>(orow) & 15) == 0;
    const bool vec_p = (reinterpret_cast<uintptr_t>(prow) & 15) == 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      eb_load8(prow + k2s[s] * 8, vec_p, pv[s]);
      eb_load8(orow + k2s[s] * 8, vec_o, ov[s]);
    }
    if (EPI == 2 && fuse) {
      const float2* nrow = reinterpret_cast<const float2*>(ep.obj) + ep.obj_off2 + row * ep.obj_ld;
      const bool vec_n = (reinterpret_cast<uintptr_t>(nrow) & 15) == 0;
#pragma unroll
      for (int s = 0; s < S; ++s) eb_load8(nrow + k2s[s] * 8, vec_n, on[s]);
    }
  }
  griddep_wait();  // PDL: Gt is the previous kernel's output; everything above is not
  griddep_launch_dependents();
  const float2* Gblk = Gt + ((size_t)f * pl.p1 + k1) * RR * M2;
  float2 Rv[S][2];
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = ((s * 32 + lane + mt2) & (P2 - 1)) + P2 * i;
      float2 acc = czero<float2>();
      if (b < M2) {
#pragma unroll
        for (int j = 0; j < RR; ++j) bmacc(acc, b1r[j], Gblk[(size_t)j * M2 + b], j & 1);
      }
      Rv[s][i] = acc;
    }
  __syncthreads();  // tables
  float2 x[S][RR];
#pragma unroll
  for (int s = 0; s < S; ++s) {
#pragma unroll
    for (int j = 0; j < RR; ++j) x[s][j] = czero<float2>();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = ((s * 32 + lane + mt2) & (P2 - 1)) + P2 * i;
      if (b < M2) gather_horner<RR>(x[s], W2s[b], static_cast<float>(b - mt2) * (1.0f / P2), Rv[s][i]);
    }
  }
  fft_dif<S, RR>(x, P2, 32, lane, tw2s, +1);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    float2 z[8], e[8];
    eb_expand8<RR>(bp.b2, x[s], z);
    if (EPI == 0) {
      float2* out = reinterpret_cast<float2*>(ep.out) + ((size_t)f * pl.n1 + row) * N2 + k2s[s] * 8;
      eb_store8(out, (reinterpret_cast<uintptr_t>(out) & 15) == 0, z);
    } else if (EPI == 1) {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float2 g = cmulc(pv[s][l], z[l]);
        ov[s][l].x -= st * g.x;
        ov[s][l].y -= st * g.y;
        e[l] = cmul(pv[s][l], ov[s][l]);
      }
      eb_store8(orow + k2s[s] * 8, vec_o, ov[s]);
    } else {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float2 g = cmulc(ov[s][l], z[l]);
        pv[s][l].x -= st * g.x;
        pv[s][l].y -= st * g.y;
        e[l] = cmul(pv[s][l], on[s][l]);
      }
      eb_store8(prow + k2s[s] * 8, (reinterpret_cast<uintptr_t>(prow) & 15) == 0, pv[s]);
    }
    if (fuse) eb_contract8<RR>(bp.b2, e, x[s]);
  }
  if (!fuse) return;
  fft_dit<S, RR>(x, P2, 32, lane, tw2s, -1);  // slot i held k2 = bitrev(i); now u2 = i
  const int hM = M2 >> 1;
  float2* rw = rb + warp * M2;
  float2* G2 = reinterpret_cast<float2*>(ep.G2) + ((size_t)f * pl.p1 + k1) * RR * M2;
  if constexpr (CL == 1) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      band_horner<RR>(W2s, M2, (s * 32 + lane + mt2) & (P2 - 1), P2, mt2, 1.0f / P2, x[s],
                      [&](int b, float2 v) { rw[(b & 1) * hM + (b >> 1)] = v; });
    __syncthreads();
    eb_stage_a<RR>(bp, rb, M2, M2, G2, threadIdx.x >> 6);
  } else {
    // the same address in the partner CTA's shared memory window
    uint32_t peer;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(smem_u32(rw)), "r"(half ^ 1));
#pragma unroll
    for (int s = 0; s < S; ++s)
      band_horner<RR>(W2s, M2, (s * 32 + lane + mt2) & (P2 - 1), P2, mt2, 1.0f / P2, x[s], [&](int b, float2 v) {
        const int o = (b & 1) * hM + (b >> 1);
        rw[o] = v;
        asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(peer + 8u * o), "f"(v.x), "f"(v.y) : "memory");
      });
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    eb_stage_a<RR>(bp, rb, M2, M2, G2, half * 2 + (threadIdx.x >> 6));
  }
}

// kb_adj_rows for one ePIE position of a p2 = 64 plan with every row's two k2
// slots on two warps (the SPL = 2 idea of kt2_fwd_rows): cluster pair of
// 256-thread CTAs, warp w <-> (row half * 4 + w / 2, slot w % 2). Both warps of a
// row run A-dagger and the D-dagger gather of both slots (cheap) and the first,
// in-thread DIF stage; each then keeps one slot: five shuffle stages on 9 values
// instead of 18, the B2-dagger expansion, the epilogue and stage B of its 32
// k2 groups, five DIT stages, and the last (slot-pairing) DIT stage after one
// exchange through shared memory. Same arithmetic per value as kb_adj_rows
// (bit-identical results); the per-warp dependent chain is about half as long.
template <int RR, int EPI>
__global__ void __launch_bounds__(256, 1)
    kb_adj_rows_split(PftDev<float> pl, EbPar<RR> bp, const float2* __restrict__ Gt, EpiArgs ep) {
  constexpr int P2 = 64, N2 = 512, LP = 6;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M2 = pl.M2, mt2 = pl.mt2;
  float2* rb = reinterpret_cast<float2*>(smem_raw);  // [8][M2]
  float2* W2s = rb + 8 * M2;                         // [M2]
  float2* tw2s = W2s + M2;                           // [32]
  float2* xch = tw2s + 32;                           // [4 rows][2 slots][RR][32]
  const int k1 = blockIdx.x >> 1, half = blockIdx.x & 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rloc = w >> 1, sl = w & 1;
  const int rowb = half * 4 + rloc;  // row of the block
  const long long row = (long long)k1 * 8 + rowb;
  const bool fuse = ep.G2 != nullptr;
  const float st = (float)ep.step;
  for (int i = threadIdx.x; i < M2; i += blockDim.x) W2s[i] = pl.W2t[i];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) tw2s[i] = pl.tw2[i];
  float b1r[RR];
#pragma unroll
  for (int j = 0; j < RR; ++j) b1r[j] = __ldg(pl.Bv1 + rowb * RR + j);
  const int k2 = bitrev(sl * 32 + lane, LP);
  float2 pv[8], ov[8], on[8];
  float2* orow = reinterpret_cast<float2*>(ep.obj) + ep.obj_off + row * ep.obj_ld;
  float2* prow = reinterpret_cast<float2*>(ep.probe) + row * N2;
  const bool vec_o = (reinterpret_cast<uintptr_t>(orow) & 15) == 0;
  const bool vec_p = (reinterpret_cast<uintptr_t>(prow) & 15) == 0;
  eb_load8(prow + k2 * 8, vec_p, pv);
  eb_load8(orow + k2 * 8, vec_o, ov);
  if (EPI == 2 && fuse) {
    const float2* nrow = reinterpret_cast<const float2*>(ep.obj) + ep.obj_off2 + row * ep.obj_ld;
    eb_load8(nrow + k2 * 8, (reinterpret_cast<uintptr_t>(nrow) & 15) == 0, on);
  }
  griddep_wait();  // PDL: Gt is the previous kernel's output; everything above is not
  griddep_launch_dependents();
  const float2* Gblk = Gt + (size_t)k1 * RR * M2;
  float2 Rv[2][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int b = ((s * 32 + lane + mt2) & (P2 - 1)) + P2 * i;
      float2 acc = czero<float2>();
      if (b < M2) {
#pragma unroll
        for (int j = 0; j < RR; ++j) bmacc(acc, b1r[j], Gblk[(size_t)j * M2 + b], j & 1);
      }
      Rv[s][i] = acc;
    }
  __syncthreads();  // tables
  float2 xh[1][RR];
  {
    float2 x[2][RR];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int j = 0; j < RR; ++j) x[s][j] = czero<float2>();
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int b = ((s * 32 + lane + mt2) & (P2 - 1)) + P2 * i;
        if (b < M2) gather_horner<RR>(x[s], W2s[b], static_cast<float>(b - mt2) * (1.0f / P2), Rv[s][i]);
      }
    }
    // first DIF stage (slot pair, h = 32), as fft_dif<2, RR> runs it in-thread
    const float2 wt = twiddle(tw2s, lane, +1);
#pragma unroll
    for (int j = 0; j < RR; ++j) xh[0][j] = sl ? cmul(csub(x[0][j], x[1][j]), wt) : cadd(x[0][j], x[1][j]);
  }
  fft_dif<1, RR>(xh, P2, 32, lane, tw2s, +1);
  {
    float2 z[8], e[8];
    eb_expand8<RR>(bp.b2, xh[0], z);
    if (EPI == 1) {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float2 g = cmulc(pv[l], z[l]);
        ov[l].x -= st * g.x;
        ov[l].y -= st * g.y;
        e[l] = cmul(pv[l], ov[l]);
      }
      eb_store8(orow + k2 * 8, vec_o, ov);
    } else {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float2 g = cmulc(ov[l], z[l]);
        pv[l].x -= st * g.x;
        pv[l].y -= st * g.y;
        e[l] = cmul(pv[l], on[l]);
      }
      eb_store8(prow + k2 * 8, vec_p, pv);
    }
    if (!fuse) return;
    eb_contract8<RR>(bp.b2, e, xh[0]);
  }
  fft_dit<1, RR>(xh, P2, 32, lane, tw2s, -1);  // the cross-lane stages of fft_dit<2, RR>
  // last DIT stage (h = 32) pairs the two slots: exchange through shared memory
  float2* mine = xch + ((rloc * 2 + sl) * RR) * 32 + lane;
  const float2* other = xch + ((rloc * 2 + (sl ^ 1)) * RR) * 32 + lane;
#pragma unroll
  for (int j = 0; j < RR; ++j) mine[j * 32] = xh[0][j];
  named_sync(1 + rloc, 64);
  {
    const float2 wt = twiddle(tw2s, lane, -1);
#pragma unroll
    for (int j = 0; j < RR; ++j) {
      const float2 o = other[j * 32];
      const float2 a = sl ? o : xh[0][j];                     // slot 0 value
      const float2 t = cmul(sl ? xh[0][j] : o, wt);           // slot 1 value x twiddle
      xh[0][j] = sl ? csub(a, t) : cadd(a, t);
    }
  }
  const int hM = M2 >> 1;
  float2* rw = rb + rowb * M2;
  uint32_t peer;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(smem_u32(rw)), "r"(half ^ 1));
  band_horner<RR>(W2s, M2, (sl * 32 + lane + mt2) & (P2 - 1), P2, mt2, 1.0f / P2, xh[0], [&](int b, float2 v) {
    const int o = (b & 1) * hM + (b >> 1);
    rw[o] = v;
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(peer + 8u * o), "f"(v.x), "f"(v.y) : "memory");
  });
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 128)
    eb_stage_a<RR>(bp, rb, M2, M2, reinterpret_cast<float2*>(ep.G2) + (size_t)k1 * RR * M2,
                   half * 2 + (threadIdx.x >> 6));
}

// grid (M2 / NB, batch), 288 threads. One strip of NB band columns of one field:
//   G[f][k1][j1][b] -> p1-point FFTs over k1 (two register passes through shared
//   memory: radix 8 x 8 for p1 = 64, radix 8 x 4 for p1 = 32) -> band rows by
//   Horner over j1 (pft.cpp:150-172, axis-1 half);
//   band != nullptr: store the band strip; dcrop + partial: sum (|band| - dcrop)^2
//   into partial[f * gridDim.x + strip] (evaluator);
//   ADJ: band residual y - dcrop y / |y| (solver.cpp:61-69), D-dagger gather in
//   the same registers, inverse FFTs over u1, -> Gout[f][k1][j1][b] (the fused
//   forward + residual + adjoint cols pass of the ePIE band stage).
// Transform (j1, bb) lives at Gs[(j1 NB + bb) LDF + ...], both passes in place:
//   p1 = 64: natural index i at i + i / 8, spectrum index m + 8 n at 9 m + n
//            (every half-warp phase on distinct banks);
//   p1 = 32: index i = t + 4 k at pad(i), spectrum index m + 8 n at pad(4 m + n),
//            pad(x) = x + x / 16.
constexpr int kEbColsT = 288;
__host__ __device__ constexpr int eb_ldf(int p1) { return p1 == 64 ? 72 : 34; }

// 4-point DFT, sign -1 (SIGN < 0) or +1, natural in / natural out.
template <int SIGN>
__device__ __forceinline__ void dft4(float2 (&a)[4]) {
  const float2 b0 = cadd(a[0], a[2]), b1 = csub(a[0], a[2]), b2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
  const float2 b3 = SIGN < 0 ? make_float2(d.y, -d.x) : make_float2(-d.y, d.x);  // -+ i d
  a[0] = cadd(b0, b2);
  a[2] = csub(b0, b2);
  a[1] = cadd(b1, b3);
  a[3] = csub(b1, b3);
}

template <int RR, int NB, bool ADJ, int P1>
__global__ void __launch_bounds__(kEbColsT, 3)
    kb_cols(PftDev<float> pl, const float2* __restrict__ G, float2* __restrict__ band,
            const float* __restrict__ dcrop, long long dstride, float2* __restrict__ Gout,
            double* __restrict__ partial) {
  constexpr int LDF = eb_ldf(P1), NF = RR * NB, NCH = NB / 2;
  constexpr int LR = P1 * RR * NCH / kEbColsT;  // 16-byte chunks of the strip per thread
  static_assert(P1 * RR * NCH % kEbColsT == 0 && NB % 2 == 0 && (P1 == 64 || P1 == 32), "strip shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  float2* Gs = reinterpret_cast<float2*>(smem_raw);  // [NF][LDF]
  float2* wP = Gs + NF * LDF;                        // W_p1^e, e < p1
  float2* W1s = wP + P1;                             // [M1] row 0 of W1
  float* dcs = reinterpret_cast<float*>(W1s + M1);   // [NB][M1 + 1]
  double* red = reinterpret_cast<double*>(
      smem_raw + (((size_t)(NF * LDF + P1 + M1) * 8 + (size_t)NB * (M1 + 1) * 4 + 7) & ~size_t(7)));
  const int bx = blockIdx.x, f = blockIdx.y, b0 = bx * NB;
  const int tid = threadIdx.x;
  const float2* Gf = G + (size_t)f * P1 * RR * M2;
  // position of natural index i / of spectrum index u = m + 8 n inside a transform
  auto pos_nat = [](int i) { return P1 == 64 ? i + (i >> 3) : i + (i >> 4); };
  auto pos_spec = [](int u) {
    if (P1 == 64) return 9 * (u & 7) + (u >> 3);
    const int x = 4 * (u & 7) + (u >> 3);
    return x + (x >> 4);
  };
  // chunk it of the strip: segment (k1, j1) of NB columns, 16-byte chunk c
  auto chunk_of = [&](int it, int& c, int& k1, int& j1) {
    c = (it >> 3) % NCH;
    const int rest = it / (8 * NCH);
    k1 = (rest % (P1 / 8)) * 8 + (it & 7);
    j1 = rest / (P1 / 8);
  };
  for (int i = tid; i < P1; i += kEbColsT) {
    const float2 w = pl.tw1[i & (P1 / 2 - 1)];
    wP[i] = (i & (P1 / 2)) ? make_float2(-w.x, -w.y) : w;
  }
  for (int i = tid; i < M1; i += kEbColsT) W1s[i] = pl.W1t[i];
  if (dcrop) {
    const float* dc = dcrop + (size_t)f * dstride;
    if constexpr (NB % 4 == 0) {
      for (int i = tid; i < (NB / 4) * M1; i += kEbColsT) {
        const int a = i / (NB / 4), h = i % (NB / 4);
        const float4 d = __ldg(reinterpret_cast<const float4*>(dc + (size_t)a * M2 + b0 + 4 * h));
        dcs[(4 * h + 0) * (M1 + 1) + a] = d.x;
        dcs[(4 * h + 1) * (M1 + 1) + a] = d.y;
        dcs[(4 * h + 2) * (M1 + 1) + a] = d.z;
        dcs[(4 * h + 3) * (M1 + 1) + a] = d.w;
      }
    } else {
      for (int i = tid; i < M1; i += kEbColsT) {
        const float2 d = __ldg(reinterpret_cast<const float2*>(dc + (size_t)i * M2 + b0));
        dcs[i] = d.x;
        dcs[(M1 + 1) + i] = d.y;
      }
    }
  }
  // programmatic dependent launch (single ePIE positions): the tables above do not
  // depend on the previous kernel; G does. The dependents are released only after
  // this kernel's own wait, so their prologues never overlap the kernel before this one.
  griddep_wait();
  griddep_launch_dependents();
  float4 q[LR];
#pragma unroll
  for (int r = 0; r < LR; ++r) {
    int c, k1, j1;
    chunk_of(tid + r * kEbColsT, c, k1, j1);
    q[r] = *reinterpret_cast<const float4*>(Gf + ((size_t)k1 * RR + j1) * M2 + b0 + 2 * c);
  }
#pragma unroll
  for (int r = 0; r < LR; ++r) {
    int c, k1, j1;
    chunk_of(tid + r * kEbColsT, c, k1, j1);
    const int idx = pos_nat(k1);
    Gs[(j1 * NB + 2 * c) * LDF + idx] = make_float2(q[r].x, q[r].y);
    Gs[(j1 * NB + 2 * c + 1) * LDF + idx] = make_float2(q[r].z, q[r].w);
  }
  __syncthreads();
  if constexpr (P1 == 64) {
    // pass 1: y[t][m] = W64^(t m) DFT8_k x[t + 8 k], in place at t + 9 m
    for (int it = tid; it < NF * 8; it += kEbColsT) {
      const int t = it & 7;
      float2* p = Gs + (it >> 3) * LDF + t;
      float2 a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = p[9 * k];
      dft8_fwd(a);
#pragma unroll
      for (int m = 1; m < 8; ++m) a[m] = cmul(a[m], wP[(m * t) & 63]);
#pragma unroll
      for (int m = 0; m < 8; ++m) p[9 * m] = a[m];
    }
    __syncthreads();
    // pass 2: X[m + 8 n] = DFT8_t y[t][m], in place at 9 m + n
    for (int it = tid; it < NF * 8; it += kEbColsT) {
      float2* p = Gs + (it >> 3) * LDF + 9 * (it & 7);
      float2 a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = p[k];
      dft8_fwd(a);
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = a[k];
    }
  } else {
    // pass 1: y[t][m] = W32^(t m) DFT8_k x[t + 4 k] (t < 4), in place at pad(t + 4 m)
    for (int it = tid; it < NF * 4; it += kEbColsT) {
      const int t = it & 3;
      float2* p = Gs + (it >> 2) * LDF;
      float2 a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = p[pos_nat(t + 4 * k)];
      dft8_fwd(a);
#pragma unroll
      for (int m = 1; m < 8; ++m) a[m] = cmul(a[m], wP[(m * t) & 31]);
#pragma unroll
      for (int m = 0; m < 8; ++m) p[pos_nat(t + 4 * m)] = a[m];
    }
    __syncthreads();
    // pass 2: X[m + 8 n] = DFT4_t y[t][m], in place at pad(4 m + n)
    for (int it = tid; it < NF * 8; it += kEbColsT) {
      const int m = it & 7;
      float2* p = Gs + (it >> 3) * LDF;
      float2 a[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = p[pos_nat(4 * m + t)];
      dft4<-1>(a);
#pragma unroll
      for (int n = 0; n < 4; ++n) p[pos_nat(4 * m + n)] = a[n];
    }
  }
  __syncthreads();
  // item (u1, bb): band rows a = u1 + mt1 (mod p1) of column bb by Horner over j1
  double local = 0.0;
  for (int it = tid; it < P1 * NB; it += kEbColsT) {
    const int u1 = it & (P1 - 1), bb = it / P1;
    float2* p = Gs + bb * LDF + pos_spec(u1);
    float2 xs[RR], xa[RR];
#pragma unroll
    for (int j = 0; j < RR; ++j) {
      xs[j] = p[j * NB * LDF];
      xa[j] = czero<float2>();
    }
    for (int a = (u1 + mt1) & (P1 - 1); a < M1; a += P1) {
      const float base = static_cast<float>(a - mt1) * (1.0f / P1);
      float2 acc = xs[RR - 1];
#pragma unroll
      for (int j = RR - 2; j >= 0; --j) acc = cfmar(acc, base, xs[j]);
      const float2 tw = W1s[a];
      float2 y = cmul(tw, acc);
      if (band) band[((size_t)f * M1 + a) * M2 + b0 + bb] = y;
      if (dcrop) {
        const float d = dcs[bb * (M1 + 1) + a];
        // evaluator (no projection): |y| as sqrt(x^2 + y^2), as ke_cols512_eval; the band
        // residual of the ePIE stage keeps hypotf (its quotient y / |y| follows)
        const float mag = ADJ ? hypotf(y.x, y.y) : sqrtf(fmaf(y.x, y.x, y.y * y.y));
        if (partial) {
          const double e = (double)mag - (double)d;
          local += e * e;
        }
        if constexpr (ADJ) {
          if (mag > 0.f) {
            const float ux = y.x / mag, uy = y.y / mag;  // phase_unit = v / |v| (solver.cpp:21-24)
            y.x -= d * ux;
            y.y -= d * uy;
          } else {
            y.x -= d;
          }
        }
      }
      if constexpr (ADJ) gather_horner<RR>(xa, tw, base, y);
    }
    if constexpr (ADJ) {
#pragma unroll
      for (int j = 0; j < RR; ++j) p[j * NB * LDF] = xa[j];
    }
  }
  if (partial) block_sum_store(local, red, partial + (size_t)f * gridDim.x + bx);
  if constexpr (ADJ) {
    __syncthreads();
    if constexpr (P1 == 64) {
      // inverse pass 1: y[t][m] = conj(W64^(t m)) IDFT8_k x[t + 8 k] (index t + 8 k at 9 t + k), in place
      for (int it = tid; it < NF * 8; it += kEbColsT) {
        const int t = it & 7;
        float2* p = Gs + (it >> 3) * LDF + 9 * t;
        float2 a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = p[k];
        dft8<+1>(a);
#pragma unroll
        for (int m = 1; m < 8; ++m) {
          const float2 w = wP[(m * t) & 63];
          a[m] = cmul(a[m], make_float2(w.x, -w.y));
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) p[m] = a[m];
      }
      __syncthreads();
      // inverse pass 2: x[m + 8 n] = IDFT8_t y[t][m] (at 9 t + m), in place: index i at i + i / 8
      for (int it = tid; it < NF * 8; it += kEbColsT) {
        float2* p = Gs + (it >> 3) * LDF + (it & 7);
        float2 a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = p[9 * k];
        dft8<+1>(a);
#pragma unroll
        for (int k = 0; k < 8; ++k) p[9 * k] = a[k];
      }
    } else {
      // inverse pass 1: y[m][t] = conj(W32^(m t)) IDFT4_n X[m + 8 n] (at pad(4 m + n)), in place
      for (int it = tid; it < NF * 8; it += kEbColsT) {
        const int m = it & 7;
        float2* p = Gs + (it >> 3) * LDF;
        float2 a[4];
#pragma unroll
        for (int n = 0; n < 4; ++n) a[n] = p[pos_nat(4 * m + n)];
        dft4<+1>(a);
#pragma unroll
        for (int t = 1; t < 4; ++t) {
          const float2 w = wP[(m * t) & 31];
          a[t] = cmul(a[t], make_float2(w.x, -w.y));
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) p[pos_nat(4 * m + t)] = a[t];
      }
      __syncthreads();
      // inverse pass 2: x[t + 4 k] = IDFT8_m y[m][t] (at pad(4 m + t)), in place: index i at pad(i)
      for (int it = tid; it < NF * 4; it += kEbColsT) {
        const int t = it & 3;
        float2* p = Gs + (it >> 2) * LDF;
        float2 a[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) a[m] = p[pos_nat(4 * m + t)];
        dft8<+1>(a);
#pragma unroll
        for (int k = 0; k < 8; ++k) p[pos_nat(4 * k + t)] = a[k];
      }
    }
    __syncthreads();
    float2* Go = Gout + (size_t)f * P1 * RR * M2;
#pragma unroll
    for (int r = 0; r < LR; ++r) {
      int c, k1, j1;
      chunk_of(tid + r * kEbColsT, c, k1, j1);
      const int idx = pos_nat(k1);
      const float2 v0 = Gs[(j1 * NB + 2 * c) * LDF + idx], v1 = Gs[(j1 * NB + 2 * c + 1) * LDF + idx];
      *reinterpret_cast<float4*>(Go + ((size_t)k1 * RR + j1) * M2 + b0 + 2 * c) = make_float4(v0.x, v0.y, v1.x, v1.y);
    }
  }
}

template <int RR>
EbPar<RR> make_ebpar(const PftDev<float>& pd) {
  EbPar<RR> b;
  for (int l = 0; l <= 4; ++l)
    for (int j = 0; j < RR; ++j) {
      b.b1[l][j] = static_cast<float>(pd.hBv1[l * RR + j]);
      b.b2[l][j] = static_cast<float>(pd.hBv2[l * RR + j]);
    }
  return b;
}

size_t eb_cols_smem(int rr, int nb, int M1, int p1) {
  size_t b = (size_t)(rr * nb * eb_ldf(p1) + p1 + M1) * 8 + (size_t)nb * (M1 + 1) * 4;
  b = (b + 7) & ~size_t(7);
  return b + 16 * sizeof(double);
}

// programmatic dependent launch between the kernels of one ePIE position (PFTG_EB_NO_PDL: off)
bool eb_pdl() {
  static const bool off = std::getenv("PFTG_EB_NO_PDL") != nullptr;
  return !off;
}

template <class K>
void eb_allow_smem(K k, size_t bytes) {
  if (bytes > 48 * 1024) PFTG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

bool eval_band_rows_ok(const PftDev<float>& pd) {
  return pd.q1 == 8 && pd.q2 == 8 && (pd.p2 == 64 || pd.p2 == 32) && pd.r1 == 9 && pd.r2 == 9 && pd.M2 % 2 == 0 &&
         pd.M2 <= pd.n2 && pd.hBv1 && pd.hBv2;
}

bool eval_band_cols_ok(const PftDev<float>& pd) {
  return (pd.p1 == 64 || pd.p1 == 32) && pd.r1 == 9 && pd.M2 % 8 == 0 &&
         eb_cols_smem(9, 8, pd.M1, pd.p1) <= 200 * 1024;
}

void launch_eval_band_rows(const PftDev<float>& pd, const float2* frame, long long ld, long long bstride,
                           const long long* offs, const float2* probe, float2* G, int batch, cudaStream_t st) {
  const auto bp = make_ebpar<9>(pd);
  const size_t smem = (size_t)(8 * pd.n2 + pd.M2 + pd.p2 / 2) * sizeof(float2);
  ProfScope prof(st, K_FWD_ROWS);
  if (pd.p2 == 64) {
    auto k = kb_rows<9, 64>;
    eb_allow_smem(k, smem);
    k<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, frame, ld, bstride, offs, probe, G);
  } else {
    auto k = kb_rows<9, 32>;
    eb_allow_smem(k, smem);
    k<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, frame, ld, bstride, offs, probe, G);
  }
  PFTG_LAUNCH_CHECK();
}

// nb = 8: throughput (evaluator, batches); nb = 4 / 2: one field over 2 x / 4 x more CTAs
// (nb = 2 only with Gout: the residual + adjoint pass of an ePIE position). Gout != nullptr: residual + adjoint (needs dcrop).
void launch_eval_band_cols(const PftDev<float>& pd, int nb, const float2* G, float2* band, const float* dcrop,
                           long long dstride, float2* Gout, double* partial, int batch, cudaStream_t st) {
  const size_t smem = eb_cols_smem(9, nb, pd.M1, pd.p1);
  const dim3 grid(pd.M2 / nb, batch);
  ProfScope prof(st, K_FWD_COLS);
  auto go = [&](auto k) {
    eb_allow_smem(k, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kEbColsT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (batch == 1 && Gout && eb_pdl()) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PFTG_CUDA(cudaLaunchKernelEx(&cfg, k, pd, G, band, dcrop, dstride, Gout, partial));
  };
  if (nb == 2) {  // one ePIE position: the most CTAs, half-filled (4.5 warps of work per CTA)
    if (pd.p1 == 64) go(kb_cols<9, 2, true, 64>);
    else go(kb_cols<9, 2, true, 32>);
  } else if (pd.p1 == 64) {
    if (nb == 8) {
      if (Gout) go(kb_cols<9, 8, true, 64>);
      else go(kb_cols<9, 8, false, 64>);
    } else {
      if (Gout) go(kb_cols<9, 4, true, 64>);
      else go(kb_cols<9, 4, false, 64>);
    }
  } else {
    if (nb == 8) {
      if (Gout) go(kb_cols<9, 8, true, 32>);
      else go(kb_cols<9, 8, false, 32>);
    } else {
      if (Gout) go(kb_cols<9, 4, true, 32>);
      else go(kb_cols<9, 4, false, 32>);
    }
  }
  PFTG_LAUNCH_CHECK();
}

bool eval_band_adj_rows_ok(const PftDev<float>& pd) {
  return eval_band_rows_ok(pd) && pd.M2 <= 2 * pd.p2 && pd.Bv1;
}

void launch_eval_band_adj_rows(const PftDev<float>& pd, int epi, const float2* Gt, const EpiArgs& ep, int batch,
                               cudaStream_t st) {
  const auto bp = make_ebpar<9>(pd);
  const size_t smem = (size_t)(9 * pd.M2 + pd.p2 / 2) * sizeof(float2);
  // single fields (ePIE positions): cluster pairs, 2 x the SMs per row block
  static const bool no_pair = std::getenv("PFTG_EB_NO_PAIR") != nullptr;
  static const bool no_split = std::getenv("PFTG_EB_NO_SPLIT") != nullptr;
  const bool pair = batch == 1 && epi >= 1 && !no_pair;
  auto launch_pair = [&](auto k, int threads, size_t sm) {
    eb_allow_smem(k, sm);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pd.p1, batch);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = eb_pdl() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    PFTG_CUDA(cudaLaunchKernelEx(&cfg, k, pd, bp, Gt, ep));
  };
  if (pair && pd.p2 == 64 && !no_split) {
    // one position of a p2 = 64 plan: the two k2 slots of a row on two warps
    const size_t sm = smem + (size_t)4 * 2 * 9 * 32 * sizeof(float2);
    if (epi == 1) launch_pair(kb_adj_rows_split<9, 1>, 256, sm);
    else launch_pair(kb_adj_rows_split<9, 2>, 256, sm);
    PFTG_LAUNCH_CHECK();
    return;
  }
  auto go = [&](auto k1, auto k2) {
    if (!pair) {
      eb_allow_smem(k1, smem);
      k1<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, Gt, ep);
      return;
    }
    launch_pair(k2, 128, smem);
  };
  if (pd.p2 == 64) {
    if (epi == 0) go(kb_adj_rows<9, 64, 0, 1>, kb_adj_rows<9, 64, 0, 2>);
    else if (epi == 1) go(kb_adj_rows<9, 64, 1, 1>, kb_adj_rows<9, 64, 1, 2>);
    else go(kb_adj_rows<9, 64, 2, 1>, kb_adj_rows<9, 64, 2, 2>);
  } else {
    if (epi == 0) go(kb_adj_rows<9, 32, 0, 1>, kb_adj_rows<9, 32, 0, 2>);
    else if (epi == 1) go(kb_adj_rows<9, 32, 1, 1>, kb_adj_rows<9, 32, 1, 2>);
    else go(kb_adj_rows<9, 32, 2, 1>, kb_adj_rows<9, 32, 2, 2>);
  }
  PFTG_LAUNCH_CHECK();
}

}  // namespace pftg
