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
    kb_rows(PftDev<float> pl, EbPar<RR> bp, const float2* __restrict__ frame, long long ld,
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
    // exit wave row, coalesced: element c = 32 m + lane
    const float2* zrow = frame + offs[f] + (long long)(k1 * 8 + warp) * ld;
    const float2* prow = probe + (size_t)(k1 * 8 + warp) * N2;
    float2 v[N2 / 32], pv[N2 / 32];
#pragma unroll
    for (int m = 0; m < N2 / 32; ++m) v[m] = __ldg(zrow + 32 * m + lane);
#pragma unroll
    for (int m = 0; m < N2 / 32; ++m) pv[m] = __ldg(prow + 32 * m + lane);
    for (int i = threadIdx.x; i < M2; i += blockDim.x) W2s[i] = pl.W2t[i];
    for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) tw2s[i] = pl.tw2[i];
#pragma unroll
    for (int m = 0; m < N2 / 32; ++m) {
      const int c = 32 * m + lane, g = c >> 3, e = c & 7;
      st[eb_chunk(g, e >> 1) * 2 + (e & 1)] = cmul(pv[m], v[m]);
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
        for (int j = 0; j < RR; ++j) bmacc(acc, b1r[j], __ldg(Gblk + (size_t)j * M2 + b), j & 1);
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

// grid (M2 / NB, batch), 288 threads. One strip of NB band columns of one field:
//   G[f][k1][j1][b] -> 64-point FFTs over k1 (two radix-8 passes in shared
//   memory) -> band rows by Horner over j1 (pft.cpp:150-172, axis-1 half);
//   band != nullptr: store the band strip; dcrop + partial: sum (|band| - dcrop)^2
//   into partial[f * gridDim.x + strip] (evaluator);
//   ADJ: band residual y - dcrop y / |y| (solver.cpp:61-69), D-dagger gather in
//   the same registers, inverse FFTs over u1, -> Gout[f][k1][j1][b] (the fused
//   forward + residual + adjoint cols pass of the ePIE band stage).
// Transform (j1, bb) lives at Gs[(j1 NB + bb) LDF + ...]: natural index i at
// i + i / 8, spectrum index m + 8 n at 9 m + n (both radix-8 passes run in
// place, every half-warp phase on distinct banks).
constexpr int kEbLdF = 72, kEbColsT = 288;

template <int RR, int NB, bool ADJ>
__global__ void __launch_bounds__(kEbColsT, 3)
    kb_cols(PftDev<float> pl, const float2* __restrict__ G, float2* __restrict__ band,
            const float* __restrict__ dcrop, long long dstride, float2* __restrict__ Gout,
            double* __restrict__ partial) {
  constexpr int P1 = 64, LDF = kEbLdF, NF = RR * NB, NCH = NB / 2;
  constexpr int LR = P1 * RR * NCH / kEbColsT;  // 16-byte chunks of the strip per thread
  constexpr int FR = NF * 8 / kEbColsT;         // radix-8 butterflies per thread and pass
  static_assert(P1 * RR * NCH % kEbColsT == 0 && NF * 8 % kEbColsT == 0 && NB % 4 == 0, "strip shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  float2* Gs = reinterpret_cast<float2*>(smem_raw);  // [NF][LDF]
  float2* w64 = Gs + NF * LDF;                       // W64^e, e < 64
  float2* W1s = w64 + 64;                            // [M1] row 0 of W1
  float* dcs = reinterpret_cast<float*>(W1s + M1);   // [NB][M1 + 1]
  double* red = reinterpret_cast<double*>(
      smem_raw + (((size_t)(NF * LDF + 64 + M1) * 8 + (size_t)NB * (M1 + 1) * 4 + 7) & ~size_t(7)));
  const int bx = blockIdx.x, f = blockIdx.y, b0 = bx * NB;
  const int tid = threadIdx.x;
  const float2* Gf = G + (size_t)f * P1 * RR * M2;
  // chunk it of the strip: segment (k1, j1) of NB columns, 16-byte chunk c
  auto chunk_of = [&](int it, int& c, int& k1, int& j1) {
    c = (it >> 3) % NCH;
    const int rest = it / (8 * NCH);
    k1 = (rest & 7) * 8 + (it & 7);
    j1 = rest >> 3;
  };
  float4 q[LR];
#pragma unroll
  for (int r = 0; r < LR; ++r) {
    int c, k1, j1;
    chunk_of(tid + r * kEbColsT, c, k1, j1);
    q[r] = __ldg(reinterpret_cast<const float4*>(Gf + ((size_t)k1 * RR + j1) * M2 + b0 + 2 * c));
  }
  for (int i = tid; i < 64; i += kEbColsT) {
    const float2 w = pl.tw1[i & 31];
    w64[i] = (i & 32) ? make_float2(-w.x, -w.y) : w;
  }
  for (int i = tid; i < M1; i += kEbColsT) W1s[i] = pl.W1t[i];
  if (dcrop) {
    const float* dc = dcrop + (size_t)f * dstride;
    for (int i = tid; i < (NB / 4) * M1; i += kEbColsT) {
      const int a = i / (NB / 4), h = i % (NB / 4);
      const float4 d = __ldg(reinterpret_cast<const float4*>(dc + (size_t)a * M2 + b0 + 4 * h));
      dcs[(4 * h + 0) * (M1 + 1) + a] = d.x;
      dcs[(4 * h + 1) * (M1 + 1) + a] = d.y;
      dcs[(4 * h + 2) * (M1 + 1) + a] = d.z;
      dcs[(4 * h + 3) * (M1 + 1) + a] = d.w;
    }
  }
#pragma unroll
  for (int r = 0; r < LR; ++r) {
    int c, k1, j1;
    chunk_of(tid + r * kEbColsT, c, k1, j1);
    const int idx = k1 + (k1 >> 3);
    Gs[(j1 * NB + 2 * c) * LDF + idx] = make_float2(q[r].x, q[r].y);
    Gs[(j1 * NB + 2 * c + 1) * LDF + idx] = make_float2(q[r].z, q[r].w);
  }
  __syncthreads();
  // pass 1: y[t][m] = W64^(t m) DFT8_k x[t + 8 k], in place at t + 9 m
#pragma unroll
  for (int r = 0; r < FR; ++r) {
    const int it = tid + r * kEbColsT;
    const int t = it & 7;
    float2* p = Gs + (it >> 3) * LDF + t;
    float2 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = p[9 * k];
    dft8_fwd(a);
#pragma unroll
    for (int m = 1; m < 8; ++m) a[m] = cmul(a[m], w64[(m * t) & 63]);
#pragma unroll
    for (int m = 0; m < 8; ++m) p[9 * m] = a[m];
  }
  __syncthreads();
  // pass 2: X[m + 8 n] = DFT8_t y[t][m], in place at 9 m + n
#pragma unroll
  for (int r = 0; r < FR; ++r) {
    const int it = tid + r * kEbColsT;
    float2* p = Gs + (it >> 3) * LDF + 9 * (it & 7);
    float2 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = p[k];
    dft8_fwd(a);
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = a[k];
  }
  __syncthreads();
  // item (u1, bb): band rows a = u1 + mt1 (mod 64) of column bb by Horner over j1
  double local = 0.0;
  for (int it = tid; it < P1 * NB; it += kEbColsT) {
    const int u1 = it & 63, bb = it >> 6;
    float2* p = Gs + bb * LDF + 9 * (u1 & 7) + (u1 >> 3);
    float2 xs[RR], xa[RR];
#pragma unroll
    for (int j = 0; j < RR; ++j) {
      xs[j] = p[j * NB * LDF];
      xa[j] = czero<float2>();
    }
    for (int a = (u1 + mt1) & 63; a < M1; a += P1) {
      const float base = static_cast<float>(a - mt1) * (1.0f / P1);
      float2 acc = xs[RR - 1];
#pragma unroll
      for (int j = RR - 2; j >= 0; --j) acc = cfmar(acc, base, xs[j]);
      const float2 tw = W1s[a];
      float2 y = cmul(tw, acc);
      if (band) band[((size_t)f * M1 + a) * M2 + b0 + bb] = y;
      if (dcrop) {
        const float d = dcs[bb * (M1 + 1) + a];
        const float mag = hypotf(y.x, y.y);
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
    // inverse pass 1: y[t][m] = conj(W64^(t m)) IDFT8_k x[t + 8 k] (index t + 8 k at 9 t + k), in place
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const int it = tid + r * kEbColsT;
      const int t = it & 7;
      float2* p = Gs + (it >> 3) * LDF + 9 * t;
      float2 a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = p[k];
      dft8<+1>(a);
#pragma unroll
      for (int m = 1; m < 8; ++m) {
        const float2 w = w64[(m * t) & 63];
        a[m] = cmul(a[m], make_float2(w.x, -w.y));
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) p[m] = a[m];
    }
    __syncthreads();
    // inverse pass 2: x[m + 8 n] = IDFT8_t y[t][m] (at 9 t + m), in place: index i at i + i / 8
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const int it = tid + r * kEbColsT;
      float2* p = Gs + (it >> 3) * LDF + (it & 7);
      float2 a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = p[9 * k];
      dft8<+1>(a);
#pragma unroll
      for (int k = 0; k < 8; ++k) p[9 * k] = a[k];
    }
    __syncthreads();
    float2* Go = Gout + (size_t)f * P1 * RR * M2;
#pragma unroll
    for (int r = 0; r < LR; ++r) {
      int c, k1, j1;
      chunk_of(tid + r * kEbColsT, c, k1, j1);
      const int idx = k1 + (k1 >> 3);
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

size_t eb_cols_smem(int rr, int nb, int M1) {
  size_t b = (size_t)(rr * nb * kEbLdF + 64 + M1) * 8 + (size_t)nb * (M1 + 1) * 4;
  b = (b + 7) & ~size_t(7);
  return b + 16 * sizeof(double);
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
  return pd.p1 == 64 && pd.r1 == 9 && pd.M2 % 8 == 0 && eb_cols_smem(9, 8, pd.M1) <= 200 * 1024;
}

void launch_eval_band_rows(const PftDev<float>& pd, const float2* frame, long long ld, const long long* offs,
                           const float2* probe, float2* G, int batch, cudaStream_t st) {
  const auto bp = make_ebpar<9>(pd);
  const size_t smem = (size_t)(8 * pd.n2 + pd.M2 + pd.p2 / 2) * sizeof(float2);
  ProfScope prof(st, K_FWD_ROWS);
  if (pd.p2 == 64) {
    auto k = kb_rows<9, 64>;
    eb_allow_smem(k, smem);
    k<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, frame, ld, offs, probe, G);
  } else {
    auto k = kb_rows<9, 32>;
    eb_allow_smem(k, smem);
    k<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, frame, ld, offs, probe, G);
  }
  PFTG_LAUNCH_CHECK();
}

// nb = 8: throughput (evaluator, batches); nb = 4: one ePIE position over 2 x more CTAs,
// one radix-8 butterfly per thread and pass. Gout != nullptr: residual + adjoint (needs dcrop).
void launch_eval_band_cols(const PftDev<float>& pd, int nb, const float2* G, float2* band, const float* dcrop,
                           long long dstride, float2* Gout, double* partial, int batch, cudaStream_t st) {
  const size_t smem = eb_cols_smem(9, nb, pd.M1);
  const dim3 grid(pd.M2 / nb, batch);
  ProfScope prof(st, K_FWD_COLS);
  auto go = [&](auto k) {
    eb_allow_smem(k, smem);
    k<<<grid, kEbColsT, smem, st>>>(pd, G, band, dcrop, dstride, Gout, partial);
  };
  if (nb == 8) {
    if (Gout) go(kb_cols<9, 8, true>);
    else go(kb_cols<9, 8, false>);
  } else {
    if (Gout) go(kb_cols<9, 4, true>);
    else go(kb_cols<9, 4, false>);
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
  const bool pair = batch == 1 && epi >= 1 && !no_pair;
  auto go = [&](auto k1, auto k2) {
    if (!pair) {
      eb_allow_smem(k1, smem);
      k1<<<dim3(pd.p1, batch), 256, smem, st>>>(pd, bp, Gt, ep);
      return;
    }
    eb_allow_smem(k2, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pd.p1, batch);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PFTG_CUDA(cudaLaunchKernelEx(&cfg, k2, pd, bp, Gt, ep));
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
