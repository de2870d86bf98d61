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

// grid (p1, batch), 256 threads: warp w <-> row k1 * 8 + w of the window.
template <int RR, int P2>
__global__ void __launch_bounds__(256, 2)
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
  // stage A on the band rows: thread (m, g) owns columns 2m, 2m + 1 and j1 = g (mod 4)
  const int g = threadIdx.x >> 6;
  float2* Gt = G + ((size_t)f * pl.p1 + k1) * RR * M2;
  for (int m = threadIdx.x & 63; m < hM; m += 64) {
    float2 te[8], to[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      te[l] = stage[l * N2 + m];
      to[l] = stage[l * N2 + hM + m];
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

// grid (M2 / 8, batch), 288 threads. G[f][k1][j1][b] -> sum over the strip of
// (|band| - dcrop)^2 into partial[f * gridDim.x + strip]; band != nullptr also
// stores the band strip (tests).
constexpr int kEbNB = 8, kEbLdF = 72, kEbColsT = 288;

template <int RR>
__global__ void __launch_bounds__(kEbColsT, 3)
    kb_cols(PftDev<float> pl, const float2* __restrict__ G, float2* __restrict__ band,
            const float* __restrict__ dcrop, long long dstride, double* __restrict__ partial) {
  constexpr int P1 = 64, NB = kEbNB, LDF = kEbLdF, NF = RR * NB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M1 = pl.M1, M2 = pl.M2, mt1 = pl.mt1;
  float2* Gs = reinterpret_cast<float2*>(smem_raw);  // [NF][LDF]: transform (j1, bb), point i at i + i / 8
  float2* w64 = Gs + NF * LDF;                       // W64^e, e < 64
  float2* W1s = w64 + 64;                            // [M1] row 0 of W1
  float* dcs = reinterpret_cast<float*>(W1s + M1);   // [NB][M1 + 1]
  double* red = reinterpret_cast<double*>(smem_raw + (((size_t)(NF * LDF + 64 + M1) * 8 + (size_t)NB * (M1 + 1) * 4 + 7) & ~size_t(7)));
  const int bx = blockIdx.x, f = blockIdx.y, b0 = bx * NB;
  const int tid = threadIdx.x;
  const float2* Gf = G + (size_t)f * P1 * RR * M2;
  // strip of G: 64-byte segments (k1, j1), four 16-byte chunks each
  float4 q[P1 * RR * 4 / kEbColsT];
#pragma unroll
  for (int r = 0; r < P1 * RR * 4 / kEbColsT; ++r) {
    const int it = tid + r * kEbColsT;
    const int c = (it >> 3) & 3, rest = it >> 5;
    const int k1 = (rest & 7) * 8 + (it & 7), j1 = rest >> 3;
    q[r] = __ldg(reinterpret_cast<const float4*>(Gf + ((size_t)k1 * RR + j1) * M2 + b0 + 2 * c));
  }
  for (int i = tid; i < 64; i += kEbColsT) {
    const float2 w = pl.tw1[i & 31];
    w64[i] = (i & 32) ? make_float2(-w.x, -w.y) : w;
  }
  for (int i = tid; i < M1; i += kEbColsT) W1s[i] = pl.W1t[i];
  if (dcrop) {
    const float* dc = dcrop + (size_t)f * dstride;
    for (int i = tid; i < 2 * M1; i += kEbColsT) {
      const int a = i >> 1, h = i & 1;
      const float4 d = __ldg(reinterpret_cast<const float4*>(dc + (size_t)a * M2 + b0 + 4 * h));
      dcs[(4 * h + 0) * (M1 + 1) + a] = d.x;
      dcs[(4 * h + 1) * (M1 + 1) + a] = d.y;
      dcs[(4 * h + 2) * (M1 + 1) + a] = d.z;
      dcs[(4 * h + 3) * (M1 + 1) + a] = d.w;
    }
  }
#pragma unroll
  for (int r = 0; r < P1 * RR * 4 / kEbColsT; ++r) {
    const int it = tid + r * kEbColsT;
    const int c = (it >> 3) & 3, rest = it >> 5;
    const int k1 = (rest & 7) * 8 + (it & 7), j1 = rest >> 3;
    const int idx = k1 + (k1 >> 3);
    Gs[(j1 * NB + 2 * c) * LDF + idx] = make_float2(q[r].x, q[r].y);
    Gs[(j1 * NB + 2 * c + 1) * LDF + idx] = make_float2(q[r].z, q[r].w);
  }
  __syncthreads();
  // pass 1: y[t][m] = W64^(t m) DFT8_k x[t + 8 k], in place at t + 8 m
#pragma unroll
  for (int r = 0; r < NF * 8 / kEbColsT; ++r) {
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
  // pass 2: X[m + 8 n] = DFT8_t y[t][m], left in place at 8 m + n
#pragma unroll
  for (int r = 0; r < NF * 8 / kEbColsT; ++r) {
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
  // band rows a = u1 + mt1 (mod 64) of column bb by Horner over j1, residual
  double local = 0.0;
  for (int it = tid; it < P1 * NB; it += kEbColsT) {
    const int u1 = it & 63, bb = it >> 6;
    const float2* p = Gs + bb * LDF + 9 * (u1 & 7) + (u1 >> 3);
    float2 xs[RR];
#pragma unroll
    for (int j = 0; j < RR; ++j) xs[j] = p[j * NB * LDF];
    for (int a = (u1 + mt1) & 63; a < M1; a += P1) {
      const float base = static_cast<float>(a - mt1) * (1.0f / P1);
      float2 acc = xs[RR - 1];
#pragma unroll
      for (int j = RR - 2; j >= 0; --j) acc = cfmar(acc, base, xs[j]);
      const float2 y = cmul(W1s[a], acc);
      if (band) band[((size_t)f * M1 + a) * M2 + b0 + bb] = y;
      if (dcrop) {
        const double e = (double)hypotf(y.x, y.y) - (double)dcs[bb * (M1 + 1) + a];
        local += e * e;
      }
    }
  }
  if (partial) block_sum_store(local, red, partial + (size_t)f * gridDim.x + bx);
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

size_t eb_cols_smem(int rr, int M1) {
  size_t b = (size_t)(rr * kEbNB * kEbLdF + 64 + M1) * 8 + (size_t)kEbNB * (M1 + 1) * 4;
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
  return pd.p1 == 64 && pd.r1 == 9 && pd.M2 % kEbNB == 0 && eb_cols_smem(9, pd.M1) <= 200 * 1024;
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

void launch_eval_band_cols(const PftDev<float>& pd, const float2* G, float2* band, const float* dcrop,
                           long long dstride, double* partial, int batch, cudaStream_t st) {
  const size_t smem = eb_cols_smem(9, pd.M1);
  auto k = kb_cols<9>;
  eb_allow_smem(k, smem);
  ProfScope prof(st, K_FWD_COLS);
  k<<<dim3(pd.M2 / kEbNB, batch), kEbColsT, smem, st>>>(pd, G, band, dcrop, dstride, partial);
  PFTG_LAUNCH_CHECK();
}

}  // namespace pftg
