// Persistent full-FFT ePIE sweep (BASELINE configs[2] / [3] windows, 256^2 and
// 512^2 complex64, sequential visit order): ONE cooperative launch per sweep
// instead of four graph nodes per scan position.
//
// The per-position operator chain is unchanged (solver.cpp:237-262, the same
// arithmetic as ke_rows{256,512}_epie / ke_cols{256,512}_proj, so the
// trajectory is bit-identical):
//   rows   X  = FFT_rows(P .* z_j)                      (first position only)
//   cols   X  = IFFT_cols(proj_d(FFT_cols(X)))          (modulus projection)
//   rows   z_j -= beta conj(P) (P z_j - IFFT_rows(X)/n); X2 = FFT_rows(P z_j)   (blind)
//   cols   X2 = IFFT_cols(proj_d(FFT_cols(X2)))
//   rows   P  -= gamma conj(z_j) (P z_j - IFFT_rows(X2)/n); X = FFT_rows(P z_{j+1})
// Between phases every CTA passes a grid-wide barrier (release add + acquire
// spin on one counter: 1.2 us on 148 CTAs, tools/grid_barrier.cu) -- the graph
// spent ~6 us per kernel node on launch and ramp for ~2 us of work. One CTA per
// SM (cooperative launch: all CTAs co-resident); rows go to 64-thread (512) or
// 32-thread (256) groups, columns to 4 (512) or 8 (256) column blocks per CTA.
#pragma once

#include "eval_fft.cuh"

namespace pftg {

template <int W>
struct ESweep {
  static constexpr int GT = W == 512 ? 64 : 32;  // threads per row transform
  static constexpr int G = 256 / GT;             // row groups per CTA
  static constexpr int NCOL = 256 / GT;          // columns per CTA block
  static constexpr int BUF = W == 512 ? kE512Buf : kE256Buf;
  static constexpr int CS = W == 512 ? kE512Buf + 2 : kE256Buf + 1;
  static constexpr int SBUF = (G * BUF > NCOL * CS) ? G * BUF : NCOL * CS;
};

template <int W, int SIGN, class Sync>
__device__ __forceinline__ void efft(float2 (&a)[8], float2* S, const float2* tws, int l, Sync&& sync) {
  if constexpr (W == 512) fft512<SIGN>(a, S, tws, l, sync);
  else fft256<SIGN>(a, S, tws, l, sync);
}

// One window row r of the rows phases (MODE: E512_FWD / E512_OBJ / E512_PROBE),
// group-private S, lane l of the row's GT threads.
template <int W, int MODE, class Sync>
__device__ __forceinline__ void esweep_row(const float2* tws, float2* S, int l, int r, Sync&& gsync, float2* frame,
                                           long long ld, long long off, float2* probe, float2* X, float2* X2,
                                           float scale, float step, int fuse, long long off_next) {
  constexpr int GT = ESweep<W>::GT;
  float2* orow = frame + off + (long long)r * ld;
  float2* prow = probe + (size_t)r * W;
  float2 a[8];
  if (MODE == E512_FWD) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(prow[l + GT * k], orow[l + GT * k]);
    efft<W, -1>(a, S, tws, l, gsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * W + l + GT * k] = a[k];
    gsync();  // S free for the group's next row
    return;
  }
  const float2* xin = (MODE == E512_OBJ ? X : X2) + (size_t)r * W;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = xin[l + GT * k];
  efft<W, +1>(a, S, tws, l, gsync);
  if (MODE == E512_OBJ) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = l + GT * k;
      float2 proj = a[k];
      proj.x *= scale;
      proj.y *= scale;
      const float2 pv = prow[c];
      float2 o = orow[c];
      const float2 resid = csub(cmul(pv, o), proj);
      const float2 gr = cmulc(pv, resid);
      o.x -= step * gr.x;
      o.y -= step * gr.y;
      orow[c] = o;
      a[k] = cmul(pv, o);
    }
    if (fuse) {
      gsync();
      efft<W, -1>(a, S, tws, l, gsync);
#pragma unroll
      for (int k = 0; k < 8; ++k) X2[(size_t)r * W + l + GT * k] = a[k];
    }
    gsync();
    return;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = l + GT * k;
    float2 proj = a[k];
    proj.x *= scale;
    proj.y *= scale;
    float2 pv = prow[c];
    const float2 o = orow[c];
    const float2 resid = csub(cmul(pv, o), proj);
    const float2 gr = cmulc(o, resid);
    pv.x -= step * gr.x;
    pv.y -= step * gr.y;
    prow[c] = pv;
    a[k] = pv;
  }
  if (fuse) {
    const float2* nrow = frame + off_next + (long long)r * ld;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = cmul(a[k], nrow[l + GT * k]);
    gsync();
    efft<W, -1>(a, S, tws, l, gsync);
#pragma unroll
    for (int k = 0; k < 8; ++k) X[(size_t)r * W + l + GT * k] = a[k];
  }
  gsync();
}

// One block of NCOL columns (the whole CTA): forward column DFT, projection
// against d, inverse column DFT, in place (ke_cols{256,512}_proj).
template <int W>
__device__ __forceinline__ void esweep_cols(const float2* tws, float2* sbuf, int cb, float2* X,
                                            const float* __restrict__ d) {
  constexpr int NCOL = ESweep<W>::NCOL, CS = ESweep<W>::CS, GT = ESweep<W>::GT;
  const int c = threadIdx.x % NCOL, t = threadIdx.x / NCOL;
  const int col = cb * NCOL + c;
  float2 a[8];
  float dv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = X[(size_t)(t + GT * k) * W + col];
    dv[k] = d[(size_t)(t + GT * k) * W + col];
  }
  float2* S = sbuf + c * CS;
  auto bsync = []() { __syncthreads(); };
  efft<W, -1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float mag = hypotf(a[k].x, a[k].y);
    a[k] = mag > 0.f ? make_float2(dv[k] * (a[k].x / mag), dv[k] * (a[k].y / mag)) : make_float2(dv[k], 0.f);
  }
  __syncthreads();
  efft<W, +1>(a, S, tws, t, bsync);
#pragma unroll
  for (int k = 0; k < 8; ++k) X[(size_t)(t + GT * k) * W + col] = a[k];
  __syncthreads();  // S free for the next block
}

__device__ __forceinline__ unsigned esweep_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over the cooperative grid: every CTA adds 1 (release) and
// waits until the counter reaches its next multiple of gridDim.x (acquire).
// The spin traps after ~2^31 polls instead of hanging forever.
__device__ __forceinline__ void esweep_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned long long spins = 0;
    while (esweep_ld_acquire(bar) < target) {
      if (++spins > (1ull << 31)) __trap();
    }
  }
  __syncthreads();
}

// positions [0, npos) in list order; offs[j] = element offset of window j in
// the frame; d: natural-order magnitudes [npos][W][W]; bar: zeroed counter.
template <int W, int BLIND>
__global__ void __launch_bounds__(256, 1) ke_epie_sweep(const float2* __restrict__ tw, float2* frame, long long ld,
                                                        const long long* __restrict__ offs, int npos, float2* probe,
                                                        float2* X, float2* X2, const float* __restrict__ d,
                                                        float scale, float beta, float gamma, unsigned* bar) {
  using E = ESweep<W>;
  __shared__ float2 tws[W / 2];
  __shared__ __align__(16) float2 sbuf[E::SBUF];
  for (int i = threadIdx.x; i < W / 2; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  const int g = threadIdx.x / E::GT, l = threadIdx.x % E::GT;
  float2* Sg = sbuf + g * E::BUF;
  auto gsync = [&]() {
    if constexpr (W == 512) named_sync(1 + g, 64);
    else __syncwarp();
  };
  unsigned target = 0;
  const int rg0 = blockIdx.x * E::G + g, rgs = gridDim.x * E::G;
  auto rows_fwd = [&](long long off) {
    for (int r = rg0; r < W; r += rgs)
      esweep_row<W, E512_FWD>(tws, Sg, l, r, gsync, frame, ld, off, probe, X, X2, 1.f, 0.f, 0, 0);
  };
  auto cols = [&](float2* XX, const float* dj) {
    for (int cb = blockIdx.x; cb < W / E::NCOL; cb += gridDim.x) esweep_cols<W>(tws, sbuf, cb, XX, dj);
  };
  if (npos <= 0) return;
  rows_fwd(offs[0]);
  esweep_barrier(bar, target);
  for (int j = 0; j < npos; ++j) {
    const long long off = offs[j];
    const float* dj = d + (size_t)j * W * W;
    cols(X, dj);
    esweep_barrier(bar, target);
    for (int r = rg0; r < W; r += rgs)
      esweep_row<W, E512_OBJ>(tws, Sg, l, r, gsync, frame, ld, off, probe, X, X2, scale, beta, BLIND, 0);
    esweep_barrier(bar, target);
    if (BLIND) {
      cols(X2, dj);
      esweep_barrier(bar, target);
      const int nxt = j + 1 < npos;
      const long long offn = nxt ? offs[j + 1] : 0;
      for (int r = rg0; r < W; r += rgs)
        esweep_row<W, E512_PROBE>(tws, Sg, l, r, gsync, frame, ld, off, probe, X, X2, scale, gamma, nxt, offn);
      esweep_barrier(bar, target);
    } else if (j + 1 < npos) {
      rows_fwd(offs[j + 1]);
      esweep_barrier(bar, target);
    }
  }
}

}  // namespace pftg
