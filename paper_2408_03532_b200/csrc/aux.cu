// The steps either side of the hot path, on the GPU:
//
//  F1  measurement simulator   simulate          (simulate.cpp:48-65)
//                              add_poisson_noise (simulate.cpp:67-79)
//                              build_cropped     (simulate.cpp:81-89) = crop_centered per position
//  F2  per-sweep metrics       relative_error, relative_error_aligned, psnr,
//                              ssim, dynamic_range (metrics.cpp:60-143) and the
//                              fill_metrics bundle (solver.cpp:141-160)
//
// simulate: d_j = |FFT2(probe .* window_j)| -- the window is read in place from
// the frame (offset + stride, no window_slice copy), the probe multiply is
// fused into the row pass, |.| into a final elementwise pass.
//
// add_poisson_noise: the reference draws from libstdc++'s
// std::poisson_distribution over one mt19937_64 stream, which has no parallel
// counterpart; here every element is an independent counter-based draw:
//   uniforms  Philox-4x32-10 (Salmon et al., SC'11), key = seed (64 bit),
//             counter = (element index lo, hi, draw block, 0); one block gives
//             two 53-bit doubles u = (hi32 << 21 ^ lo32 >> 11) * 2^-53;
//   Poisson   lambda < 10: inversion by sequential search (one uniform);
//             lambda >= 10: Hoermann's PTRS transformed rejection with squeeze
//             (Hoermann 1993), the sampler numpy uses for large lambda.
// The law is the reference's (d <- sqrt(Poisson(scale d^2) / scale)); the
// stream is not (statistical parity, tested by moments and by comparison with
// the reference's own noise on the same input).
//
// Metrics: FP64 accumulation, per-CTA partials reduced in a fixed order (so
// results are deterministic run to run); SSIM uses the reference's 11-tap
// Gaussian (sigma 1.5), valid region, K1 = 0.01, K2 = 0.03.
#include <cuda_runtime.h>

#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pftg.h"
#include "internal.hpp"

namespace pftg {
namespace {

template <class R>
using Cx = typename CT<R>::C;

// ------------------------------------------------------------------ F1
template <class R>
__global__ void k_abs(const Cx<R>* __restrict__ X, R* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Cx<R> v = X[i];
    d[i] = hypot(v.x, v.y);  // std::abs(complex) (field.cpp:76)
  }
}

struct Philox {
  static __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    const unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const unsigned lo0 = M0 * c.x, hi0 = __umulhi(M0, c.x);
    const unsigned lo1 = M1 * c.z, hi1 = __umulhi(M1, c.z);
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  static __device__ __forceinline__ uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// Stream of uniforms in [0, 1) for one element: blocks of two doubles.
struct Uniforms {
  uint2 key;
  unsigned long long idx;
  unsigned blk = 0;
  double buf[2];
  int left = 0;
  __device__ double next() {
    if (left == 0) {
      const uint4 r = Philox::gen(make_uint4((unsigned)idx, (unsigned)(idx >> 32), blk++, 0u), key);
      buf[0] = (double)(((unsigned long long)r.x << 21) ^ (r.y >> 11)) * 0x1.0p-53;
      buf[1] = (double)(((unsigned long long)r.z << 21) ^ (r.w >> 11)) * 0x1.0p-53;
      left = 2;
    }
    return buf[2 - left--];
  }
};

__device__ long long poisson_draw(double lam, Uniforms& u) {
  if (!(lam > 0.0)) return 0;
  if (lam < 10.0) {
    // inversion: smallest k with F(k) >= u
    const double uu = u.next();
    double p = exp(-lam), F = p;
    long long k = 0;
    while (uu > F && k < 1000) {
      ++k;
      p *= lam / (double)k;
      F += p;
    }
    return k;
  }
  // PTRS (Hoermann 1993)
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double U = u.next() - 0.5, V = u.next();
    const double us = 0.5 - fabs(U);
    const long long k = (long long)floor((2.0 * a / us + b) * U + lam + 0.43);
    if (us >= 0.07 && V <= vr) return k;
    if (k < 0 || (us < 0.013 && V > us)) continue;
    if (log(V) + log(invalpha) - log(a / (us * us) + b) <= -lam + (double)k * loglam - lgamma((double)k + 1.0))
      return k;
  }
}

template <class R>
__global__ void k_poisson(R* __restrict__ d, long long n, double scale, uint2 key) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = (double)d[i];
    Uniforms u{key, (unsigned long long)i};
    const long long k = poisson_draw(scale * v * v, u);
    d[i] = (R)sqrt((double)k / scale);  // simulate.cpp:74-75
  }
}

int grid_of(long long n) {
  const long long g = (n + 255) / 256;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 16));
}

void check_window(long long r0, long long c0, std::size_t wr, std::size_t wc, std::size_t fr, std::size_t fc) {
  if (r0 < 0 || c0 < 0 || r0 + (long long)wr > (long long)fr || c0 + (long long)wc > (long long)fc)
    throw std::out_of_range("scan: window (" + std::to_string(r0) + ", " + std::to_string(c0) + ") outside the frame");
}

template <class R>
void simulate_dev(const void* frame, std::size_t fr, std::size_t fc, const void* probe, std::size_t wr,
                  std::size_t wc, const int64_t* offsets, std::size_t npos, void* d, cudaStream_t st) {
  check_fft_len(wr);
  check_fft_len(wc);
  const long long n = (long long)wr * wc;
  std::vector<long long> offs(npos);
  for (std::size_t j = 0; j < npos; ++j) {
    check_window(offsets[2 * j], offsets[2 * j + 1], wr, wc, fr, fc);
    offs[j] = offsets[2 * j] * (long long)fc + offsets[2 * j + 1];
  }
  Scratch doffs(sizeof(long long) * npos, st);
  PFTG_CUDA(cudaMemcpyAsync(doffs.p, offs.data(), sizeof(long long) * npos, cudaMemcpyHostToDevice, st));
  const std::size_t chunk = std::max<std::size_t>(1, std::min<std::size_t>(npos, (128u << 20) / (sizeof(Cx<R>) * n)));
  Scratch X(sizeof(Cx<R>) * n * chunk, st);
  for (std::size_t c0 = 0; c0 < npos; c0 += chunk) {
    const int nb = (int)std::min(chunk, npos - c0);
    RowSrc<R> src{static_cast<const Cx<R>*>(frame), (long long)fc, 0, doffs.as<long long>() + c0,
                  static_cast<const Cx<R>*>(probe)};
    RowEpiArgs ep{};
    launch_fft_rows<R>(ROW_DIT_NATURAL, EPI_STORE, (int)wr, (int)wc, src, X.as<Cx<R>>(), n, -1, 1.0, ep, nb, st);
    launch_fft_cols<R>(COL_NATURAL, (int)wr, (int)wc, X.as<Cx<R>>(), n, nullptr, 0, nullptr, 0, -1, nullptr, nb, st);
    k_abs<R><<<grid_of(n * nb), 256, 0, st>>>(X.as<Cx<R>>(), static_cast<R*>(d) + c0 * n, n * nb);
    PFTG_LAUNCH_CHECK();
  }
  // offsets scratch is released stream-ordered; the host vector must outlive the copy
  PFTG_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------------ F2
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kWin = 11;         // SSIM window (metrics.cpp:19)

__constant__ double c_gauss[kWin];

// Quantities accumulated in one pass over the region (all FP64).
enum { S_XR_RE = 0, S_XR_IM, S_NUM, S_DEN, S_MAGNUM, S_MAGDEN, S_PHNUM, S_PHDEN, S_NQ };
enum { M_MAGMIN = 0, M_MAGMAX, M_PHMIN, M_PHMAX, M_NQ };

__device__ __forceinline__ double phase_of(double re, double im) {
  return (re == 0.0 && im == 0.0) ? 0.0 : atan2(im, re);  // field.cpp:80-87
}

template <class C>
__device__ __forceinline__ void load_pair(const C* x, const C* r, long long ix, long long ir, double& xr, double& xi,
                                          double& rr, double& ri) {
  const C a = x[ix], b = r[ir];
  xr = (double)a.x;
  xi = (double)a.y;
  rr = (double)b.x;
  ri = (double)b.y;
}

// Pass 1 partial sums per CTA: sum x conj(ref), |x-ref|^2, |ref|^2, magnitude
// and phase error sums, truth magnitude / phase extrema.
template <class C>
__global__ void k_metrics_pass1(const C* __restrict__ x, long long ldx, const C* __restrict__ r, long long ldr,
                                int rows, int cols, double* __restrict__ part, double* __restrict__ ext) {
  double s[S_NQ] = {};
  double mn[2] = {INFINITY, INFINITY}, mx[2] = {-INFINITY, -INFINITY};
  const long long n = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(i / cols), b = (int)(i % cols);
    double xr, xi, rr, ri;
    load_pair(x, r, a * ldx + b, a * ldr + b, xr, xi, rr, ri);
    s[S_XR_RE] += xr * rr + xi * ri;  // x conj(ref)
    s[S_XR_IM] += xi * rr - xr * ri;
    const double dr = xr - rr, di = xi - ri;
    s[S_NUM] += dr * dr + di * di;
    s[S_DEN] += rr * rr + ri * ri;
    const double mxv = hypot(xr, xi), mrv = hypot(rr, ri);
    s[S_MAGNUM] += (mxv - mrv) * (mxv - mrv);
    s[S_MAGDEN] += mrv * mrv;
    const double px = phase_of(xr, xi), pr = phase_of(rr, ri);
    s[S_PHNUM] += (px - pr) * (px - pr);
    s[S_PHDEN] += pr * pr;
    mn[0] = fmin(mn[0], mrv);
    mx[0] = fmax(mx[0], mrv);
    mn[1] = fmin(mn[1], pr);
    mx[1] = fmax(mx[1], pr);
  }
  __shared__ double sh[kRedThreads];
  for (int q = 0; q < S_NQ + M_NQ; ++q) {
    double v = q < S_NQ ? s[q] : (q == S_NQ ? mn[0] : q == S_NQ + 1 ? mx[0] : q == S_NQ + 2 ? mn[1] : mx[1]);
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
      if ((int)threadIdx.x < h) {
        const double o = sh[threadIdx.x + h];
        if (q < S_NQ) sh[threadIdx.x] += o;
        else if (q == S_NQ || q == S_NQ + 2) sh[threadIdx.x] = fmin(sh[threadIdx.x], o);
        else sh[threadIdx.x] = fmax(sh[threadIdx.x], o);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (q < S_NQ) part[(size_t)q * gridDim.x + blockIdx.x] = sh[0];
      else ext[(size_t)(q - S_NQ) * gridDim.x + blockIdx.x] = sh[0];
    }
    __syncthreads();
  }
}

// Pass 2: sum |c x - ref|^2 with the aligning unit phase c (metrics.cpp:83-96).
template <class C>
__global__ void k_metrics_aligned(const C* __restrict__ x, long long ldx, const C* __restrict__ r, long long ldr,
                                  int rows, int cols, double cre, double cim, double* __restrict__ part) {
  double acc = 0.0;
  const long long n = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(i / cols), b = (int)(i % cols);
    double xr, xi, rr, ri;
    load_pair(x, r, a * ldx + b, a * ldr + b, xr, xi, rr, ri);
    const double yr = cre * xr - cim * xi - rr, yi = cre * xi + cim * xr - ri;
    acc += yr * yr + yi * yi;
  }
  __shared__ double sh[kRedThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) sh[threadIdx.x] += sh[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// SSIM over the valid region (metrics.cpp:112-136) of QTY(x) vs QTY(ref),
// QTY 0 = magnitude, 1 = phase. One 16 x 16 tile of outputs per CTA; per-CTA
// partial sum of the SSIM map.
constexpr int kTile = 16;
template <class C, int QTY>
__global__ void k_ssim(const C* __restrict__ x, long long ldx, const C* __restrict__ r, long long ldr, int rows,
                       int cols, double c1, double c2, double* __restrict__ part) {
  constexpr int IN = kTile + kWin - 1;  // 26
  __shared__ double sx[IN][IN], sr[IN][IN];
  __shared__ double hs[5][IN][kTile];
  const int orow = rows - kWin + 1, ocol = cols - kWin + 1;
  const int tr0 = blockIdx.y * kTile, tc0 = blockIdx.x * kTile;
  for (int i = threadIdx.x; i < IN * IN; i += blockDim.x) {
    const int a = i / IN, b = i % IN;
    const int ga = tr0 + a, gb = tc0 + b;
    double vx = 0.0, vr = 0.0;
    if (ga < rows && gb < cols) {
      double xr, xi, rr, ri;
      load_pair(x, r, ga * ldx + gb, ga * ldr + gb, xr, xi, rr, ri);
      vx = QTY == 0 ? hypot(xr, xi) : phase_of(xr, xi);
      vr = QTY == 0 ? hypot(rr, ri) : phase_of(rr, ri);
    }
    sx[a][b] = vx;
    sr[a][b] = vr;
  }
  __syncthreads();
  // horizontal pass (filter_valid, metrics.cpp:33-40): IN rows x kTile cols, 5 fields
  for (int i = threadIdx.x; i < IN * kTile; i += blockDim.x) {
    const int a = i / kTile, b = i % kTile;
    double f0 = 0, f1 = 0, f2 = 0, f3 = 0, f4 = 0;
#pragma unroll
    for (int t = 0; t < kWin; ++t) {
      const double g = c_gauss[t], vx = sx[a][b + t], vr = sr[a][b + t];
      f0 += g * vx;
      f1 += g * vr;
      f2 += g * (vx * vx);
      f3 += g * (vr * vr);
      f4 += g * (vx * vr);
    }
    hs[0][a][b] = f0;
    hs[1][a][b] = f1;
    hs[2][a][b] = f2;
    hs[3][a][b] = f3;
    hs[4][a][b] = f4;
  }
  __syncthreads();
  double acc = 0.0;
  {
    const int a = threadIdx.x / kTile, b = threadIdx.x % kTile;
    if (tr0 + a < orow && tc0 + b < ocol) {
      double m[5] = {};
#pragma unroll
      for (int t = 0; t < kWin; ++t) {
        const double g = c_gauss[t];
#pragma unroll
        for (int q = 0; q < 5; ++q) m[q] += g * hs[q][a + t][b];
      }
      const double mx = m[0], my = m[1];
      const double vx = m[2] - mx * mx, vy = m[3] - my * my, cxy = m[4] - mx * my;
      acc = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
    }
  }
  __shared__ double red[kTile * kTile];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

void upload_gauss() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && done[dev]) return;
  double g[kWin], sum = 0.0;  // ssim_kernel (metrics.cpp:18-29)
  for (int i = 0; i < kWin; ++i) {
    const double dd = i - (kWin - 1) / 2.0;
    g[i] = std::exp(-dd * dd / (2 * 1.5 * 1.5));
    sum += g[i];
  }
  for (auto& v : g) v /= sum;
  PFTG_CUDA(cudaMemcpyToSymbol(c_gauss, g, sizeof g));
  if (dev < 64) done[dev] = true;
}

double ratio_sqrt(double num, double den) {  // metrics.cpp:69-70
  if (den == 0.0) return num == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
  return std::sqrt(num / den);
}

template <class R>
void fill_metrics_dev(const void* xv, std::size_t ldx, const void* rv, std::size_t ldr, std::size_t rows,
                      std::size_t cols, double* out, cudaStream_t st) {
  if (rows == 0 || cols == 0) throw std::invalid_argument("fill_metrics: empty region");
  if (ldx < cols || ldr < cols) throw std::invalid_argument("fill_metrics: leading dimension < cols");
  if (rows < (std::size_t)kWin || cols < (std::size_t)kWin)
    throw std::invalid_argument("ssim: images must be at least 11x11");
  using C = Cx<R>;
  const C* x = static_cast<const C*>(xv);
  const C* r = static_cast<const C*>(rv);
  upload_gauss();
  const int tx = (int)((cols - kWin + 1 + kTile - 1) / kTile), ty = (int)((rows - kWin + 1 + kTile - 1) / kTile);
  Scratch part(sizeof(double) * (S_NQ + M_NQ + 1) * kRedBlocks, st), sp(sizeof(double) * 2 * tx * ty, st);
  double* p1 = part.as<double>();
  double* ext = p1 + S_NQ * kRedBlocks;
  double* p2 = ext + M_NQ * kRedBlocks;
  k_metrics_pass1<C><<<kRedBlocks, kRedThreads, 0, st>>>(x, (long long)ldx, r, (long long)ldr, (int)rows, (int)cols,
                                                        p1, ext);
  PFTG_LAUNCH_CHECK();
  std::vector<double> h((S_NQ + M_NQ) * kRedBlocks);
  PFTG_CUDA(cudaMemcpyAsync(h.data(), p1, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
  PFTG_CUDA(cudaStreamSynchronize(st));
  double s[S_NQ] = {};
  for (int q = 0; q < S_NQ; ++q)
    for (int b = 0; b < kRedBlocks; ++b) s[q] += h[(size_t)q * kRedBlocks + b];
  double e[M_NQ] = {INFINITY, -INFINITY, INFINITY, -INFINITY};
  for (int b = 0; b < kRedBlocks; ++b) {
    const double* hx = h.data() + S_NQ * kRedBlocks;
    e[0] = std::fmin(e[0], hx[0 * kRedBlocks + b]);
    e[1] = std::fmax(e[1], hx[1 * kRedBlocks + b]);
    e[2] = std::fmin(e[2], hx[2 * kRedBlocks + b]);
    e[3] = std::fmax(e[3], hx[3 * kRedBlocks + b]);
  }
  // aligning phase c = conj(s) / |s| (metrics.cpp:86-88)
  const double mag = std::hypot(s[S_XR_RE], s[S_XR_IM]);
  const double cre = mag > 0.0 ? s[S_XR_RE] / mag : 1.0, cim = mag > 0.0 ? -s[S_XR_IM] / mag : 0.0;
  k_metrics_aligned<C><<<kRedBlocks, kRedThreads, 0, st>>>(x, (long long)ldx, r, (long long)ldr, (int)rows,
                                                          (int)cols, cre, cim, p2);
  PFTG_LAUNCH_CHECK();
  // dynamic ranges of the truth (metrics.cpp:138-141)
  const double rng_mag = (e[1] - e[0]) > 0.0 ? e[1] - e[0] : 1.0;
  const double rng_ph = (e[3] - e[2]) > 0.0 ? e[3] - e[2] : 1.0;
  double* ssim_part = sp.as<double>();
  const double cm1 = (0.01 * rng_mag) * (0.01 * rng_mag), cm2 = (0.03 * rng_mag) * (0.03 * rng_mag);
  const double cp1 = (0.01 * rng_ph) * (0.01 * rng_ph), cp2 = (0.03 * rng_ph) * (0.03 * rng_ph);
  k_ssim<C, 0><<<dim3(tx, ty), kTile * kTile, 0, st>>>(x, (long long)ldx, r, (long long)ldr, (int)rows, (int)cols, cm1,
                                                      cm2, ssim_part);
  PFTG_LAUNCH_CHECK();
  k_ssim<C, 1><<<dim3(tx, ty), kTile * kTile, 0, st>>>(x, (long long)ldx, r, (long long)ldr, (int)rows, (int)cols, cp1,
                                                      cp2, ssim_part + tx * ty);
  PFTG_LAUNCH_CHECK();
  std::vector<double> h2(kRedBlocks), hs(2 * tx * ty);
  PFTG_CUDA(cudaMemcpyAsync(h2.data(), p2, sizeof(double) * kRedBlocks, cudaMemcpyDeviceToHost, st));
  PFTG_CUDA(cudaMemcpyAsync(hs.data(), ssim_part, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, st));
  PFTG_CUDA(cudaStreamSynchronize(st));
  double anum = 0.0, sm = 0.0, sph = 0.0;
  for (double v : h2) anum += v;
  for (int i = 0; i < tx * ty; ++i) {
    sm += hs[i];
    sph += hs[tx * ty + i];
  }
  const double n = (double)rows * (double)cols, nv = (double)(rows - kWin + 1) * (double)(cols - kWin + 1);
  auto psnr = [&](double sq, double range) {  // metrics.cpp:98-110
    const double mse = sq / n;
    if (mse == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(range * range / mse);
  };
  out[0] = ratio_sqrt(s[S_NUM], s[S_DEN]);        // rel_err
  out[1] = ratio_sqrt(anum, s[S_DEN]);            // rel_err_aligned
  out[2] = ratio_sqrt(s[S_MAGNUM], s[S_MAGDEN]);  // rel_err_mag
  out[3] = ratio_sqrt(s[S_PHNUM], s[S_PHDEN]);    // rel_err_phase
  out[4] = sm / nv;                               // ssim_mag
  out[5] = sph / nv;                              // ssim_phase
  out[6] = psnr(s[S_MAGNUM], rng_mag);            // psnr_mag
  out[7] = psnr(s[S_PHNUM], rng_ph);              // psnr_phase
}

}  // namespace
}  // namespace pftg

using namespace pftg;

namespace {
template <class F>
int guarded_aux(F&& f) {
  try {
    f();
    return PFTG_OK;
  } catch (const cuda_error& e) {
    set_error(e.what());
    return PFTG_ECUDA;
  } catch (const std::invalid_argument& e) {
    set_error(std::string("invalid_argument: ") + e.what());
    return PFTG_EINVAL;
  } catch (const std::out_of_range& e) {
    set_error(std::string("out_of_range: ") + e.what());
    return PFTG_ERANGE;
  } catch (const std::logic_error& e) {
    set_error(std::string("logic_error: ") + e.what());
    return PFTG_ELOGIC;
  } catch (const std::exception& e) {
    set_error(std::string("runtime_error: ") + e.what());
    return PFTG_ERUNTIME;
  }
}
void dtype_ok(int dtype) {
  if (dtype != PFTG_C64 && dtype != PFTG_C128) throw std::invalid_argument("pftg: dtype must be PFTG_C64 or PFTG_C128");
}
}  // namespace

extern "C" {

int pftg_simulate_dev(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr, size_t wc,
                      const int64_t* offsets, size_t npos, void* d, void* stream) {
  return guarded_aux([&] {
    dtype_ok(dtype);
    if (npos == 0) return;
    ensure_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == PFTG_C64) simulate_dev<float>(frame, fr, fc, probe, wr, wc, offsets, npos, d, st);
    else simulate_dev<double>(frame, fr, fc, probe, wr, wc, offsets, npos, d, st);
  });
}

int pftg_add_poisson_noise_dev(int dtype, void* d, size_t n, double scale, uint64_t seed, void* stream) {
  return guarded_aux([&] {
    dtype_ok(dtype);
    if (!(scale > 0.0)) throw std::invalid_argument("add_poisson_noise: need scale > 0");  // simulate.cpp:68
    if (n == 0) return;
    ensure_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
    if (dtype == PFTG_C64) k_poisson<float><<<grid_of(n), 256, 0, st>>>(static_cast<float*>(d), (long long)n, scale, key);
    else k_poisson<double><<<grid_of(n), 256, 0, st>>>(static_cast<double*>(d), (long long)n, scale, key);
    PFTG_LAUNCH_CHECK();
  });
}

int pftg_fill_metrics_dev(int dtype, const void* x, size_t ld_x, const void* ref, size_t ld_ref, size_t rows,
                          size_t cols, double* out, void* stream) {
  return guarded_aux([&] {
    dtype_ok(dtype);
    if (!out) throw std::invalid_argument("fill_metrics: null output");
    ensure_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == PFTG_C64) fill_metrics_dev<float>(x, ld_x, ref, ld_ref, rows, cols, out, st);
    else fill_metrics_dev<double>(x, ld_x, ref, ld_ref, rows, cols, out, st);
  });
}

}  // extern "C"
