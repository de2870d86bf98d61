// Full 2-D FFT passes for the modulus projection, the full-FFT ePIE stage and
// the forward-model/residual evaluator.
//
// Reference: fast_fft2 / fast_ifft2 (/root/reference/proj/core/src/fft.cpp:92-104,175-183,
// FFTW, forward unnormalized, inverse x 1/n), project_modulus
// (solver.cpp:35-42), pie_object_update / epie_probe_update (solver.cpp:44-59),
// objective_value (solver.cpp:89-102).
//
// Layout trick: the spectrum between the forward and inverse transforms is
// never put in natural order. Rows are transformed with DIF (natural ->
// bit-reversed positions) and stored position-for-position (coalesced);
// columns likewise; the modulus projection reads the measured magnitudes
// pre-permuted into the same bit-reversed layout (d_perm, built once per data
// set) or gathers them; the inverse runs DIT (bit-reversed -> natural). So
// project_modulus is three HBM/L2 passes: rows-DIF, cols-DIF+project+DIT,
// rows-DIT (+ fused ePIE update).
#pragma once

#include "common.cuh"

namespace pftg {

// Row source: value(r, c) = [probe[r*n2+c] *] base[off + r*ld + c]
template <class R>
struct RowSrc {
  using C = typename CT<R>::C;
  const C* base;
  long long ld;
  long long bstride;      // per-batch element offset when offs == nullptr
  const long long* offs;  // per-batch element offsets (scan positions)
  const C* probe;
};

enum RowMode {
  ROW_DIF_STORE = 0,   // natural source -> DIF -> store positions into X
  ROW_DIT_NATURAL = 1, // natural source, bitrev gather -> DIT -> natural store (API fft2/ifft2)
  ROW_DIT_PROJ = 2,    // X (bitrev positions) -> DIT -> x 1/n -> epilogue
};

enum RowEpi {
  EPI_STORE = 0,       // out[f][r][c] = proj
  EPI_OBJ = 1,         // object window -= beta conj(P) (P o - proj); optional DIF of new exit -> X2
  EPI_PROBE = 2,       // probe -= gamma conj(o) (P o - proj)
};

struct RowEpiArgs {
  void* out;           // EPI_STORE destination / X2 for EPI_OBJ fused forward
  long long out_bstride;
  void* obj;           // object frame
  long long obj_ld;
  const long long* obj_offs;  // per batch element window offset
  void* probe;
  double step;
  int fuse_next;       // EPI_OBJ: also DIF the new exit wave into out
};

template <int S>
__host__ __device__ inline int fft_lanes(int n) { return n / S < 32 ? n / S : 32; }

// Shared-memory swizzle for bit-reversed gathers over a length-2^lg axis: the
// lanes of a warp read indices bitrev(s*32 + lane) = (bitrev5(lane) << (lg-5)) | c,
// which all fall in one bank in a linear layout. XOR-ing the low 4 bits with
// the bits above (lg-5) spreads them over 16 banks (2 wavefronts per 256 B,
// the minimum for 8-byte elements); a bijection on [0, 2^lg) (Gray-code style:
// each low bit is XOR-ed with a strictly higher one). Identity for lg <= 5.
__device__ __forceinline__ int fft_swz(int i, int lg) {
  const int sh = lg - 5;
  return sh > 0 ? i ^ ((i >> sh) & 15) : i;
}

// grid = (ceil(rows / rows_per_cta), batch); block 256.
// Each lane group (P lanes, S slots) transforms one row of length n2 = P*S.
template <class R, int S, int MODE, int EPI>
__global__ void __launch_bounds__(256) k_fft_rows(int n1, int n2, int lg2, const typename CT<R>::C* __restrict__ tw,
                                                  RowSrc<R> src, typename CT<R>::C* __restrict__ X,
                                                  long long x_bstride, int sign, double scale,
                                                  RowEpiArgs ep) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tws = reinterpret_cast<C*>(smem_raw);
  for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  const int P = n2 / S;  // <= 32
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gpw = 32 / P, lig = lane & (P - 1), giw = lane / P;
  const int f = blockIdx.y;
  const int rows_per_cta = nwarps * gpw;
  const int r = blockIdx.x * rows_per_cta + warp * gpw + giw;
  const bool valid = r < n1;
  C x[S][1];
  const long long soff = src.offs ? src.offs[f] : (long long)f * src.bstride;
  const C* srow = src.base + soff + (long long)r * src.ld;
  const C* prow = src.probe ? src.probe + (long long)r * n2 : nullptr;
  if (MODE == ROW_DIF_STORE) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = s * P + lig;
      C v = czero<C>();
      if (valid) {
        v = srow[c];
        if (prow) v = cmul(prow[c], v);
      }
      x[s][0] = v;
    }
    fft_dif<S, 1>(x, n2, P, lig, tws, sign);
    if (!valid) return;
    C* xr = X + (size_t)f * x_bstride + (size_t)r * n2;
#pragma unroll
    for (int s = 0; s < S; ++s) xr[s * P + lig] = x[s][0];
    return;
  }
  if (MODE == ROW_DIT_NATURAL) {
    // coalesced natural loads into this row's shared-memory buffer, then the
    // bit-reversed gather from shared memory (swizzled: conflict-free)
    C* rb = tws + ((n2 / 2 + 2) & ~1) + (size_t)(warp * gpw + giw) * n2;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = s * P + lig;
      C v = czero<C>();
      if (valid) {
        v = srow[c];
        if (prow) v = cmul(prow[c], v);
      }
      rb[fft_swz(c, lg2)] = v;
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < S; ++s) x[s][0] = rb[fft_swz(bitrev(s * P + lig, lg2), lg2)];
    fft_dit<S, 1>(x, n2, P, lig, tws, sign);
    if (!valid) return;
    C* xr = X + (size_t)f * x_bstride + (size_t)r * n2;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      C v = x[s][0];
      if (scale != 1.0) { v.x *= (R)scale; v.y *= (R)scale; }
      xr[s * P + lig] = v;
    }
    return;
  }
  // ROW_DIT_PROJ: X holds the projected spectrum with columns in bit-reversed
  // positions; output row is natural. The reference scales after the
  // backward transform (fft.cpp:99-102).
  {
    const C* xr = X + (size_t)f * x_bstride + (size_t)r * n2;
#pragma unroll
    for (int s = 0; s < S; ++s) x[s][0] = valid ? xr[s * P + lig] : czero<C>();
    fft_dit<S, 1>(x, n2, P, lig, tws, sign);
    if (EPI == EPI_STORE) {
      if (!valid) return;
      C* out = reinterpret_cast<C*>(ep.out) + (size_t)f * ep.out_bstride + (size_t)r * n2;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        C v = x[s][0];
        v.x *= (R)scale;
        v.y *= (R)scale;
        out[s * P + lig] = v;
      }
      return;
    }
    const long long ooff = ep.obj_offs ? ep.obj_offs[f] : 0;
    C* orow = reinterpret_cast<C*>(ep.obj) + ooff + (long long)r * ep.obj_ld;
    C* pr = reinterpret_cast<C*>(ep.probe) + (long long)r * n2;
    const R st = (R)ep.step;
    if (EPI == EPI_OBJ) {
      // invalid rows stay in the group (no early exit) for the fused shuffles
      C e[S][1];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        e[s][0] = czero<C>();
        if (!valid) continue;
        const int c = s * P + lig;
        C proj = x[s][0];
        proj.x *= (R)scale;
        proj.y *= (R)scale;
        const C pv = pr[c];
        C o = orow[c];
        const C resid = csub(cmul(pv, o), proj);  // probe*z - projected
        const C g = cmulc(pv, resid);
        o.x -= st * g.x;
        o.y -= st * g.y;
        orow[c] = o;
        e[s][0] = cmul(pv, o);
      }
      if (ep.fuse_next) {
        // forward row FFT of the new exit wave probe .* z_new (solver.cpp:256)
        fft_dif<S, 1>(e, n2, P, lig, tws, -1);
        if (!valid) return;
        C* x2 = reinterpret_cast<C*>(ep.out) + (size_t)f * ep.out_bstride + (size_t)r * n2;
#pragma unroll
        for (int s = 0; s < S; ++s) x2[s * P + lig] = e[s][0];
      }
      return;
    }
    if (!valid) return;
    // EPI_PROBE
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int c = s * P + lig;
      C proj = x[s][0];
      proj.x *= (R)scale;
      proj.y *= (R)scale;
      C pv = pr[c];
      const C o = orow[c];
      const C resid = csub(cmul(pv, o), proj);
      const C g = cmulc(o, resid);
      pv.x -= st * g.x;
      pv.y -= st * g.y;
      pr[c] = pv;
    }
  }
}

enum ColMode {
  COL_PROJECT = 0,     // DIF (natural rows) -> modulus projection -> DIT ; in place
  COL_EVAL = 1,        // DIF -> sum (|X| - d)^2 per CTA
  COL_NATURAL = 2,     // bitrev gather -> DIT -> natural (API fft2/ifft2)
  COL_EVAL_NAT = 3,    // rows already natural: bitrev gather -> DIT -> sum (|X| - d)^2, d natural
};

// grid = (n2 / nc, batch), block 256. Strip of nc columns x n1 rows in smem.
// dmode: 0 = d already in the bit-reversed layout (d_perm), 1 = natural d,
// gathered as d[bitrev(row)][bitrev(col)].
template <class R, int S, int MODE>
__global__ void __launch_bounds__(256) k_fft_cols(int n1, int n2, int lg1, int lg2, int nc,
                                                  const typename CT<R>::C* __restrict__ tw,
                                                  typename CT<R>::C* __restrict__ X, long long x_bstride,
                                                  const R* __restrict__ d, long long d_bstride,
                                                  const long long* __restrict__ d_index, int dmode,
                                                  int sign, double* __restrict__ partial) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = nc + 1, ldd = nc + 1;  // padded: conflict-free column reads of the strip / d strip
  C* strip = reinterpret_cast<C*>(smem_raw);
  C* tws = strip + (size_t)n1 * ld;
  R* ds = reinterpret_cast<R*>(tws + n1 / 2 + 1);
  double* red = reinterpret_cast<double*>(smem_raw);  // reused after the strip is dead (COL_EVAL)
  const int f = blockIdx.y, c0 = blockIdx.x * nc;
  C* Xf = X + (size_t)f * x_bstride;
  for (int i = threadIdx.x; i < n1 / 2; i += blockDim.x) tws[i] = tw[i];
  // strip loads: 8 independent loads in flight per thread (nc is a power of two)
  const int tot = n1 * nc, lnc = __ffs(nc) - 1, cm = nc - 1;
  for (int base = threadIdx.x; base < tot; base += 8 * blockDim.x) {
    C v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * blockDim.x;
      if (i < tot) v[u] = Xf[(size_t)(i >> lnc) * n2 + c0 + (i & cm)];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * blockDim.x;
      if (i < tot) strip[(size_t)fft_swz(i >> lnc, lg1) * ld + (i & cm)] = v[u];
    }
  }
  const R* df = nullptr;
  if (MODE != COL_NATURAL) {
    const long long di = d_index ? d_index[f] : f;
    df = d + di * d_bstride;
    if (dmode == 0) {
      for (int base = threadIdx.x; base < tot; base += 8 * blockDim.x) {
        R v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * blockDim.x;
          if (i < tot) v[u] = df[(size_t)(i >> lnc) * n2 + c0 + (i & cm)];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * blockDim.x;
          if (i < tot) ds[(size_t)(i >> lnc) * ldd + (i & cm)] = v[u];
        }
      }
    }
  }
  __syncthreads();
  const int P = n1 / S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gpw = 32 / P, lig = lane & (P - 1), giw = lane / P;
  double local = 0.0;
  for (int base = warp * gpw; base < nc; base += nwarps * gpw) {
    const int cc = base + giw;
    const bool valid = cc < nc;
    C x[S][1];
    if (MODE == COL_NATURAL) {
#pragma unroll
      for (int s = 0; s < S; ++s)
        x[s][0] = valid ? strip[(size_t)fft_swz(bitrev(s * P + lig, lg1), lg1) * ld + cc] : czero<C>();
      fft_dit<S, 1>(x, n1, P, lig, tws, sign);
      if (valid) {
#pragma unroll
        for (int s = 0; s < S; ++s) strip[(size_t)fft_swz(s * P + lig, lg1) * ld + cc] = x[s][0];
      }
      continue;
    }
    if (MODE == COL_EVAL_NAT) {
      // natural-order spectrum column vs the natural measured magnitudes (coalesced d strip)
#pragma unroll
      for (int s = 0; s < S; ++s)
        x[s][0] = valid ? strip[(size_t)fft_swz(bitrev(s * P + lig, lg1), lg1) * ld + cc] : czero<C>();
      fft_dit<S, 1>(x, n1, P, lig, tws, -1);
      if (valid) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const C v = x[s][0];
          const double e = (double)hypot(v.x, v.y) - (double)ds[(size_t)(s * P + lig) * ldd + cc];
          local += e * e;
        }
      }
      continue;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) x[s][0] = valid ? strip[(size_t)fft_swz(s * P + lig, lg1) * ld + cc] : czero<C>();
    fft_dif<S, 1>(x, n1, P, lig, tws, -1);
    // modulus projection: X <- d * X/|X|  (|X| == 0 -> d)   (solver.cpp:39-40)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int rp = s * P + lig;  // bit-reversed row position
      R dv = 0;
      if (valid) {
        if (dmode == 0) dv = ds[(size_t)rp * ldd + cc];
        else dv = df[(size_t)bitrev(rp, lg1) * n2 + bitrev(c0 + cc, lg2)];
      }
      const C v = x[s][0];
      const R mag = hypot(v.x, v.y);
      if (MODE == COL_EVAL) {
        if (valid) {
          const double e = (double)mag - (double)dv;
          local += e * e;
        }
      } else {
        C pv;
        if (mag > R(0)) {
          pv.x = dv * (v.x / mag);
          pv.y = dv * (v.y / mag);
        } else {
          pv.x = dv;
          pv.y = 0;
        }
        x[s][0] = pv;
      }
    }
    if (MODE == COL_EVAL) continue;
    fft_dit<S, 1>(x, n1, P, lig, tws, +1);
    if (valid) {
#pragma unroll
      for (int s = 0; s < S; ++s) strip[(size_t)fft_swz(s * P + lig, lg1) * ld + cc] = x[s][0];
    }
  }
  if (MODE == COL_EVAL || MODE == COL_EVAL_NAT) {
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    __syncthreads();
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += red[w];
      partial[(size_t)f * gridDim.x + blockIdx.x] = s;
    }
    return;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tot; i += blockDim.x)
    Xf[(size_t)(i >> lnc) * n2 + c0 + (i & cm)] = strip[(size_t)fft_swz(i >> lnc, lg1) * ld + (i & cm)];
}

// d_perm[f][rp][cp] = d[f][bitrev(rp)][bitrev(cp)]  (float or double)
template <class R>
__global__ void k_permute_d(const R* __restrict__ d, R* __restrict__ dp, int n1, int n2, int lg1, int lg2,
                            long long count) {
  const long long tot = count * n1 * n2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / ((long long)n1 * n2);
    const int rem = (int)(i % ((long long)n1 * n2));
    const int rp = rem / n2, cp = rem % n2;
    dp[i] = d[f * n1 * n2 + (long long)bitrev(rp, lg1) * n2 + bitrev(cp, lg2)];
  }
}

}  // namespace pftg
