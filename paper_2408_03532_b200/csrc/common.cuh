// Shared device helpers for the B200 PFT / ePIE kernels (sm_100a).
//
// Complex values are float2 (complex64) or double2 (complex128), interleaved
// (re, im) exactly like the reference ComplexField storage
// (/root/reference/proj/core/include/ptycho/field.hpp:37-65).
//
// Short FFTs run in registers across a "lane group": a transform of length
// P*S is held by P lanes (P = min(len, 32)) with S slots each; element index
// i = slot*P + lane. Stages whose butterfly distance h >= P pair two slots of
// the same thread; stages with h < P pair lanes via __shfl_xor_sync. Every
// thread carries a batch of NB independent transforms (e.g. all r
// polynomial-coefficient columns) so each shuffle stage has NB-way ILP.
//   fft_dif: natural-order input  -> bit-reversed output
//   fft_dit: bit-reversed input   -> natural-order output
// Both are unnormalized; sign = -1 forward, +1 backward (FFTW convention used by
// the reference, /root/reference/proj/core/src/fft_internal.hpp:25-26).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

// Profiling experiments (stage-skipping switches used to split a kernel's time
// between its phases) exist only in a -DPFTG_PROFILING build of the library
// (tools/); in the product build PFTG_DBG is a compile-time false and the
// experiment branches are compiled out.
#ifdef PFTG_PROFILING
#define PFTG_DBG(d, m) ((((d) & (m)) != 0))
#else
#define PFTG_DBG(d, m) (false && (d))
#endif

namespace pftg {

template <class R>
struct CT;
template <>
struct CT<float> {
  using C = float2;
  static __host__ __device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
};
template <>
struct CT<double> {
  using C = double2;
  static __host__ __device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
};

template <class C>
struct RT;
template <>
struct RT<float2> { using R = float; };
template <>
struct RT<double2> { using R = double; };

template <class C>
__device__ __forceinline__ C cadd(C a, C b) { a.x += b.x; a.y += b.y; return a; }
template <class C>
__device__ __forceinline__ C csub(C a, C b) { a.x -= b.x; a.y -= b.y; return a; }
template <class C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
// conj(a) * b
template <class C>
__device__ __forceinline__ C cmulc(C a, C b) {
  C r;
  r.x = a.x * b.x + a.y * b.y;
  r.y = a.x * b.y - a.y * b.x;
  return r;
}
// acc += a * b
template <class C>
__device__ __forceinline__ void cmac(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <class C>
__device__ __forceinline__ void cmacc(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// acc += B * z where B is the plan's B[l][j] entry, which is purely real for
// even j and purely imaginary for odd j (/root/reference/proj/core/src/minimax.cpp:326-330,
// pft.cpp:52-61); bv holds its nonzero part. 2 FMA per complex MAC.
template <class C, class R>
__device__ __forceinline__ void bmac(C& acc, R bv, C z, bool odd) {
  if (!odd) {
    acc.x = fma(bv, z.x, acc.x);
    acc.y = fma(bv, z.y, acc.y);
  } else {
    acc.x = fma(-bv, z.y, acc.x);
    acc.y = fma(bv, z.x, acc.y);
  }
}
// acc += conj(B) * z
template <class C, class R>
__device__ __forceinline__ void bmacc(C& acc, R bv, C z, bool odd) {
  if (!odd) {
    acc.x = fma(bv, z.x, acc.x);
    acc.y = fma(bv, z.y, acc.y);
  } else {
    acc.x = fma(bv, z.y, acc.x);
    acc.y = fma(-bv, z.x, acc.y);
  }
}
// acc * s + x (Horner step with a real base)
template <class C, class R>
__device__ __forceinline__ C cfmar(C acc, R s, C x) {
  acc.x = fma(acc.x, s, x.x);
  acc.y = fma(acc.y, s, x.y);
  return acc;
}
template <class C, class R>
__device__ __forceinline__ C cscale(C a, R s) { a.x *= s; a.y *= s; return a; }

// ---- complex64: packed f32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2) ----
// One packed instruction updates both halves of a complex value; each half is
// rounded exactly like the scalar FFMA/FADD/FMUL it replaces. Non-template
// overloads, so every complex64 caller of the helpers above picks them up.
__device__ __forceinline__ unsigned long long f2pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 f2upk(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2pk(a)), "l"(f2pk(b)), "l"(f2pk(c)));
  return f2upk(d);
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(d);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(d);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(d);
}
// a * b = a.x (b.x, b.y) + a.y (-b.y, b.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return f2fma(make_float2(a.x, a.x), b, f2mul(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
}
// conj(a) * b = a.x (b.x, b.y) + a.y (b.y, -b.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return f2fma(make_float2(a.x, a.x), b, f2mul(make_float2(a.y, a.y), make_float2(b.y, -b.x)));
}
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc = f2fma(make_float2(a.x, a.x), b, acc);
  acc = f2fma(make_float2(a.y, a.y), make_float2(-b.y, b.x), acc);
}
__device__ __forceinline__ void cmacc(float2& acc, float2 a, float2 b) {
  acc = f2fma(make_float2(a.x, a.x), b, acc);
  acc = f2fma(make_float2(a.y, a.y), make_float2(b.y, -b.x), acc);
}
__device__ __forceinline__ void bmac(float2& acc, float bv, float2 z, bool odd) {
  acc = odd ? f2fma(make_float2(-bv, bv), make_float2(z.y, z.x), acc) : f2fma(make_float2(bv, bv), z, acc);
}
__device__ __forceinline__ void bmacc(float2& acc, float bv, float2 z, bool odd) {
  acc = odd ? f2fma(make_float2(bv, -bv), make_float2(z.y, z.x), acc) : f2fma(make_float2(bv, bv), z, acc);
}
__device__ __forceinline__ float2 cfmar(float2 acc, float s, float2 x) { return f2fma(acc, make_float2(s, s), x); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return f2mul(a, make_float2(s, s)); }

// e + (-i) o and e - (-i) o
template <class C>
__device__ __forceinline__ C cadd_mi(C e, C o) { e.x += o.y; e.y -= o.x; return e; }
template <class C>
__device__ __forceinline__ C csub_mi(C e, C o) { e.x -= o.y; e.y += o.x; return e; }
__device__ __forceinline__ float2 cadd_mi(float2 e, float2 o) { return f2fma(make_float2(o.y, o.x), make_float2(1.f, -1.f), e); }
__device__ __forceinline__ float2 csub_mi(float2 e, float2 o) { return f2fma(make_float2(o.y, o.x), make_float2(-1.f, 1.f), e); }

template <class C>
__device__ __forceinline__ C czero() { C r; r.x = 0; r.y = 0; return r; }

template <class C>
__device__ __forceinline__ C shfl_xor(C v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  return v;
}

__host__ __device__ __forceinline__ int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

__device__ __forceinline__ int bitrev(int i, int bits) { return static_cast<int>(__brev(static_cast<unsigned>(i)) >> (32 - bits)) & ((1 << bits) - 1); }

// Twiddle lookup: tw[k] = exp(-2*pi*i*k/len) for k < len/2 (forward); sign=+1 conjugates.
template <class C>
__device__ __forceinline__ C twiddle(const C* tw, int k, int sign) {
  C w = tw[k];
  if (sign > 0) w.y = -w.y;
  return w;
}

// DIF over the lane group. x[s][b]: slot s, batch b. len = P*S, P <= 32 lanes
// (lanes of a group are lane_in_group = lane & (P-1); groups are P-aligned).
// tw: table for length len.
template <int S, int NB, class C>
__device__ __forceinline__ void fft_dif(C (&x)[S][NB], int len, int P, int lig, const C* tw,
                                        int sign) {
  // in-thread stages: h = len/2 ... P   (pairs slot s and s + h/P)
#pragma unroll
  for (int hs = S / 2; hs >= 1; hs >>= 1) {
    const int h = hs * P;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if ((s & hs) == 0) {
        const int i = s * P + lig;
        const C w = twiddle(tw, (i & (h - 1)) * (len / (2 * h)), sign);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const C a = x[s][b], c = x[s + hs][b];
          x[s][b] = cadd(a, c);
          x[s + hs][b] = cmul(csub(a, c), w);
        }
      }
    }
  }
  // cross-lane stages: h = P/2 ... 1. Branch-free butterfly: x' = (s x + o) w'
  // with s = -1, w' = w on the upper lane and s = +1, w' = 1 on the lower one
  // (bit-identical to the select form for finite values: o - x and x + o are
  // single roundings, and a product with (1, 0) is exact).
  using Rr = typename RT<C>::R;
#pragma unroll
  for (int h = P / 2; h >= 1; h >>= 1) {
    const bool upper = (lig & h) != 0;
    C w = twiddle(tw, (lig & (h - 1)) * (len / (2 * h)), sign);
    if (!upper) w = CT<Rr>::mk(Rr(1), Rr(0));
    const Rr sg = upper ? Rr(-1) : Rr(1);
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const C o = shfl_xor(x[s][b], h);
        x[s][b] = cmul(cfmar(x[s][b], sg, o), w);
      }
  }
}

// DIT over the lane group: bit-reversed input -> natural output.
template <int S, int NB, class C>
__device__ __forceinline__ void fft_dit(C (&x)[S][NB], int len, int P, int lig, const C* tw,
                                        int sign) {
  using Rr = typename RT<C>::R;
#pragma unroll
  for (int h = 1; h < P; h <<= 1) {
    const bool upper = (lig & h) != 0;
    C w = twiddle(tw, (lig & (h - 1)) * (len / (2 * h)), sign);
    if (!upper) w = CT<Rr>::mk(Rr(1), Rr(0));
    const Rr sg = upper ? Rr(-1) : Rr(1);
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        // lower: a + w*c ; upper: a - w*c, where c is the upper element (branch-free, see fft_dif)
        const C mine = cmul(x[s][b], w);
        const C o = shfl_xor(mine, h);
        x[s][b] = cfmar(mine, sg, o);
      }
  }
#pragma unroll
  for (int hs = 1; hs < S; hs <<= 1) {
    const int h = hs * P;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if ((s & hs) == 0) {
        const int i = s * P + lig;
        const C w = twiddle(tw, (i & (h - 1)) * (len / (2 * h)), sign);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const C a = x[s][b];
          const C t = cmul(x[s + hs][b], w);
          x[s][b] = cadd(a, t);
          x[s + hs][b] = csub(a, t);
        }
      }
    }
  }
}

// Non-negative t mod p (/root/reference/proj/core/src/pft.cpp:25-29).
__host__ __device__ __forceinline__ int mod_nonneg(int t, int p) {
  int m = t % p;
  return m < 0 ? m + p : m;
}

// Band contraction by Horner's rule (complex64 hot path). The plan's band
// matrix is W[j][b] = tw(b) * base_b^j with base_b = (b - mt) / p and
// tw(b) = W[0][b] (plan.cpp / pft.cpp:75-88), so
//   out[b] = sum_j W[j][b] x[j] = tw(b) * (x0 + base_b (x1 + base_b (x2 + ...))):
// 2 real FMAs per tap instead of 4, and one table load per output instead of
// r. base_b is exact in binary floating point (integer over a power of two).
template <int RB, class C, class R, class Emit>
__device__ __forceinline__ void band_horner(const C* __restrict__ W0, int M, int a0, int step, int mt, R inv_p,
                                            const C (&x)[RB], Emit&& emit) {
  for (int a = a0; a < M; a += step) {
    const R base = static_cast<R>(a - mt) * inv_p;
    C acc = x[RB - 1];
#pragma unroll
    for (int j = RB - 2; j >= 0; --j) acc = cfmar(acc, base, x[j]);
    emit(a, cmul(W0[a], acc));
  }
}

// Adjoint of the Horner band (D-dagger gather term): x[j] += conj(W[j][b]) g
// = base_b^j * (conj(tw(b)) g), with the powers of base_b built incrementally.
template <int RB, class C, class R>
__device__ __forceinline__ void gather_horner(C (&x)[RB], C tw, R base, C g) {
  C p = cmulc(tw, g);
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    x[j] = cadd(x[j], p);
    if (j + 1 < RB) p = cscale(p, base);
  }
}


}  // namespace pftg
