// 1-D partial Fourier transform: pft::pft_apply_1d
// (pft.hpp:33-38, pft.cpp:78-101) for batches of independent n-vectors.
//
//   C[k][j]  = sum_l z[k q + l] B[l][j]        reshape(z, p x q) * B   (pft.cpp:85-88)
//   C^[u][j] = sum_k C[k][j] e^{-2 pi i k u / p}                     (pft.cpp:89, FFTW_FORWARD)
//   out[i]   = sum_j C^[(i - mt) mod p][j] W[i][j],  i in [0, 2mt]   (pft.cpp:91-99)
//
// Three stream-ordered passes over a per-call scratch C laid out [v][j][k]
// (column j of a vector contiguous, so the p-point transform reads it as one run):
//  k1_contract  one warp per (vector, k) row: lanes stride the q row elements
//               (coalesced, each z element read once from HBM), j-chunks of 16
//               accumulators per lane, butterfly warp reduction;
//  k1_fft       one CTA per (vector, j): the column in shared memory, iterative
//               radix-2 DIT for power-of-two p, direct O(p^2) DFT otherwise;
//  k1_band      one thread per (vector, i): the W contraction, ascending j like
//               the reference.
// The 1-D PFT is not on a BASELINE workload; it serves the reference's 1-D API
// (the 2-D operator is the separable product of two of these, pft.hpp:40-43).
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pftg.h"
#include "internal.hpp"

namespace pftg {
void set_error(const std::string& m);
void ensure_device();
}  // namespace pftg

using namespace pftg;

namespace {

template <class R>
using Cx = typename CT<R>::C;

template <class R>
__device__ __forceinline__ Cx<R> cmac(Cx<R> acc, Cx<R> a, Cx<R> b) {
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
  return acc;
}

constexpr int kJC = 16;  // accumulators per lane per j-chunk

template <class R>
__global__ void __launch_bounds__(256) k1_contract(const Cx<R>* __restrict__ z, const Cx<R>* __restrict__ B,
                                                   Cx<R>* __restrict__ Cs, long long rows_total, int p, int q, int r) {
  const long long row = blockIdx.x * 8LL + (threadIdx.x >> 5);  // (vector, k)
  if (row >= rows_total) return;
  const int lane = threadIdx.x & 31;
  const long long v = row / p;
  const int k = (int)(row % p);
  const Cx<R>* zr = z + row * q;  // rows of consecutive vectors are back to back
  for (int j0 = 0; j0 < r; j0 += kJC) {
    Cx<R> acc[kJC];
#pragma unroll
    for (int t = 0; t < kJC; ++t) acc[t] = Cx<R>{R(0), R(0)};
    for (int l = lane; l < q; l += 32) {
      const Cx<R> zv = zr[l];
      const Cx<R>* Bl = B + (long long)l * r + j0;
#pragma unroll
      for (int t = 0; t < kJC; ++t)
        if (j0 + t < r) acc[t] = cmac<R>(acc[t], zv, Bl[t]);
    }
#pragma unroll
    for (int t = 0; t < kJC; ++t) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[t].x += __shfl_xor_sync(0xffffffffu, acc[t].x, o);
        acc[t].y += __shfl_xor_sync(0xffffffffu, acc[t].y, o);
      }
    }
    // lane t stores column j0 + t (registers indexed by a compile-time t)
#pragma unroll
    for (int t = 0; t < kJC; ++t)
      if (lane == t && j0 + t < r) Cs[(v * r + j0 + t) * p + k] = acc[t];
  }
}

template <class R>
__global__ void __launch_bounds__(256) k1_fft(Cx<R>* __restrict__ Cs, int p, int logp) {
  extern __shared__ unsigned char smem_raw[];
  Cx<R>* s = reinterpret_cast<Cx<R>*>(smem_raw);
  Cx<R>* col = Cs + (long long)blockIdx.x * p;  // one (vector, j) column
  if (logp >= 0) {
    for (int i = threadIdx.x; i < p; i += blockDim.x) s[__brev((unsigned)i) >> (32 - logp)] = col[i];
    __syncthreads();
    for (int half = 1; half < p; half <<= 1) {
      for (int t = threadIdx.x; t < p / 2; t += blockDim.x) {
        const int pos = t & (half - 1);
        const int i0 = ((t - pos) << 1) + pos, i1 = i0 + half;
        R sn, cs;
        sincospi(-(R)pos / (R)half, &sn, &cs);  // e^{-2 pi i pos / (2 half)}
        const Cx<R> a = s[i0], b = s[i1];
        const Cx<R> bw{b.x * cs - b.y * sn, b.x * sn + b.y * cs};
        s[i0] = Cx<R>{a.x + bw.x, a.y + bw.y};
        s[i1] = Cx<R>{a.x - bw.x, a.y - bw.y};
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < p; i += blockDim.x) col[i] = s[i];
  } else {
    for (int i = threadIdx.x; i < p; i += blockDim.x) s[i] = col[i];
    __syncthreads();
    for (int u = threadIdx.x; u < p; u += blockDim.x) {
      Cx<R> acc{R(0), R(0)};
      long long e = 0;  // (k u) mod p, exact
      for (int k = 0; k < p; ++k) {
        R sn, cs;
        sincospi(-2 * (R)e / (R)p, &sn, &cs);
        acc = cmac<R>(acc, s[k], Cx<R>{cs, sn});
        e += u;
        if (e >= p) e -= p;
      }
      col[u] = acc;  // s holds the input copy, so the global store cannot race the reads
    }
  }
}

template <class R>
__global__ void __launch_bounds__(256) k1_band(const Cx<R>* __restrict__ Cs, const Cx<R>* __restrict__ W,
                                               Cx<R>* __restrict__ out, long long total, int p, int mt, int r) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int m = 2 * mt + 1;
  if (g >= total) return;
  const long long v = g / m;
  const int i = (int)(g % m);
  int u = (i - mt) % p;
  if (u < 0) u += p;
  const Cx<R>* c = Cs + v * r * (long long)p + u;
  Cx<R> acc{R(0), R(0)};
  for (int j = 0; j < r; ++j) acc = cmac<R>(acc, c[(long long)j * p], W[(long long)i * r + j]);
  out[g] = acc;
}

template <class R>
struct Dev1D {
  Cx<R>* B = nullptr;
  Cx<R>* W = nullptr;
};

}  // namespace

// pft::PftPlan1D (pft.hpp:25-31): host tables + lazily uploaded device copies
// per (device, precision); immutable once created.
struct pftg_plan1d {
  Axis a;
  mutable std::mutex mu;
  mutable std::map<int, Dev1D<float>> d32;
  mutable std::map<int, Dev1D<double>> d64;
  ~pftg_plan1d() {
    for (auto& kv : d32) {
      cudaFree(kv.second.B);
      cudaFree(kv.second.W);
    }
    for (auto& kv : d64) {
      cudaFree(kv.second.B);
      cudaFree(kv.second.W);
    }
  }
};

namespace {

template <class R>
std::map<int, Dev1D<R>>& dev_map(const pftg_plan1d& p);
template <>
std::map<int, Dev1D<float>>& dev_map<float>(const pftg_plan1d& p) { return p.d32; }
template <>
std::map<int, Dev1D<double>>& dev_map<double>(const pftg_plan1d& p) { return p.d64; }

template <class R>
Dev1D<R> plan_dev1d(const pftg_plan1d& p) {
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(p.mu);
  auto& m = dev_map<R>(p);
  auto it = m.find(dev);
  if (it != m.end()) return it->second;
  auto cast = [](const std::vector<cd>& v) {
    std::vector<Cx<R>> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = Cx<R>{(R)v[i].real(), (R)v[i].imag()};
    return o;
  };
  const auto hb = cast(p.a.B), hw = cast(p.a.W);
  Dev1D<R> d;
  PFTG_CUDA(cudaMalloc(&d.B, sizeof(Cx<R>) * hb.size()));
  PFTG_CUDA(cudaMalloc(&d.W, sizeof(Cx<R>) * hw.size()));
  // uploads complete (stream synchronized) before any caller stream can read the tables
  cudaStream_t up;
  PFTG_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  PFTG_CUDA(cudaMemcpyAsync(d.B, hb.data(), sizeof(Cx<R>) * hb.size(), cudaMemcpyHostToDevice, up));
  PFTG_CUDA(cudaMemcpyAsync(d.W, hw.data(), sizeof(Cx<R>) * hw.size(), cudaMemcpyHostToDevice, up));
  PFTG_CUDA(cudaStreamSynchronize(up));
  PFTG_CUDA(cudaStreamDestroy(up));
  m.emplace(dev, d);
  return d;
}

constexpr int kMaxP = 8192;

template <class R>
std::size_t fft_smem(int p) {
  return sizeof(Cx<R>) * (std::size_t)p;
}

template <class R>
void apply1d(const pftg_plan1d& plan, const void* z, void* out, std::size_t batch, cudaStream_t st) {
  const Axis& a = plan.a;
  const int p = (int)a.p, q = (int)a.q, r = a.r, mt = (int)a.mt;
  if (p > kMaxP)
    throw std::invalid_argument("pft_apply_1d: the GPU slice FFT supports p <= " + std::to_string(kMaxP));
  const Dev1D<R> d = plan_dev1d<R>(plan);
  Cx<R>* Cs = nullptr;
  PFTG_CUDA(cudaMallocAsync(&Cs, sizeof(Cx<R>) * batch * (std::size_t)p * r, st));
  const long long rows = (long long)batch * p;
  k1_contract<R><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(static_cast<const Cx<R>*>(z), d.B, Cs, rows, p, q, r);
  PFTG_LAUNCH_CHECK();
  const bool pow2 = (p & (p - 1)) == 0;
  int logp = -1;
  if (pow2)
    for (logp = 0; (1 << logp) < p; ++logp) {
    }
  const std::size_t sm = fft_smem<R>(p);
  // per call: the opt-in is per (kernel, device) and costs ~1 us
  PFTG_CUDA(cudaFuncSetAttribute(k1_fft<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k1_fft<R><<<(unsigned)(batch * r), 256, sm, st>>>(Cs, p, logp);
  PFTG_LAUNCH_CHECK();
  const long long total = (long long)batch * (2 * mt + 1);
  k1_band<R><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(Cs, d.W, static_cast<Cx<R>*>(out), total, p, mt, r);
  PFTG_LAUNCH_CHECK();
  PFTG_CUDA(cudaFreeAsync(Cs, st));
}

template <class F>
int guarded1d(F&& f) {
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

void check1d(const pftg_plan1d* p) {
  if (!p) throw std::invalid_argument("pftg: null 1-D plan");
}

}  // namespace

extern "C" {

int pftg_plan_1d(const pftg_table* t, size_t n, size_t mt, size_t p, double eps, pftg_plan1d** out) {
  return guarded1d([&] {
    if (!t) throw std::invalid_argument("pftg_plan_1d: null scope table");
    if (!out) throw std::invalid_argument("pftg_plan_1d: null output");
    auto h = std::make_unique<pftg_plan1d>();
    h->a = plan_1d(n, mt, p, eps, t->t);
    *out = h.release();
  });
}

int pftg_plan1d_from_tables(size_t n, size_t p, size_t mt, int r, const double* B, const double* W, double eps,
                            pftg_plan1d** out) {
  return guarded1d([&] {
    if (!out) throw std::invalid_argument("pftg_plan1d_from_tables: null output");
    // pft_plan_1d's domain (pft.cpp:35-40)
    if (p < 2 || p > n || n % p != 0) throw std::invalid_argument("pft_plan_1d: p must divide n, 2 <= p <= n");
    if (n / p < 2) throw std::invalid_argument("pft_plan_1d: need q = n/p >= 2");
    if (mt < 1 || 2 * mt > n) throw std::invalid_argument("pft_plan_1d: need 1 <= mt and 2*mt <= n");
    if (r < 1) throw std::invalid_argument("pft_plan_1d: need r >= 1");
    if (!B || !W) throw std::invalid_argument("pftg_plan1d_from_tables: null table");
    auto h = std::make_unique<pftg_plan1d>();
    Axis& a = h->a;
    a.n = n;
    a.p = p;
    a.q = n / p;
    a.mt = mt;
    a.r = r;
    a.eps = eps;
    const cd* b = reinterpret_cast<const cd*>(B);
    const cd* w = reinterpret_cast<const cd*>(W);
    a.B.assign(b, b + a.q * (size_t)r);
    a.W.assign(w, w + (2 * mt + 1) * (size_t)r);
    *out = h.release();
  });
}

int pftg_plan1d_load(const char* path, pftg_plan1d** out) {
  return guarded1d([&] {
    if (!path || !out) throw std::invalid_argument("pftg_plan1d_load: null argument");
    auto h = std::make_unique<pftg_plan1d>();
    plan_load_1d(h->a, path);
    *out = h.release();
  });
}

int pftg_plan1d_save(const pftg_plan1d* plan, const char* path) {
  return guarded1d([&] {
    check1d(plan);
    if (!path) throw std::invalid_argument("pftg_plan1d_save: null path");
    plan_save_1d(plan->a, path);
  });
}

int pftg_plan1d_info(const pftg_plan1d* plan, int64_t* info) {
  return guarded1d([&] {
    check1d(plan);
    info[0] = (int64_t)plan->a.n;
    info[1] = (int64_t)plan->a.p;
    info[2] = (int64_t)plan->a.q;
    info[3] = (int64_t)plan->a.mt;
    info[4] = plan->a.r;
  });
}

int pftg_plan1d_tables(const pftg_plan1d* plan, double* B, double* W) {
  return guarded1d([&] {
    check1d(plan);
    std::copy(plan->a.B.begin(), plan->a.B.end(), reinterpret_cast<cd*>(B));
    std::copy(plan->a.W.begin(), plan->a.W.end(), reinterpret_cast<cd*>(W));
  });
}

void pftg_plan1d_free(pftg_plan1d* plan) { delete plan; }

int pftg_apply_1d_dev(const pftg_plan1d* plan, int dtype, const void* z, void* out, size_t batch, void* stream) {
  return guarded1d([&] {
    check1d(plan);
    if (dtype != PFTG_C64 && dtype != PFTG_C128) throw std::invalid_argument("pftg: dtype must be PFTG_C64 or PFTG_C128");
    if (batch == 0) return;
    ensure_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == PFTG_C64) apply1d<float>(*plan, z, out, batch, st);
    else apply1d<double>(*plan, z, out, batch, st);
  });
}

int pftg_apply_1d_host(const pftg_plan1d* plan, int dtype, const void* z, void* out, size_t batch) {
  return guarded1d([&] {
    check1d(plan);
    if (dtype != PFTG_C64 && dtype != PFTG_C128) throw std::invalid_argument("pftg: dtype must be PFTG_C64 or PFTG_C128");
    if (batch == 0) return;
    ensure_device();
    const std::size_t es = dtype == PFTG_C64 ? 8 : 16;
    const std::size_t zin = es * batch * plan->a.n, zout = es * batch * (2 * plan->a.mt + 1);
    cudaStream_t st;
    PFTG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void *dz = nullptr, *dout = nullptr;
    try {
      PFTG_CUDA(cudaMallocAsync(&dz, zin, st));
      PFTG_CUDA(cudaMallocAsync(&dout, zout, st));
      PFTG_CUDA(cudaMemcpyAsync(dz, z, zin, cudaMemcpyHostToDevice, st));
      if (dtype == PFTG_C64) apply1d<float>(*plan, dz, dout, batch, st);
      else apply1d<double>(*plan, dz, dout, batch, st);
      PFTG_CUDA(cudaMemcpyAsync(out, dout, zout, cudaMemcpyDeviceToHost, st));
      PFTG_CUDA(cudaFreeAsync(dz, st));
      PFTG_CUDA(cudaFreeAsync(dout, st));
      PFTG_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    PFTG_CUDA(cudaStreamDestroy(st));
  });
}

}  // extern "C"
