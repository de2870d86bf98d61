// Device-resident hybrid_solve (PFT-warm-started ePIE).
//
// Reference: /root/reference/proj/core/src/solver.cpp:173-302. Semantics kept:
//  - positions visited in list order, or shuffled per sweep with the
//    reference's mt19937_64 Fisher-Yates stream (solver.cpp:164-169, 223, 236);
//  - stage = band iff sweep <= pft_sweeps (233); band plan defaults
//    mt = window/8, p = mt (195-198); dcrop = crop_centered(d) (202-208);
//  - band stage per position: resid = band_residual(P z_j); z_j -= beta_pft
//    conj(P) resid; blind: resid2 from the updated z_j, P -= gamma_pft conj(z_j)
//    resid2 (243-251);
//  - FFT stage: pie_object_update then (blind) epie_probe_update with the
//    projection of the updated exit wave (253-259);
//  - per sweep: objective over all positions (287), divergence guards
//    (291-295) and the relative-change stop (296-299).
//  - per sweep, when tv_lambda_mag / tv_lambda_phase > 0: one TV gradient
//    step on |z| and arg z of the whole frame, step lambda * (beta_pft in the
//    band stage, beta in the FFT stage), recomposed by polar (264-279); k_tv.
//
// Each position is 3 (non-blind) or 5 (blind) kernel launches that keep the
// patch, spectrum and PFT intermediates in L2; a whole sweep is captured once
// into a CUDA graph (sequential order) and replayed.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include "band_sweep.cuh"
#include "epie_sweep.cuh"
#include "eval_fft.cuh"
#include "../../include/pftg.h"
#include "internal.hpp"

namespace pftg {
void set_error(const std::string& m);
}

using namespace pftg;

namespace {

template <class R>
__global__ void k_norm_finite(const typename CT<R>::C* __restrict__ a, long long n, double* __restrict__ out) {
  // out[0] += sum |a|^2 per CTA partial (written to out[blockIdx.x]); out[gridDim.x + blockIdx.x] = nonfinite count
  double s = 0.0, bad = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const auto v = a[i];
    if (!isfinite(v.x) || !isfinite(v.y)) bad += 1.0;
    s += (double)v.x * v.x + (double)v.y * v.y;
  }
  __shared__ double sh[2][32];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = s;
    sh[1][threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0, tb = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      ts += sh[0][w];
      tb += sh[1][w];
    }
    out[blockIdx.x] = ts;
    out[gridDim.x + blockIdx.x] = tb;
  }
}

template <class R>
__global__ void k_diff_norm(const typename CT<R>::C* __restrict__ a, const typename CT<R>::C* __restrict__ b,
                            long long n, double* __restrict__ out) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double dx = (double)a[i].x - b[i].x, dy = (double)a[i].y - b[i].y;
    s += dx * dx + dy * dy;
  }
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    out[blockIdx.x] = t;
  }
}

template <class R>
__global__ void k_crop_real(const R* __restrict__ d, R* __restrict__ out, int w1, int w2, int mt1, int mt2,
                            long long count) {
  const long long M = 4LL * mt1 * mt2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < M * count;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / M;
    const int rem = (int)(i % M);
    const int a = rem / (2 * mt2), b = rem % (2 * mt2);
    out[i] = d[f * (long long)w1 * w2 + (long long)mod_nonneg(a - mt1, w1) * w2 + mod_nonneg(b - mt2, w2)];
  }
}

constexpr int kRedBlocks = 296;

// TV step (solver.cpp:71-87 tv_gradient, 264-279): psi'(t) = t / sqrt(t^2 + 1e-6^2)
// over the 4-neighbourhood with one-sided edges, on mag = |z| and ph = arg z
// (phase of 0 is 0, field.cpp:80-87), then z = polar(mag - lm g(mag), ph - lp g(ph)).
// A 32 x 8 tile stages mag / ph with a one-pixel halo in shared memory, so each
// pixel's atan2 / hypot runs ~1.3 times instead of 5. Out-of-place (out != z).
template <class R>
__device__ __forceinline__ R tv_psi(R t) {
  const R delta = R(1e-6);
  return t / sqrt(t * t + delta * delta);
}

template <class R>
__global__ void __launch_bounds__(256) k_tv(const typename CT<R>::C* __restrict__ z, typename CT<R>::C* __restrict__ out,
                                            int rows, int cols, R lm, R lp) {
  __shared__ R sm[10][34], sp[10][34];
  const int i0 = blockIdx.y * 8, j0 = blockIdx.x * 32;
  for (int t = threadIdx.y * 32 + threadIdx.x; t < 10 * 34; t += 256) {
    const int ti = t / 34, tj = t % 34;
    const int i = i0 + ti - 1, j = j0 + tj - 1;
    R m = 0, ph = 0;
    if (i >= 0 && i < rows && j >= 0 && j < cols) {
      const auto v = z[(long long)i * cols + j];
      m = hypot(v.x, v.y);
      ph = (v.x == R(0) && v.y == R(0)) ? R(0) : atan2(v.y, v.x);
    }
    sm[ti][tj] = m;
    sp[ti][tj] = ph;
  }
  __syncthreads();
  const int i = i0 + threadIdx.y, j = j0 + threadIdx.x;
  if (i >= rows || j >= cols) return;
  const int a = threadIdx.y + 1, b = threadIdx.x + 1;
  R gm = 0, gp = 0;
  if (i + 1 < rows) {
    gm -= tv_psi(sm[a + 1][b] - sm[a][b]);
    gp -= tv_psi(sp[a + 1][b] - sp[a][b]);
  }
  if (i > 0) {
    gm += tv_psi(sm[a][b] - sm[a - 1][b]);
    gp += tv_psi(sp[a][b] - sp[a - 1][b]);
  }
  if (j + 1 < cols) {
    gm -= tv_psi(sm[a][b + 1] - sm[a][b]);
    gp -= tv_psi(sp[a][b + 1] - sp[a][b]);
  }
  if (j > 0) {
    gm += tv_psi(sm[a][b] - sm[a][b - 1]);
    gp += tv_psi(sp[a][b] - sp[a][b - 1]);
  }
  R m = sm[a][b], ph = sp[a][b];
  if (lm > R(0)) m -= lm * gm;
  if (lp > R(0)) ph -= lp * gp;
  R sn, cs;
  sincos(ph, &sn, &cs);
  typename CT<R>::C o;
  o.x = m * cs;  // std::polar (libstdc++): (rho cos theta, rho sin theta)
  o.y = m * sn;
  out[(long long)i * cols + j] = o;
}

}  // namespace

struct pftg_solver {
  int dtype = PFTG_C64;
  std::size_t fr = 0, fc = 0, wr = 0, wc = 0, npos = 0;
  pftg_solver_config cfg{};
  std::vector<long long> offs;  // linear offsets r0*fc + c0, reference list order
  std::vector<std::size_t> order;
  std::mt19937_64 shuffle_rng;
  std::unique_ptr<pftg_plan> plan;
  cudaStream_t st = nullptr;
  void* frame = nullptr;
  void* probe = nullptr;
  void* prev = nullptr;
  void* tv = nullptr;  // TV step output (frame-sized)
  unsigned* bar = nullptr;  // grid-barrier counter of the persistent FFT-stage sweep
  void* d = nullptr;
  void* dperm = nullptr;
  void* dcrop = nullptr;
  long long* doffs = nullptr;  // per list position
  int graph_launches[2][K_NUM] = {};  // kernel launches captured per graph (credited per replay)
  void* G = nullptr;
  void* Gt = nullptr;
  void* X = nullptr;
  void* X2 = nullptr;
  void* Xe = nullptr;  // evaluator chunk
  double* part = nullptr;
  double* red = nullptr;
  std::size_t eval_chunk = 1;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // [band, fft]
  std::vector<double> objective, wall;
  int sweeps_run = 0;
  int flags = 0;
  bool fwd_ready = false;  // enqueue state: the next position's forward rows are already fused in
  double frame_guard = 0, probe_guard = 0;
  double t_accum = 0;

  ~pftg_solver() {
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    void* bufs[] = {frame, probe, prev, tv, bar, d, dperm, dcrop, doffs, G, Gt, X, X2, Xe, part, red};
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

template <class R>
using Cx = typename CT<R>::C;

// Full-FFT stage and objective on the radix-8 register FFT kernels (eval_fft.cuh):
// complex64 512 x 512 windows. PFTG_EPIE_LANEFFT=1 keeps the lane-group kernels.
inline bool use_fft512(const pftg_solver& s) {
  const bool off = knobs().epie_lanefft;
  return !off && s.wr == 512 && s.wc == 512;
}
// The same for the per-position FFT stage of 256 x 256 windows (BASELINE configs[2]).
inline bool use_fft256(const pftg_solver& s) {
  const bool off = knobs().epie_lanefft;
  return !off && s.wr == 256 && s.wc == 256;
}

// Launch with programmatic stream serialization (also inside stream capture: the
// graph gets programmatic edges). The kernels release their dependents only after
// their own griddepcontrol.wait, so a kernel's prologue and operand prefetch overlap
// its predecessor, never the kernel before that. PFTG_FFT_NO_PDL=1: plain launches.
template <class... KA, class... A>
void launch_pdl_pos(void (*kernel)(KA...), dim3 grid, dim3 block, cudaStream_t st, A&&... args) {
  static const bool off = std::getenv("PFTG_FFT_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PFTG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

// jn: the next position in this sweep's visit order (-1 for the last): blind
// FFT-stage positions fuse the next position's forward row transform into
// their probe-update kernel (cross-position fusion, 5 -> 4 launches each).
template <class R>
void enqueue_position(pftg_solver& s, std::size_t j, bool band, long long jn) {
  const cudaStream_t st = s.st;
  const int n1 = (int)s.wr, n2 = (int)s.wc;
  const long long n = (long long)n1 * n2;
  Cx<R>* frame = static_cast<Cx<R>*>(s.frame);
  Cx<R>* probe = static_cast<Cx<R>*>(s.probe);
  const long long* doff = s.doffs + j;
  const bool blind = s.cfg.blind != 0;
  if (band) {
    const PftDev<R>& pd = plan_dev<R>(*s.plan);
    const long long mb = (long long)pd.M1 * pd.M2;
    const R* dc = static_cast<const R*>(s.dcrop) + (long long)j * mb;
    // 16-byte column pairs when the window starts on an even column of an even-width frame
    const int vec = (s.offs[j] % 2 == 0) && (s.fc % 2 == 0) && (s.wc % 2 == 0);
    Src<R> src{frame, (long long)s.fc, 0, doff, probe, vec};
    if (!s.fwd_ready) launch_fwd_rows<R>(pd, src, static_cast<Cx<R>*>(s.G), 1, st);
    launch_fwd_cols<R>(pd, 1, static_cast<Cx<R>*>(s.G), nullptr, dc, mb, static_cast<Cx<R>*>(s.Gt), nullptr, 1, st);
    EpiArgs ep{};
    ep.obj = frame;
    ep.obj_ld = (long long)s.fc;
    ep.obj_off = s.offs[j];
    ep.probe = probe;
    ep.step = s.cfg.beta_pft;
    ep.G2 = blind ? s.G : nullptr;
    ep.vec_ok = vec;
    ep.dbg = knobs().debug_adj;
    launch_adj_rows<R>(pd, 1, static_cast<Cx<R>*>(s.Gt), ep, 1, st);
    if (blind) {
      launch_fwd_cols<R>(pd, 1, static_cast<Cx<R>*>(s.G), nullptr, dc, mb, static_cast<Cx<R>*>(s.Gt), nullptr, 1,
                         st);
      ep.step = s.cfg.gamma_pft;
      // cross-position fusion: the probe-update rows kernel also runs the next
      // position's forward rows pass (its exit wave P' z_next) into G
      ep.G2 = jn >= 0 ? s.G : nullptr;
      ep.obj_off2 = jn >= 0 ? s.offs[jn] : 0;
      launch_adj_rows<R>(pd, 2, static_cast<Cx<R>*>(s.Gt), ep, 1, st);
    }
    s.fwd_ready = blind && jn >= 0;
    return;
  }
  if constexpr (sizeof(R) == 4) {
    if (use_fft512(s)) {
      // 512 x 512 complex64 windows (BASELINE configs[3]): radix-8 register FFTs, natural-order spectrum
      // columns per CTA of the projection pass: 8 (64 CTAs x 512 threads, 64-byte row segments):
      // FFT stage 47.1k -> 47.8k updates/s over 4; 2 (256 CTAs): 37.4k
      static const int c512 = std::getenv("PFTG_FFT512_NCOL") ? std::atoi(std::getenv("PFTG_FFT512_NCOL")) : 8;
      auto launch_cols512 = [&](cudaStream_t st_, float2* Xp, const float* dp_, const float2* twp) {
        if (c512 == 2) launch_pdl_pos(ke_cols512_proj<2>, dim3(256), dim3(128), st_, Xp, dp_, twp);
        else if (c512 == 8) launch_pdl_pos(ke_cols512_proj<8>, dim3(64), dim3(512), st_, Xp, dp_, twp);
        else launch_pdl_pos(ke_cols512_proj<4>, dim3(128), dim3(256), st_, Xp, dp_, twp);
      };
      const float2* tw = fft_twiddles<float>(512);
      float2* fr = reinterpret_cast<float2*>(frame);
      float2* pr = reinterpret_cast<float2*>(probe);
      float2* X = static_cast<float2*>(s.X);
      float2* X2 = static_cast<float2*>(s.X2);
      const float* dn = static_cast<const float*>(s.d) + (long long)j * n;
      const float scale = 1.0f / static_cast<float>(n);
      if (!s.fwd_ready) {
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows512_epie<E512_FWD>, dim3(128), dim3(256), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, 1.f, 0.f, 0,
                                                         0);
      }
      {
        ProfScope prof(st, K_FFT_COLS);
        launch_cols512(st, X, dn, tw);
      }
      {
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows512_epie<E512_OBJ>, dim3(128), dim3(256), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, scale,
                                                       (float)s.cfg.beta, blind ? 1 : 0, 0);
      }
      if (blind) {
        {
          ProfScope prof(st, K_FFT_COLS);
          launch_cols512(st, X2, dn, tw);
        }
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows512_epie<E512_PROBE>, dim3(128), dim3(256), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, scale,
                                                         (float)s.cfg.gamma, jn >= 0 ? 1 : 0,
                                                         jn >= 0 ? s.offs[jn] : 0);
      }
      s.fwd_ready = blind && jn >= 0;
      PFTG_LAUNCH_CHECK();
      return;
    }
    if (use_fft256(s)) {
      // 64 CTAs of four rows / four columns each; PFTG_FFT256_GRID=128 (two each, 128 SMs per
      // position) measured slower: FFT stage 74.5k -> 68.7k updates/s (16-byte row segments
      // in the column pass)
      static const int k256g = std::getenv("PFTG_FFT256_GRID") ? std::atoi(std::getenv("PFTG_FFT256_GRID")) : 64;
      auto launch_cols256 = [&](cudaStream_t st_, float2* Xp, const float* dp_, const float2* twp) {
        // 8 columns per CTA (32 CTAs) measured slower here: 73.6k -> 67.7k updates/s
        static const int c256 = std::getenv("PFTG_FFT256_NCOL") ? std::atoi(std::getenv("PFTG_FFT256_NCOL")) : 4;
        if (k256g == 128) launch_pdl_pos(ke_cols256_proj<2>, dim3(128), dim3(64), st_, Xp, dp_, twp);
        else if (c256 == 8) launch_pdl_pos(ke_cols256_proj<8>, dim3(32), dim3(256), st_, Xp, dp_, twp);
        else launch_pdl_pos(ke_cols256_proj<4>, dim3(64), dim3(128), st_, Xp, dp_, twp);
      };
      const float2* tw = fft_twiddles<float>(256);
      float2* fr = reinterpret_cast<float2*>(frame);
      float2* pr = reinterpret_cast<float2*>(probe);
      float2* X = static_cast<float2*>(s.X);
      float2* X2 = static_cast<float2*>(s.X2);
      const float* dn = static_cast<const float*>(s.d) + (long long)j * n;
      const float scale = 1.0f / static_cast<float>(n);
      if (!s.fwd_ready) {
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows256_epie<E512_FWD>, dim3(k256g), dim3(8192 / k256g), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, 1.f, 0.f, 0,
                                                        0);
      }
      {
        ProfScope prof(st, K_FFT_COLS);
        launch_cols256( st, X, dn, tw);
      }
      {
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows256_epie<E512_OBJ>, dim3(k256g), dim3(8192 / k256g), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, scale,
                                                      (float)s.cfg.beta, blind ? 1 : 0, 0);
      }
      if (blind) {
        {
          ProfScope prof(st, K_FFT_COLS);
          launch_cols256( st, X2, dn, tw);
        }
        ProfScope prof(st, K_FFT_ROWS);
        launch_pdl_pos(ke_rows256_epie<E512_PROBE>, dim3(k256g), dim3(8192 / k256g), st, tw, fr, (long long)s.fc, s.offs[j], pr, X, X2, scale,
                                                        (float)s.cfg.gamma, jn >= 0 ? 1 : 0,
                                                        jn >= 0 ? s.offs[jn] : 0);
      }
      s.fwd_ready = blind && jn >= 0;
      PFTG_LAUNCH_CHECK();
      return;
    }
  }
  const R* dp = static_cast<const R*>(s.dperm) + (long long)j * n;
  RowSrc<R> src{frame, (long long)s.fc, 0, doff, probe};
  RowEpiArgs ep{};
  launch_fft_rows<R>(ROW_DIF_STORE, EPI_STORE, n1, n2, src, static_cast<Cx<R>*>(s.X), n, -1, 1.0, ep, 1, st);
  launch_fft_cols<R>(COL_PROJECT, n1, n2, static_cast<Cx<R>*>(s.X), n, dp, n, nullptr, 0, -1, nullptr, 1, st);
  ep.obj = frame;
  ep.obj_ld = (long long)s.fc;
  ep.obj_offs = doff;
  ep.probe = probe;
  ep.step = s.cfg.beta;
  ep.out = s.X2;
  ep.out_bstride = n;
  ep.fuse_next = blind ? 1 : 0;
  const double scale = 1.0 / static_cast<double>(n);
  launch_fft_rows<R>(ROW_DIT_PROJ, EPI_OBJ, n1, n2, src, static_cast<Cx<R>*>(s.X), n, +1, scale, ep, 1, st);
  if (blind) {
    launch_fft_cols<R>(COL_PROJECT, n1, n2, static_cast<Cx<R>*>(s.X2), n, dp, n, nullptr, 0, -1, nullptr, 1, st);
    ep.step = s.cfg.gamma;
    ep.fuse_next = 0;
    launch_fft_rows<R>(ROW_DIT_PROJ, EPI_PROBE, n1, n2, src, static_cast<Cx<R>*>(s.X2), n, +1, scale, ep, 1, st);
  }
}

template <class R>
void enqueue_positions(pftg_solver& s, bool band);
template <class R>
void enqueue_tv(pftg_solver& s, bool band);

// Full-FFT stage, complex64 256^2 / 512^2 windows, list order: the whole sweep
// as one cooperative persistent kernel (epie_sweep.cuh). PFTG_NO_PERSIST=1 keeps
// the per-position graph of four kernels.
template <class R>
bool persistent_fft(const pftg_solver& s, bool band) {
  // Default since the per-position kernels prefetch their epilogue operands and are chained by
  // programmatic dependent launch: the graph (cfg3 FFT stage 74.0k updates/s, cfg4 46.6k) beats
  // this sweep (49.5k / 44.0k). PFTG_PERSIST=1 selects the persistent sweeps.
  static const bool want = std::getenv("PFTG_PERSIST") != nullptr;
  return want && sizeof(R) == 4 && !band && !s.cfg.shuffled && !knobs().no_persist && (use_fft512(s) || use_fft256(s));
}

template <class R>
void launch_persistent_fft(pftg_solver& s) {
  int dev = 0, nsm = 0, coop = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  PFTG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  PFTG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) throw cuda_error("pftg: cooperative launch unsupported");
  const int W = (int)s.wr;
  const float2* tw = fft_twiddles<float>(W);
  float2* fr = static_cast<float2*>(s.frame);
  float2* pr = static_cast<float2*>(s.probe);
  float2* X = static_cast<float2*>(s.X);
  float2* X2 = static_cast<float2*>(s.X2);
  const float* d = static_cast<const float*>(s.d);
  long long ld = (long long)s.fc;
  const long long* offs = s.doffs;
  int npos = (int)s.npos;
  float scale = 1.0f / static_cast<float>((long long)W * W), beta = (float)s.cfg.beta, gamma = (float)s.cfg.gamma;
  unsigned* bar = s.bar;
  void* args[] = {&tw, &fr, &ld, &offs, &npos, &pr, &X, &X2, &d, &scale, &beta, &gamma, &bar};
  const bool blind = s.cfg.blind != 0;
  void* k = W == 512 ? (blind ? (void*)ke_epie_sweep<512, 1> : (void*)ke_epie_sweep<512, 0>)
                     : (blind ? (void*)ke_epie_sweep<256, 1> : (void*)ke_epie_sweep<256, 0>);
  PFTG_CUDA(cudaMemsetAsync(s.bar, 0, sizeof(unsigned), s.st));
  ProfScope prof(s.st, K_FFT_ROWS);
  PFTG_CUDA(cudaLaunchCooperativeKernel(k, dim3(nsm), dim3(256), args, 0, s.st));
}

// PFT-band stage, blind, list order, complex64 q = 8 plans with r = 9 and
// p = 32 / 64 (BASELINE configs[2] / [3]): the sweep as one cooperative
// persistent kernel (band_sweep.cuh) after the first position's forward rows
// pass. PFTG_NO_PERSIST=1 keeps the per-position graph.
template <class R>
bool persistent_band(const pftg_solver& s, bool band) {
  if (sizeof(R) != 4 || !band || !s.cfg.blind || s.cfg.shuffled || knobs().no_persist || !s.plan) return false;
  const pftg::Axis& a1 = s.plan->a1;
  const pftg::Axis& a2 = s.plan->a2;
  // the per-position graph of the axis-reordered kernels (eval_band.cu: kb_adj_rows, and
  // kb_cols for p = 64) is faster than this sweep of the streaming kernels' bodies
  if (!(knobs().eval_band_old & 8)) return false;
  return a1.q == 8 && a2.q == 8 && a1.r == 9 && a2.r == 9 && a1.p == a2.p && (a1.p == 32 || a1.p == 64) &&
         a1.n == a2.n && a1.mt == a2.mt;
}

template <class R, int Q, int RR, int P>
void launch_persistent_band(pftg_solver& s) {
  const PftDev<R>& pd = plan_dev<R>(*s.plan);
  PftDev<R> pc = pd;  // single-position cols strips (launch_fwd_cols' narrowing)
  while (pc.nb > 1 && (long long)((pc.M2 + pc.nb - 1) / pc.nb) < 148) pc.nb /= 2;
  BPar<R, Q, RR> bp;
  for (int l = 0; l <= Q / 2; ++l)
    for (int j = 0; j < RR; ++j) {
      bp.b1[l][j] = static_cast<R>(pd.hBv1[l * RR + j]);
      bp.b2[l][j] = static_cast<R>(pd.hBv2[l * RR + j]);
    }
  const size_t rows_sm = fast_rows_smem<R>(pd.n2, Q, RR, pd.M2, P) + 16 + adj_prefetch_smem<R>(pd.n2, Q);
  const size_t smem = std::max(rows_sm, cols_smem_bytes(pc));
  if (smem > 227 * 1024) throw std::invalid_argument("pftg: persistent band sweep does not fit shared memory");
  constexpr int S1 = P / 32 > 0 ? P / 32 : 1, RB = 10;
  auto k = kb_band_sweep<R, Q, RR, P, S1, RB>;
  PFTG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  PFTG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // the first position's forward rows pass (probe .* window 0) -> G
  const int vec0 = (s.offs[0] % 2 == 0) && (s.fc % 2 == 0) && (s.wc % 2 == 0);
  Src<R> src{static_cast<Cx<R>*>(s.frame), (long long)s.fc, 0, s.doffs, static_cast<Cx<R>*>(s.probe), vec0};
  launch_fwd_rows<R>(pd, src, static_cast<Cx<R>*>(s.G), 1, s.st);
  Cx<R>* frame = static_cast<Cx<R>*>(s.frame);
  Cx<R>* probe = static_cast<Cx<R>*>(s.probe);
  Cx<R>* G = static_cast<Cx<R>*>(s.G);
  Cx<R>* Gt = static_cast<Cx<R>*>(s.Gt);
  const R* dcrop = static_cast<const R*>(s.dcrop);
  long long ld = (long long)s.fc, mb = (long long)pd.M1 * pd.M2;
  const long long* offs = s.doffs;
  int npos = (int)s.npos, vec_base = (s.fc % 2 == 0) && (s.wc % 2 == 0);
  double beta = s.cfg.beta_pft, gamma = s.cfg.gamma_pft;
  unsigned* bar = s.bar;
  void* args[] = {(void*)&pd, &pc, &bp, &frame, &ld, &offs, &npos, &probe, &G, &Gt, &dcrop, &mb, &beta, &gamma,
                  &vec_base, &bar};
  PFTG_CUDA(cudaMemsetAsync(s.bar, 0, sizeof(unsigned), s.st));
  ProfScope prof(s.st, K_ADJ_ROWS);
  PFTG_CUDA(cudaLaunchCooperativeKernel((void*)k, dim3(nsm), dim3(kBandSweepThreads), args, smem, s.st));
}

template <class R>
void enqueue_sweep(pftg_solver& s, bool band) {
  if (persistent_fft<R>(s, band)) {
    if constexpr (sizeof(R) == 4) launch_persistent_fft<R>(s);
  } else if (persistent_band<R>(s, band)) {
    if constexpr (sizeof(R) == 4) {
      if (s.plan->a1.p == 32) launch_persistent_band<R, 8, 9, 32>(s);
      else launch_persistent_band<R, 8, 9, 64>(s);
    }
  } else {
    enqueue_positions<R>(s, band);
  }
  enqueue_tv<R>(s, band);
}

template <class R>
void enqueue_positions(pftg_solver& s, bool band) {
  s.fwd_ready = false;
  for (std::size_t t = 0; t < s.npos; ++t)
    enqueue_position<R>(s, s.order[t], band, t + 1 < s.npos ? (long long)s.order[t + 1] : -1);
  s.fwd_ready = false;
}

template <class R>
void enqueue_tv(pftg_solver& s, bool band) {
  if (s.cfg.tv_lambda_mag > 0.0 || s.cfg.tv_lambda_phase > 0.0) {
    // solver.cpp:264-279: step lambda * step_scale, step_scale = beta_pft (band) or beta (FFT)
    const double step = band ? s.cfg.beta_pft : s.cfg.beta;
    const dim3 grid((unsigned)((s.fc + 31) / 32), (unsigned)((s.fr + 7) / 8));
    k_tv<R><<<grid, dim3(32, 8), 0, s.st>>>(static_cast<const Cx<R>*>(s.frame), static_cast<Cx<R>*>(s.tv),
                                             (int)s.fr, (int)s.fc, (R)(s.cfg.tv_lambda_mag * step),
                                             (R)(s.cfg.tv_lambda_phase * step));
    PFTG_LAUNCH_CHECK();
    PFTG_CUDA(cudaMemcpyAsync(s.frame, s.tv, sizeof(Cx<R>) * s.fr * s.fc, cudaMemcpyDeviceToDevice, s.st));
  }
}

// out[j] = sum_k part[j * nstrips + k], k ascending (deterministic)
__global__ void k_sum_strips_pos(const double* __restrict__ part, int nstrips, int count, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  double s = 0.0;
  for (int k = 0; k < nstrips; ++k) s += part[(size_t)j * nstrips + k];
  out[j] = s;
}

template <class R>
double objective(pftg_solver& s) {
  // (1/N) sum_j (1/n) sum_k (|X_jk| - d_jk)^2  (Parseval form of solver.cpp:89-102)
  const int n1 = (int)s.wr, n2 = (int)s.wc;
  const long long n = (long long)n1 * n2;
  const bool f512 = sizeof(R) == 4 && use_fft512(s);
  const int strips = f512 ? 64 : fft_cols_strips<R>(n2);
  for (std::size_t c0 = 0; c0 < s.npos; c0 += s.eval_chunk) {
    const int nb = (int)std::min(s.eval_chunk, s.npos - c0);
    if constexpr (sizeof(R) == 4) {
      if (f512) {
        const float2* tw = fft_twiddles<float>(512);
        {
          ProfScope prof(s.st, K_FFT_ROWS);
          ke_rows512<4><<<dim3(32, nb), 256, 0, s.st>>>(static_cast<const float2*>(s.frame), (long long)s.fc,
                                                         s.doffs + c0, static_cast<const float2*>(s.probe), tw,
                                                         static_cast<float2*>(s.Xe));
        }
        ProfScope prof(s.st, K_FFT_COLS);
        ke_cols512_eval<<<dim3(64, nb), 512, 0, s.st>>>(static_cast<const float2*>(s.Xe),
                                                        static_cast<const float*>(s.d) + c0 * n, tw,
                                                        s.part + c0 * strips);
        PFTG_LAUNCH_CHECK();
        continue;
      }
    }
    RowSrc<R> src{static_cast<const Cx<R>*>(s.frame), (long long)s.fc, 0, s.doffs + c0,
                  static_cast<const Cx<R>*>(s.probe)};
    RowEpiArgs ep{};
    launch_fft_rows<R>(ROW_DIF_STORE, EPI_STORE, n1, n2, src, static_cast<Cx<R>*>(s.Xe), n, -1, 1.0, ep, nb, s.st);
    launch_fft_cols<R>(COL_EVAL, n1, n2, static_cast<Cx<R>*>(s.Xe), n, static_cast<const R*>(s.dperm) + c0 * n, n,
                       nullptr, 0, -1, s.part + c0 * strips, nb, s.st);
  }
  // per-position sums of the strip partials on the device (same strip order as the host
  // loop they replace): npos doubles cross PCIe per sweep instead of npos x strips
  Scratch psum(sizeof(double) * s.npos, s.st);
  k_sum_strips_pos<<<(unsigned)((s.npos + 127) / 128), 128, 0, s.st>>>(s.part, strips, (int)s.npos, psum.as<double>());
  PFTG_LAUNCH_CHECK();
  std::vector<double> h(s.npos);
  PFTG_CUDA(cudaMemcpyAsync(h.data(), psum.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s.st));
  PFTG_CUDA(cudaStreamSynchronize(s.st));
  double acc = 0.0;
  for (std::size_t j = 0; j < s.npos; ++j) acc += h[j] / static_cast<double>(n);
  return acc / static_cast<double>(s.npos);
}

template <class R>
void norm_finite(pftg_solver& s, const void* a, long long n, double* norm, bool* finite) {
  k_norm_finite<R><<<kRedBlocks, 256, 0, s.st>>>(static_cast<const Cx<R>*>(a), n, s.red);
  PFTG_LAUNCH_CHECK();
  std::vector<double> h(2 * kRedBlocks);
  PFTG_CUDA(cudaMemcpyAsync(h.data(), s.red, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s.st));
  PFTG_CUDA(cudaStreamSynchronize(s.st));
  double t = 0, bad = 0;
  for (int i = 0; i < kRedBlocks; ++i) {
    t += h[i];
    bad += h[kRedBlocks + i];
  }
  *norm = std::sqrt(t);
  *finite = bad == 0.0;
}

template <class R>
void run(pftg_solver& s, int max_sweeps) {
  const int total = s.cfg.pft_sweeps + s.cfg.fft_sweeps;
  int done = 0;
  const long long fn = (long long)s.fr * s.fc, pn = (long long)s.wr * s.wc;
  while (s.sweeps_run < total && (s.flags & 3) == 0 && (max_sweeps <= 0 || done < max_sweeps)) {
    const int sweep = s.sweeps_run + 1;
    const bool band = sweep <= s.cfg.pft_sweeps;
    const auto t0 = std::chrono::steady_clock::now();
    if (s.cfg.tol > 0.0)
      PFTG_CUDA(cudaMemcpyAsync(s.prev, s.frame, sizeof(Cx<R>) * fn, cudaMemcpyDeviceToDevice, s.st));
    if (s.cfg.shuffled) {
      // Fisher-Yates with explicit modulo draws (solver.cpp:164-169)
      for (std::size_t i = s.order.size(); i > 1; --i) {
        const std::size_t j = static_cast<std::size_t>(s.shuffle_rng() % i);
        std::swap(s.order[i - 1], s.order[j]);
      }
      enqueue_sweep<R>(s, band);
    } else if (persistent_fft<R>(s, band) || persistent_band<R>(s, band)) {
      enqueue_sweep<R>(s, band);  // cooperative launches (+ TV): nothing to capture
    } else {
      cudaGraphExec_t& g = s.graph[band ? 0 : 1];
      int* delta = s.graph_launches[band ? 0 : 1];
      if (!g) {
        int before[K_NUM], after[K_NUM];
        prof_launch_snapshot(before);
        cudaGraph_t graph;
        PFTG_CUDA(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue_sweep<R>(s, band);
        } catch (...) {
          cudaStreamEndCapture(s.st, &graph);
          throw;
        }
        PFTG_CUDA(cudaStreamEndCapture(s.st, &graph));
        PFTG_CUDA(cudaGraphInstantiate(&g, graph, 0));
        cudaGraphDestroy(graph);
        prof_launch_snapshot(after);
        for (int k = 0; k < K_NUM; ++k) delta[k] = after[k] - before[k];
      } else {
        prof_add_launches(delta);  // a replay launches every captured kernel again
      }
      PFTG_CUDA(cudaGraphLaunch(g, s.st));
    }
    PFTG_CUDA(cudaStreamSynchronize(s.st));
    s.sweeps_run = sweep;
    ++done;
    s.t_accum += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s.wall.push_back(s.t_accum);
    const auto t1 = std::chrono::steady_clock::now();
    const bool eval = s.cfg.objective_every <= 1 || (sweep % s.cfg.objective_every) == 0 || sweep == total;
    s.objective.push_back(eval ? objective<R>(s) : std::nan(""));
    double fnrm, pnrm;
    bool ffin, pfin;
    norm_finite<R>(s, s.frame, fn, &fnrm, &ffin);
    norm_finite<R>(s, s.probe, pn, &pnrm, &pfin);
    bool stop_tol = false;
    if (ffin && pfin && fnrm <= s.frame_guard && pnrm <= s.probe_guard && s.cfg.tol > 0.0) {
      double pv;
      bool pf;
      norm_finite<R>(s, s.prev, fn, &pv, &pf);
      if (pv == 0.0) {
        std::fprintf(stderr, "relative_change_below: zero reference norm, not stopping\n");
      } else {
        k_diff_norm<R><<<kRedBlocks, 256, 0, s.st>>>(static_cast<const Cx<R>*>(s.frame),
                                                     static_cast<const Cx<R>*>(s.prev), fn, s.red);
        PFTG_LAUNCH_CHECK();
        std::vector<double> h(kRedBlocks);
        PFTG_CUDA(cudaMemcpyAsync(h.data(), s.red, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s.st));
        PFTG_CUDA(cudaStreamSynchronize(s.st));
        double num = 0;
        for (double v : h) num += v;
        stop_tol = std::sqrt(num) / pv <= s.cfg.tol;
      }
    }
    // objective + guards are part of the reference's per-sweep cost (solver.cpp:286-299)
    s.t_accum += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    if (!ffin || !pfin || fnrm > s.frame_guard || pnrm > s.probe_guard) {
      s.flags |= 1;
      break;
    }
    if (stop_tol) {
      s.flags |= 2;
      break;
    }
  }
}

template <class R>
void create(pftg_solver& s, const void* frame, const void* probe, const int64_t* offsets, const void* d,
            const pftg_table* table) {
  const long long fn = (long long)s.fr * s.fc, pn = (long long)s.wr * s.wc;
  check_fft_len(s.wr);
  check_fft_len(s.wc);
  for (std::size_t j = 0; j < s.npos; ++j) {
    const long long r0 = offsets[2 * j], c0 = offsets[2 * j + 1];
    // The reference does not bounds-check offsets (scan.cpp:14-22); reading
    // out of the device frame would fault, so reject it here instead.
    if (r0 < 0 || c0 < 0 || r0 + (long long)s.wr > (long long)s.fr || c0 + (long long)s.wc > (long long)s.fc)
      throw std::out_of_range("scan: window outside the frame");
    s.offs.push_back(r0 * (long long)s.fc + c0);
  }
  s.order.resize(s.npos);
  std::iota(s.order.begin(), s.order.end(), std::size_t{0});
  s.shuffle_rng.seed(s.cfg.seed);
  PFTG_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
  PFTG_CUDA(cudaMalloc(&s.frame, sizeof(Cx<R>) * fn));
  PFTG_CUDA(cudaMalloc(&s.probe, sizeof(Cx<R>) * pn));
  PFTG_CUDA(cudaMemcpyAsync(s.frame, frame, sizeof(Cx<R>) * fn, cudaMemcpyHostToDevice, s.st));
  PFTG_CUDA(cudaMemcpyAsync(s.probe, probe, sizeof(Cx<R>) * pn, cudaMemcpyHostToDevice, s.st));
  if (s.cfg.tol > 0.0) PFTG_CUDA(cudaMalloc(&s.prev, sizeof(Cx<R>) * fn));
  if (s.cfg.tv_lambda_mag > 0.0 || s.cfg.tv_lambda_phase > 0.0) PFTG_CUDA(cudaMalloc(&s.tv, sizeof(Cx<R>) * fn));
  PFTG_CUDA(cudaMalloc(&s.d, sizeof(R) * pn * s.npos));
  // uploads are ordered on s.st ahead of the kernels that read them
  PFTG_CUDA(cudaMemcpyAsync(s.d, d, sizeof(R) * pn * s.npos, cudaMemcpyHostToDevice, s.st));
  PFTG_CUDA(cudaMalloc(&s.dperm, sizeof(R) * pn * s.npos));
  k_permute_d<R><<<148 * 16, 256, 0, s.st>>>(static_cast<const R*>(s.d), static_cast<R*>(s.dperm), (int)s.wr,
                                             (int)s.wc, ilog2((int)s.wr), ilog2((int)s.wc), (long long)s.npos);
  PFTG_LAUNCH_CHECK();
  PFTG_CUDA(cudaMalloc(&s.doffs, sizeof(long long) * std::max<std::size_t>(s.npos, 1)));
  PFTG_CUDA(cudaMemcpyAsync(s.doffs, s.offs.data(), sizeof(long long) * s.npos, cudaMemcpyHostToDevice, s.st));
  PFTG_CUDA(cudaStreamSynchronize(s.st));
  PFTG_CUDA(cudaMalloc(&s.X, sizeof(Cx<R>) * pn));
  PFTG_CUDA(cudaMalloc(&s.X2, sizeof(Cx<R>) * pn));
  // per-sweep objective: up to 512 MB of spectra per launch pair (fewer launch tails)
  s.eval_chunk = std::max<std::size_t>(1, std::min<std::size_t>(s.npos, (512ull << 20) / (sizeof(Cx<R>) * pn)));
  PFTG_CUDA(cudaMalloc(&s.Xe, sizeof(Cx<R>) * pn * s.eval_chunk));
  PFTG_CUDA(cudaMalloc(&s.part, sizeof(double) * std::max(64, fft_cols_strips<R>((int)s.wc)) *
                                    std::max<std::size_t>(s.npos, 1)));
  PFTG_CUDA(cudaMalloc(&s.red, sizeof(double) * 2 * kRedBlocks));
  PFTG_CUDA(cudaMalloc(&s.bar, sizeof(unsigned)));
  (void)fft_twiddles<R>((int)s.wr);
  (void)fft_twiddles<R>((int)s.wc);
  if (s.cfg.pft_sweeps > 0) {
    // solver.cpp:194-209
    const std::size_t mt1 = s.cfg.mt1 ? (std::size_t)s.cfg.mt1 : s.wr / 8;
    const std::size_t mt2 = s.cfg.mt2 ? (std::size_t)s.cfg.mt2 : s.wc / 8;
    const std::size_t p1 = s.cfg.p1 ? (std::size_t)s.cfg.p1 : mt1;
    const std::size_t p2 = s.cfg.p2 ? (std::size_t)s.cfg.p2 : mt2;
    if (!table) throw std::invalid_argument("hybrid_solve: band stage needs a scope table");
    s.plan = std::make_unique<pftg_plan>();
    s.plan->a1 = plan_1d(s.wr, mt1, p1, s.cfg.eps_pft, table->t);
    s.plan->a2 = plan_1d(s.wc, mt2, p2, s.cfg.eps_pft, table->t);
    const PftDev<R>& pd = plan_dev<R>(*s.plan);
    const long long mb = 4LL * mt1 * mt2;
    PFTG_CUDA(cudaMalloc(&s.dcrop, sizeof(R) * mb * s.npos));
    k_crop_real<R><<<148 * 16, 256, 0, s.st>>>(static_cast<const R*>(s.d), static_cast<R*>(s.dcrop), (int)s.wr,
                                               (int)s.wc, (int)mt1, (int)mt2, (long long)s.npos);
    PFTG_LAUNCH_CHECK();
    const std::size_t gsz = (std::size_t)pd.p1 * pd.r1 * pd.M2;
    PFTG_CUDA(cudaMalloc(&s.G, sizeof(Cx<R>) * gsz));
    PFTG_CUDA(cudaMalloc(&s.Gt, sizeof(Cx<R>) * gsz));
  }
  double fnrm, pnrm;
  bool f1, f2;
  norm_finite<R>(s, s.frame, fn, &fnrm, &f1);
  norm_finite<R>(s, s.probe, pn, &pnrm, &f2);
  // solver.cpp:227-228
  s.probe_guard = 1e6 * std::max(pnrm, 1e-300);
  s.frame_guard = 1e6 * std::max(fnrm, 1e-300);
}

template <class F>
int guarded(F&& f) {
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

}  // namespace

extern "C" {

int pftg_solver_create(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr, size_t wc,
                       const int64_t* offsets, size_t npos, const void* d, const pftg_solver_config* cfg,
                       const pftg_table* table, pftg_solver** out) {
  return guarded([&] {
    if (dtype != PFTG_C64 && dtype != PFTG_C128) throw std::invalid_argument("pftg: bad dtype");
    if (!cfg) throw std::invalid_argument("hybrid_solve: null config");
    if (cfg->pft_sweeps < 0 || cfg->fft_sweeps < 0) throw std::invalid_argument("hybrid_solve: negative sweep budget");
    if (npos == 0) throw std::invalid_argument("hybrid_solve: no scan positions");
    if (wr > fr || wc > fc) throw std::invalid_argument("hybrid_solve: window larger than frame");
    ensure_device();
    auto s = std::make_unique<pftg_solver>();
    s->dtype = dtype;
    s->fr = fr;
    s->fc = fc;
    s->wr = wr;
    s->wc = wc;
    s->npos = npos;
    s->cfg = *cfg;
    if (dtype == PFTG_C64) create<float>(*s, frame, probe, offsets, d, table);
    else create<double>(*s, frame, probe, offsets, d, table);
    *out = s.release();
  });
}

int pftg_solver_run(pftg_solver* s, int max_sweeps) {
  return guarded([&] {
    if (!s) throw std::invalid_argument("pftg: null solver");
    if (s->dtype == PFTG_C64) run<float>(*s, max_sweeps);
    else run<double>(*s, max_sweeps);
  });
}

int pftg_solver_trace(const pftg_solver* s, double* objective, double* wall_s, int* sweeps_run, int* flags) {
  return guarded([&] {
    if (!s) throw std::invalid_argument("pftg: null solver");
    for (std::size_t i = 0; i < s->objective.size(); ++i) {
      if (objective) objective[i] = s->objective[i];
      if (wall_s) wall_s[i] = s->wall[i];
    }
    if (sweeps_run) *sweeps_run = s->sweeps_run;
    if (flags) *flags = s->flags;
  });
}

int pftg_solver_result(const pftg_solver* s, void* frame, void* probe) {
  return guarded([&] {
    if (!s) throw std::invalid_argument("pftg: null solver");
    const std::size_t cs = s->dtype == PFTG_C64 ? 8 : 16;
    PFTG_CUDA(cudaStreamSynchronize(s->st));
    // the solver's work runs on its non-blocking stream: read back in stream order
    if (frame) PFTG_CUDA(cudaMemcpyAsync(frame, s->frame, cs * s->fr * s->fc, cudaMemcpyDeviceToHost, s->st));
    if (probe) PFTG_CUDA(cudaMemcpyAsync(probe, s->probe, cs * s->wr * s->wc, cudaMemcpyDeviceToHost, s->st));
    PFTG_CUDA(cudaStreamSynchronize(s->st));
  });
}

int pftg_solver_device_state(const pftg_solver* s, void** frame, void** probe) {
  return guarded([&] {
    if (!s) throw std::invalid_argument("pftg: null solver");
    if (frame) *frame = s->frame;
    if (probe) *probe = s->probe;
  });
}

void pftg_solver_free(pftg_solver* s) { delete s; }

}  // extern "C"
