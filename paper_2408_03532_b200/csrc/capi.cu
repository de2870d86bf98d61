// C-ABI implementation (include/pftg.h): plans, PFT operators, full FFTs,
// modulus projection, scan geometry, updates and the evaluator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pftg.h"
#include "eval_fft.cuh"
#include <thread>

#include "internal.hpp"

namespace pftg {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& m) { g_err = m; }

const Knobs& knobs() {
  static const Knobs k = [] {
    auto on = [](const char* n) { return std::getenv(n) != nullptr; };
    auto num = [](const char* n) {
      const char* v = std::getenv(n);
      return v ? std::atoi(v) : 0;
    };
    Knobs o{};
    o.no_pdl = on("PFTG_NO_PDL");
    o.no_tma = on("PFTG_NO_TMA");
    o.no_ws = on("PFTG_NO_WS");
    o.no_wide = on("PFTG_NO_WIDE");
    o.no_split = on("PFTG_NO_SPLIT");
    o.no_local_cols = on("PFTG_NO_LOCAL_COLS");
    o.eval_lanefft = on("PFTG_EVAL_LANEFFT");
    o.epie_lanefft = on("PFTG_EPIE_LANEFFT");
    o.tma_ns = num("PFTG_TMA_NS");
    o.cols_grid = num("PFTG_COLS_GRID");
    o.eval_chunk = num("PFTG_EVAL_CHUNK");
    o.eval_pchunk = num("PFTG_EVAL_PCHUNK");
    o.eval_one_stream = on("PFTG_EVAL_ONE_STREAM");
    o.eval_band_old = num("PFTG_EVAL_BAND_OLD");
    o.no_tile = on("PFTG_NO_TILE");
    o.force_tile = on("PFTG_TILE");
    o.host_chunk_mb = num("PFTG_HOST_CHUNK_MB");
    o.no_persist = on("PFTG_NO_PERSIST");
    o.no_prefetch = on("PFTG_NO_PREFETCH");
#ifdef PFTG_PROFILING
    o.debug_tma = num("PFTG_DEBUG_TMA");
    o.debug_ws = num("PFTG_DEBUG_WS");
    o.debug_adj = num("PFTG_DEBUG_ADJ");
    o.debug_cols = num("PFTG_DEBUG_COLS");
    o.debug_adjcols = num("PFTG_DEBUG_ADJCOLS");
    o.debug_wide_adj = on("PFTG_DEBUG_WIDE_ADJ");
#endif
    return o;
  }();
  return k;
}

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line, what);
  throw cuda_error(buf);
}

void ensure_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw cuda_error("pftg: no CUDA device available (this library has no CPU fallback)");
  }
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static bool checked[64] = {};
  if (dev < 64 && checked[dev]) return;
  std::lock_guard<std::mutex> lock(mu);
  int major = 0;
  PFTG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw cuda_error("pftg: built for sm_100a (B200); device has compute capability major " +
                                    std::to_string(major));
  // Scratch buffers come from the stream-ordered default pool; keep freed
  // memory cached instead of returning it to the driver at every sync.
  cudaMemPool_t pool;
  PFTG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  std::uint64_t keep = ~std::uint64_t(0);
  PFTG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  if (dev < 64) checked[dev] = true;
}

// One non-blocking side stream per device (fork / join with events; shared by
// concurrent callers, which only serializes their side work).
cudaStream_t side_stream() {
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  std::lock_guard<std::mutex> lock(mu);
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t s;
  PFTG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  streams.emplace(dev, s);
  return s;
}

void check_fft_len(std::size_t n) {
  if (n < 2 || n > 1024 || (n & (n - 1)) != 0)
    throw std::invalid_argument("pftg: GPU fft2 supports power-of-two sizes in [2, 1024], got " +
                                std::to_string(n));
}

// ---- per-kernel timing hook ----
namespace {
struct ProfState {
  std::mutex mu;
  bool on = false;
  int mode = 0;  // pftg_profile_mode: 0 events, 1 events + spin, 2 launch counts only
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  int launches[K_NUM] = {};
};
ProfState& prof() {
  static ProfState p;
  return p;
}
cudaEvent_t new_event() {
  cudaEvent_t e;
  PFTG_CUDA(cudaEventCreate(&e));
  return e;
}
bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}
}  // namespace

void prof_launch_snapshot(int* out) {
  ProfState& p = prof();
  std::lock_guard<std::mutex> lock(p.mu);
  std::copy(p.launches, p.launches + K_NUM, out);
}

void prof_add_launches(const int* delta) {
  ProfState& p = prof();
  std::lock_guard<std::mutex> lock(p.mu);
  for (int k = 0; k < K_NUM; ++k) p.launches[k] += delta[k];
}

// Profiling only: keeps the stream busy for ~ns so the start event and the
// timed launch are both enqueued before the GPU reaches them -- the event
// interval then measures the kernel, not host-side submission gaps.
__global__ void k_prof_spin(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

ProfScope::ProfScope(cudaStream_t s, int k) : kid(k), st(s) {
  ProfState& p = prof();
  {
    std::lock_guard<std::mutex> lock(p.mu);
    ++p.launches[k];
    if (!p.on || p.mode == 2) return;
  }
  if (capturing(st)) return;
  e0 = new_event();
  if (prof().mode == 1) k_prof_spin<<<1, 32, 0, st>>>(30000ull);
  PFTG_CUDA(cudaEventRecord(e0, st));
}

ProfScope::~ProfScope() {
  if (!e0) return;
  cudaEvent_t e1;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, st);
  ProfState& p = prof();
  std::lock_guard<std::mutex> lock(p.mu);
  p.ev.push_back({kid, {e0, e1}});
}

Scratch::Scratch(std::size_t bytes, cudaStream_t s) : st(s) {
  if (bytes == 0) bytes = 16;
  PFTG_CUDA(cudaMallocAsync(&p, bytes, s));
}
Scratch::~Scratch() {
  if (p) cudaFreeAsync(p, st);
}

namespace {

template <class T>
T* dev_upload(const std::vector<T>& h) {
  T* d = nullptr;
  PFTG_CUDA(cudaMalloc(&d, sizeof(T) * std::max<std::size_t>(h.size(), 1)));
  // Stream-ordered copy + synchronize: a plain cudaMemcpy from pageable memory
  // may return before the DMA lands, and the tables are then read by kernels on
  // non-blocking streams that do not order after the legacy stream.
  if (!h.empty()) {
    PFTG_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, cudaStreamPerThread));
    PFTG_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  }
  return d;
}

int ilog2_exact(std::size_t n) {
  int l = 0;
  while ((std::size_t(1) << l) < n) ++l;
  return l;
}

// Nonzero part of B[l][j] (pure real for even j, pure imaginary for odd j,
// minimax.cpp:326-330). Plans loaded from files must keep that structure.
template <class R>
std::vector<R> b_values(const Axis& a) {
  std::vector<R> v(a.q * a.r);
  for (std::size_t l = 0; l < a.q; ++l)
    for (int j = 0; j < a.r; ++j) {
      const cd b = a.B[l * a.r + j];
      const double zero_part = (j % 2 == 0) ? b.imag() : b.real();
      if (zero_part != 0.0)
        throw std::invalid_argument(
            "pftg: plan B must be real for even j and imaginary for odd j (minimax.cpp:326-330)");
      v[l * a.r + j] = static_cast<R>((j % 2 == 0) ? b.real() : b.imag());
    }
  return v;
}

template <class R>
std::vector<typename CT<R>::C> w_transposed(const Axis& a) {
  const std::size_t M = 2 * a.mt;
  std::vector<typename CT<R>::C> v(static_cast<std::size_t>(a.r) * M);
  for (int j = 0; j < a.r; ++j)
    for (std::size_t i = 0; i < M; ++i) {
      const cd w = a.W[i * a.r + j];
      v[j * M + i] = CT<R>::mk(static_cast<R>(w.real()), static_cast<R>(w.imag()));
    }
  return v;
}

template <class R>
std::vector<typename CT<R>::C> twiddles_host(std::size_t p) {
  std::vector<typename CT<R>::C> v(std::max<std::size_t>(p / 2, 1));
  for (std::size_t k = 0; k < p / 2; ++k) {
    const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(p);
    v[k] = CT<R>::mk(static_cast<R>(std::cos(a)), static_cast<R>(std::sin(a)));
  }
  return v;
}

void check_gpu_axis(const Axis& a, const char* which) {
  const bool pow2 = a.p >= 2 && (a.p & (a.p - 1)) == 0;
  if (!pow2 || a.p > 128)
    throw std::invalid_argument(std::string("pftg: GPU PFT needs power-of-two p in [2, 128] (axis ") + which +
                                ", p=" + std::to_string(a.p) + ")");
  if (a.r < 1 || a.r > 16)
    throw std::invalid_argument(std::string("pftg: GPU PFT supports 1 <= r <= 16 (axis ") + which + ")");
  if (a.n > (1u << 20)) throw std::invalid_argument("pftg: axis too long");
}

template <class R>
void upload(const pftg_plan& p, DevTables<R>& t, PftDev<R>& pd) {
  check_gpu_axis(p.a1, "1");
  check_gpu_axis(p.a2, "2");
  t.Bv1 = dev_upload(b_values<R>(p.a1));
  t.Bv2 = dev_upload(b_values<R>(p.a2));
  t.W1t = dev_upload(w_transposed<R>(p.a1));
  t.W2t = dev_upload(w_transposed<R>(p.a2));
  t.tw1 = dev_upload(twiddles_host<R>(p.a1.p));
  t.tw2 = dev_upload(twiddles_host<R>(p.a2.p));
  pd.n1 = static_cast<int>(p.a1.n);
  pd.n2 = static_cast<int>(p.a2.n);
  pd.p1 = static_cast<int>(p.a1.p);
  pd.p2 = static_cast<int>(p.a2.p);
  pd.q1 = static_cast<int>(p.a1.q);
  pd.q2 = static_cast<int>(p.a2.q);
  pd.mt1 = static_cast<int>(p.a1.mt);
  pd.mt2 = static_cast<int>(p.a2.mt);
  pd.r1 = p.a1.r;
  pd.r2 = p.a2.r;
  pd.M1 = 2 * pd.mt1;
  pd.M2 = 2 * pd.mt2;
  pd.lp1 = ilog2_exact(p.a1.p);
  pd.lp2 = ilog2_exact(p.a2.p);
  pd.Bv1 = t.Bv1;
  pd.Bv2 = t.Bv2;
  pd.W1t = t.W1t;
  pd.W2t = t.W2t;
  pd.tw1 = t.tw1;
  pd.tw2 = t.tw2;
  pd.nb = choose_nb(pd);
  if (p.hbv1.empty()) {
    p.hbv1 = b_values<double>(p.a1);
    p.hbv2 = b_values<double>(p.a2);
  }
  pd.hBv1 = p.hbv1.data();
  pd.hBv2 = p.hbv2.data();
}

template <class R>
void free_tables(DevTables<R>& t) {
  cudaFree(t.Bv1);
  cudaFree(t.Bv2);
  cudaFree(t.W1t);
  cudaFree(t.W2t);
  cudaFree(t.tw1);
  cudaFree(t.tw2);
  t = DevTables<R>{};
}

}  // namespace

namespace {
template <class R>
const PftDev<R>& plan_dev_impl(const pftg_plan& p, std::map<int, std::unique_ptr<DevPlan<R>>>& per_dev) {
  ensure_device();
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(p.mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    auto dp = std::make_unique<DevPlan<R>>();
    try {
      upload(p, dp->t, dp->pd);
    } catch (...) {
      free_tables(dp->t);
      throw;
    }
    it = per_dev.emplace(dev, std::move(dp)).first;
  }
  return it->second->pd;  // stable address: entries are never erased while the plan lives
}
}  // namespace

template <>
const PftDev<float>& plan_dev<float>(const pftg_plan& p) {
  return plan_dev_impl<float>(p, p.dev32);
}

template <>
const PftDev<double>& plan_dev<double>(const pftg_plan& p) {
  return plan_dev_impl<double>(p, p.dev64);
}

// ---------------------------------------------------------------- operators
namespace {

template <class R>
using Cx = typename CT<R>::C;

// 16-byte column pairs are safe: 16-byte aligned base, even row length and batch stride.
bool vec_ok(const void* p, long long ld, long long bstride) {
  return (reinterpret_cast<std::uintptr_t>(p) % 16 == 0) && ld % 2 == 0 && bstride % 2 == 0;
}

// Fields per chunk so the chunk's G workspace (~p1*r1*M2 complex per field)
// stays well inside L2 between the rows and cols passes.
// The batch is split into equal chunks (e.g. 100 fields -> 2 x 50, not 73 + 27) so
// every rows launch ends with a well-filled last round of tiles.
// 48 MB of G per chunk: with the evict-first hint on the streamed fields it
// stays L2-resident (126 MB L2). PFTG_CHUNK_MB overrides the budget (profiling).
template <class R>
std::size_t chunk_fields(const PftDev<R>& pd, std::size_t batch = 0) {
  const std::size_t g = sizeof(Cx<R>) * (std::size_t)pd.p1 * pd.r1 * pd.M2;
  std::size_t mb = 48;
  if (const char* e = std::getenv("PFTG_CHUNK_MB")) mb = std::max(1, std::atoi(e));
  std::size_t c = (mb << 20) / std::max<std::size_t>(g, 1);
  c = std::max<std::size_t>(1, std::min<std::size_t>(c, 65535));
  if (batch > c) {
    const std::size_t k = (batch + c - 1) / c;
    c = (batch + k - 1) / k;
  }
  return c;
}

template <class R>
void apply_dev(const pftg_plan* plan, const void* z, void* band, std::size_t batch, cudaStream_t st,
               std::size_t call_batch = 0) {
  const PftDev<R>& pd = plan_dev<R>(*plan);
  // the path is chosen on the caller's whole batch (host-buffer chunks included),
  // so a call gives bit-identical results through either entry point
  if (tile_path_ok(pd, call_batch ? call_batch : batch)) {  // small batches: >= p1 p2 CTAs per stage (pft_tile.cu)
    tile_apply<R>(pd, z, (long long)pd.n1 * pd.n2, band, (int)batch, st);
    return;
  }
  const std::size_t chunk = std::min(batch, chunk_fields(pd, batch));
  const std::size_t gsz = (std::size_t)g_field_elems<R>(pd);
  Scratch G(sizeof(Cx<R>) * gsz * chunk, st);
  const std::size_t nz = (std::size_t)pd.n1 * pd.n2, nb = (std::size_t)pd.M1 * pd.M2;
  for (std::size_t b0 = 0; b0 < batch; b0 += chunk) {
    const int nbat = static_cast<int>(std::min(chunk, batch - b0));
    Src<R> src{static_cast<const Cx<R>*>(z) + b0 * nz, pd.n2, (long long)nz, nullptr, nullptr,
               vec_ok(z, pd.n2, nz)};
    const bool strip = launch_fwd_rows<R>(pd, src, G.as<Cx<R>>(), nbat, st, vec_ok(band, pd.M2, nb));
    launch_fwd_cols<R>(pd, 0, G.as<Cx<R>>(), static_cast<Cx<R>*>(band) + b0 * nb, nullptr, 0, nullptr, nullptr,
                       nbat, st, strip);
  }
}

template <class R>
void adjoint_dev(const pftg_plan* plan, const void* band, void* z, std::size_t batch, cudaStream_t st,
                 std::size_t call_batch = 0) {
  const PftDev<R>& pd = plan_dev<R>(*plan);
  if (tile_path_ok(pd, call_batch ? call_batch : batch)) {
    tile_adjoint<R>(pd, band, z, (long long)pd.n1 * pd.n2, (int)batch, st);
    return;
  }
  const std::size_t chunk = std::min(batch, chunk_fields(pd, batch));
  const std::size_t gsz = (std::size_t)pd.p1 * pd.r1 * pd.M2;
  Scratch G(sizeof(Cx<R>) * gsz * chunk, st);
  const std::size_t nz = (std::size_t)pd.n1 * pd.n2, nb = (std::size_t)pd.M1 * pd.M2;
  for (std::size_t b0 = 0; b0 < batch; b0 += chunk) {
    const int nbat = static_cast<int>(std::min(chunk, batch - b0));
    launch_adj_cols<R>(pd, static_cast<const Cx<R>*>(band) + b0 * nb, G.as<Cx<R>>(), nbat, st);
    EpiArgs ep{};
    ep.out = static_cast<Cx<R>*>(z) + b0 * nz;
    ep.vec_ok = vec_ok(z, pd.n2, nz);
    launch_adj_rows<R>(pd, 0, G.as<Cx<R>>(), ep, nbat, st);
  }
}

template <class R>
void band_residual_dev(const pftg_plan* plan, const void* exit_wave, const void* dcrop, void* out,
                       std::size_t batch, cudaStream_t st) {
  const PftDev<R>& pd = plan_dev<R>(*plan);
  const std::size_t chunk = std::min(batch, chunk_fields(pd, batch));
  const std::size_t gsz = (std::size_t)pd.p1 * pd.r1 * pd.M2;
  Scratch G(sizeof(Cx<R>) * gsz * chunk, st), Gt(sizeof(Cx<R>) * gsz * chunk, st);
  const std::size_t nz = (std::size_t)pd.n1 * pd.n2, nb = (std::size_t)pd.M1 * pd.M2;
  for (std::size_t b0 = 0; b0 < batch; b0 += chunk) {
    const int nbat = static_cast<int>(std::min(chunk, batch - b0));
    Src<R> src{static_cast<const Cx<R>*>(exit_wave) + b0 * nz, pd.n2, (long long)nz, nullptr, nullptr,
               vec_ok(exit_wave, pd.n2, nz)};
    launch_fwd_rows<R>(pd, src, G.as<Cx<R>>(), nbat, st);
    launch_fwd_cols<R>(pd, 1, G.as<Cx<R>>(), nullptr, static_cast<const R*>(dcrop) + b0 * nb, (long long)nb,
                       Gt.as<Cx<R>>(), nullptr, nbat, st);
    EpiArgs ep{};
    ep.out = static_cast<Cx<R>*>(out) + b0 * nz;
    ep.vec_ok = vec_ok(out, pd.n2, nz);
    launch_adj_rows<R>(pd, 0, Gt.as<Cx<R>>(), ep, nbat, st);
  }
}

// Host-buffer variants: a three-stage ring. One stream per stage -- H2D copy,
// compute, D2H copy -- and NSLOT device buffer sets; chunk i uses slot i % NSLOT.
// The H2D stream never waits for a D2H (it only waits until the compute of
// chunk i - NSLOT has consumed the slot's input), so the H2D copy engine runs
// back to back over the whole batch while the D2H engine trails it by one
// chunk: the call costs max(H2D bytes, D2H bytes) / PCIe rate plus one chunk
// of fill and drain. (Two ping-pong streams each serialising H2D -> compute
// -> D2H left one direction idle whenever the other stream's copy ran long.)
// Events are recorded in issue order, so a wait on slot k's event always
// refers to chunk i - NSLOT (never-recorded events count as complete).
constexpr int NSLOT = 3;
struct HostRing {
  cudaStream_t s[3];  // 0: H2D, 1: compute, 2: D2H
  cudaEvent_t h2d[NSLOT], comp[NSLOT], d2h[NSLOT];
};
HostRing& host_ring() {
  // per (host thread, device), created once
  thread_local HostRing rings[64];
  thread_local bool made[64] = {};
  int dev = 0;
  PFTG_CUDA(cudaGetDevice(&dev));
  if (dev >= 64) throw std::runtime_error("pftg: device index out of range");
  HostRing& r = rings[dev];
  if (!made[dev]) {
    for (auto& s : r.s) PFTG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int k = 0; k < NSLOT; ++k) {
      PFTG_CUDA(cudaEventCreateWithFlags(&r.h2d[k], cudaEventDisableTiming));
      PFTG_CUDA(cudaEventCreateWithFlags(&r.comp[k], cudaEventDisableTiming));
      PFTG_CUDA(cudaEventCreateWithFlags(&r.d2h[k], cudaEventDisableTiming));
    }
    made[dev] = true;
  }
  return r;
}

// in(slot, b0, m, st): H2D of chunk [b0, b0 + m); op(slot, m, st): compute;
// out(slot, b0, m, st): D2H. Device buffers come from the stream-ordered pool
// on the compute stream (alloc(slot)); the copy streams are forked from it.
template <class In, class Op, class Out>
void host_ring_run(std::size_t batch, std::size_t chunk, In&& in, Op&& op, Out&& out) {
  HostRing& r = host_ring();
  cudaEvent_t fork = r.comp[0];
  PFTG_CUDA(cudaEventRecord(fork, r.s[1]));  // buffers allocated on s[1] before this point
  PFTG_CUDA(cudaStreamWaitEvent(r.s[0], fork));
  PFTG_CUDA(cudaStreamWaitEvent(r.s[2], fork));
  // the first chunks ramp up (chunk/4, chunk/2, chunk, ...): the D2H engine,
  // the busier direction (band + back-projection), starts after a short H2D
  int k = 0, i = 0;
  for (std::size_t b0 = 0; b0 < batch; ++i, k = (k + 1) % NSLOT) {
    const std::size_t c = i == 0 ? std::max<std::size_t>(1, chunk / 4) : i == 1 ? std::max<std::size_t>(1, chunk / 2)
                                                                              : chunk;
    const std::size_t m = std::min(c, batch - b0);
    if (i >= NSLOT) PFTG_CUDA(cudaStreamWaitEvent(r.s[0], r.comp[k]));  // slot input consumed
    in(k, b0, m, r.s[0]);
    PFTG_CUDA(cudaEventRecord(r.h2d[k], r.s[0]));
    PFTG_CUDA(cudaStreamWaitEvent(r.s[1], r.h2d[k]));
    if (i >= NSLOT) PFTG_CUDA(cudaStreamWaitEvent(r.s[1], r.d2h[k]));  // slot outputs drained
    op(k, m, r.s[1]);
    PFTG_CUDA(cudaEventRecord(r.comp[k], r.s[1]));
    PFTG_CUDA(cudaStreamWaitEvent(r.s[2], r.comp[k]));
    out(k, b0, m, r.s[2]);
    PFTG_CUDA(cudaEventRecord(r.d2h[k], r.s[2]));
    b0 += m;
  }
  // join: the buffers are released on the compute stream after the last copies
  PFTG_CUDA(cudaEventRecord(r.h2d[0], r.s[0]));
  PFTG_CUDA(cudaStreamWaitEvent(r.s[1], r.h2d[0]));
  PFTG_CUDA(cudaEventRecord(r.d2h[0], r.s[2]));
  PFTG_CUDA(cudaStreamWaitEvent(r.s[1], r.d2h[0]));
}

template <class R, class Op>
void host_pipeline(std::size_t batch, std::size_t in_elems, std::size_t out_elems, const void* in, void* out,
                   std::size_t chunk, Op&& op) {
  using C = Cx<R>;
  HostRing& r = host_ring();
  {
    std::vector<std::unique_ptr<Scratch>> bufs;
    C *din[NSLOT], *dout[NSLOT];
    for (int k = 0; k < NSLOT; ++k) {
      bufs.emplace_back(new Scratch(sizeof(C) * in_elems * chunk, r.s[1]));
      din[k] = bufs.back()->as<C>();
      bufs.emplace_back(new Scratch(sizeof(C) * out_elems * chunk, r.s[1]));
      dout[k] = bufs.back()->as<C>();
    }
    host_ring_run(
        batch, chunk,
        [&](int k, std::size_t b0, std::size_t m, cudaStream_t s) {
          PFTG_CUDA(cudaMemcpyAsync(din[k], static_cast<const C*>(in) + b0 * in_elems, sizeof(C) * in_elems * m,
                                    cudaMemcpyHostToDevice, s));
        },
        [&](int k, std::size_t m, cudaStream_t s) { op(din[k], dout[k], m, s); },
        [&](int k, std::size_t b0, std::size_t m, cudaStream_t s) {
          PFTG_CUDA(cudaMemcpyAsync(static_cast<C*>(out) + b0 * out_elems, dout[k], sizeof(C) * out_elems * m,
                                    cudaMemcpyDeviceToHost, s));
        });
  }
  PFTG_CUDA(cudaStreamSynchronize(r.s[1]));
}

std::size_t host_chunk(std::size_t batch, std::size_t bytes_per_field) {
  // ~32 MiB per copy: concurrent H2D + D2H run at ~49.7 GB/s each from 16-32 MiB
  // copies on (48.3 at 8 MiB, tools/pcie_probe.cu); the ramped first chunks
  // keep the pipeline fill short.
  const std::size_t mb = knobs().host_chunk_mb > 0 ? (std::size_t)knobs().host_chunk_mb : 32;
  std::size_t c = (mb << 20) / std::max<std::size_t>(bytes_per_field, 1);
  c = std::max<std::size_t>(1, c);
  return std::min(c, std::max<std::size_t>(1, (batch + 1) / 2));
}

// ---- full transforms ----
template <class R>
void fft2_dev(const void* z, void* out, std::size_t rows, std::size_t cols, std::size_t batch, int inverse,
              cudaStream_t st) {
  check_fft_len(rows);
  check_fft_len(cols);
  const int n1 = (int)rows, n2 = (int)cols;
  const long long n = (long long)n1 * n2;
  const int sign = inverse ? +1 : -1;
  const double scale = inverse ? 1.0 / static_cast<double>(n) : 1.0;
  RowSrc<R> src{static_cast<const Cx<R>*>(z), n2, n, nullptr, nullptr};
  RowEpiArgs ep{};
  launch_fft_rows<R>(ROW_DIT_NATURAL, EPI_STORE, n1, n2, src, static_cast<Cx<R>*>(out), n, sign, scale, ep,
                     (int)batch, st);
  launch_fft_cols<R>(COL_NATURAL, n1, n2, static_cast<Cx<R>*>(out), n, nullptr, 0, nullptr, 0, sign, nullptr,
                     (int)batch, st);
}

template <class R>
void project_modulus_dev(const void* exit_wave, const void* d, void* out, std::size_t rows, std::size_t cols,
                         std::size_t batch, cudaStream_t st) {
  check_fft_len(rows);
  check_fft_len(cols);
  const int n1 = (int)rows, n2 = (int)cols;
  const long long n = (long long)n1 * n2;
  Scratch X(sizeof(Cx<R>) * n * batch, st);
  RowSrc<R> src{static_cast<const Cx<R>*>(exit_wave), n2, n, nullptr, nullptr};
  RowEpiArgs ep{};
  launch_fft_rows<R>(ROW_DIF_STORE, EPI_STORE, n1, n2, src, X.as<Cx<R>>(), n, -1, 1.0, ep, (int)batch, st);
  launch_fft_cols<R>(COL_PROJECT, n1, n2, X.as<Cx<R>>(), n, static_cast<const R*>(d), n, nullptr, 1, -1, nullptr,
                     (int)batch, st);
  ep.out = out;
  ep.out_bstride = n;
  launch_fft_rows<R>(ROW_DIT_PROJ, EPI_STORE, n1, n2, src, X.as<Cx<R>>(), n, +1, 1.0 / static_cast<double>(n),
                     ep, (int)batch, st);
}

// ---- elementwise kernels ----
template <class C>
__global__ void k_window_slice(const C* __restrict__ frame, long long fc, C* __restrict__ out, int wr, int wc,
                               const long long* __restrict__ offs, int npos) {
  const long long per = (long long)wr * wc;
  const long long tot = per * npos;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const long long j = i / per;
    const int rem = (int)(i % per);
    const int r = rem / wc, c = rem % wc;
    out[i] = frame[offs[j] + (long long)r * fc + c];
  }
}

template <class C>
__global__ void k_set_window(C* __restrict__ frame, long long fc, const C* __restrict__ patch, int wr, int wc,
                             long long off) {
  const long long tot = (long long)wr * wc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / wc), c = (int)(i % wc);
    frame[off + (long long)r * fc + c] = patch[i];
  }
}

// mode 0: zj -= s conj(P) (P zj - proj); mode 1: P -= s conj(zj) (P zj - proj)
template <class C>
__global__ void k_update(C* __restrict__ a, const C* __restrict__ b, const C* __restrict__ proj, long long n,
                         double s, int mode) {
  using R = typename RT<C>::R;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const C zj = mode == 0 ? a[i] : b[i];
    const C pr = mode == 0 ? b[i] : a[i];
    const C resid = csub(cmul(pr, zj), proj[i]);
    const C g = mode == 0 ? cmulc(pr, resid) : cmulc(zj, resid);
    C v = a[i];
    v.x -= (R)s * g.x;
    v.y -= (R)s * g.y;
    a[i] = v;
  }
}

template <class R>
__global__ void k_crop(const R* __restrict__ spec, R* __restrict__ out, int rows, int cols, int mt1, int mt2,
                       long long batch) {
  const long long M = 4LL * mt1 * mt2;
  const long long tot = M * batch;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / M;
    const int rem = (int)(i % M);
    const int a = rem / (2 * mt2), b = rem % (2 * mt2);
    const int r = mod_nonneg(a - mt1, rows), c = mod_nonneg(b - mt2, cols);
    out[i] = spec[f * rows * cols + (long long)r * cols + c];
  }
}

// The reference does not bounds-check scan offsets (scan.cpp:14-22); on the
// device an out-of-frame window would be an illegal access that leaves the
// CUDA context unusable, so every window is checked (std::out_of_range).
void check_window(long long r0, long long c0, std::size_t wr, std::size_t wc, std::size_t fr, std::size_t fc) {
  if (r0 < 0 || c0 < 0 || r0 + (long long)wr > (long long)fr || c0 + (long long)wc > (long long)fc)
    throw std::out_of_range("scan: window (" + std::to_string(r0) + ", " + std::to_string(c0) + ") of " +
                            std::to_string(wr) + " x " + std::to_string(wc) + " outside the " + std::to_string(fr) +
                            " x " + std::to_string(fc) + " frame");
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 32));
}

// ---- evaluator ----
// out[j] = sum_k part[j * nstrips + k], k ascending (deterministic)
__global__ void k_sum_strips(const double* __restrict__ part, int nstrips, int count, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  double s = 0.0;
  for (int k = 0; k < nstrips; ++k) s += part[(size_t)j * nstrips + k];
  out[j] = s;
}

template <class R>
void evaluate_dev(const void* frame, std::size_t fr, std::size_t fc, const void* probe, std::size_t wr,
                  std::size_t wc, const int64_t* offsets, std::size_t npos, std::size_t pb, std::size_t pe,
                  const void* d, const pftg_plan* plan, const void* dcrop, double* fft_sum, double* band_sum,
                  cudaStream_t st) {
  check_fft_len(wr);
  check_fft_len(wc);
  if (pb > pe || pe > npos) throw std::out_of_range("scan: position index out of range");
  const int n1 = (int)wr, n2 = (int)wc;
  const long long n = (long long)n1 * n2;
  const std::size_t count = pe - pb;
  std::vector<long long> offs(count);
  for (std::size_t j = 0; j < count; ++j) {
    check_window(offsets[2 * (pb + j)], offsets[2 * (pb + j) + 1], wr, wc, fr, fc);
    offs[j] = offsets[2 * (pb + j)] * (long long)fc + offsets[2 * (pb + j) + 1];
  }
  const PftDev<R>* pd = plan ? &plan_dev<R>(*plan) : nullptr;
  if (pd && (pd->n1 != n1 || pd->n2 != n2))
    throw std::invalid_argument("band_residual: plan does not match the window shape");
  // spectra per chunk: up to 4 GB (all 1600 positions of configs[4] in one pair of
  // launches; B200 has the HBM for it): fewer, longer launches -- 512 MB chunks 4.70 ms,
  // 1.6 GB 4.62 ms, one chunk 4.58 ms per 1600 positions; equal chunks beyond that
  std::size_t chunk = std::max<std::size_t>(1, (4ull << 30) / (sizeof(Cx<R>) * n));
  if (knobs().eval_chunk > 0) chunk = (std::size_t)knobs().eval_chunk;
  if (count > chunk) chunk = (count + (count + chunk - 1) / chunk - 1) / ((count + chunk - 1) / chunk);
  chunk = std::max<std::size_t>(1, std::min<std::size_t>(count, chunk));
  Scratch doffs(sizeof(long long) * std::max<std::size_t>(count, 1), st);
  if (count) PFTG_CUDA(cudaMemcpyAsync(doffs.p, offs.data(), sizeof(long long) * count, cudaMemcpyHostToDevice, st));
  Scratch X(sizeof(Cx<R>) * n * chunk, st);
  // complex64 512 x 512 windows (BASELINE configs[4]): radix-8 register FFT kernels (eval_fft.cuh)
  const bool fast512 = sizeof(R) == 4 && n1 == 512 && n2 == 512 && !knobs().eval_lanefft;
  const int nstrips = fast512 ? 64 : fft_cols_strips<R>(n2);
  Scratch part(sizeof(double) * nstrips * std::max<std::size_t>(count, 1), st);
  std::unique_ptr<Scratch> G, bpart;
  int bstrips = 0;
  // the band chain's own chunk: more positions per persistent rows launch
  // (fewer tail rounds, fewer launches) than the spectra budget allows the FFT part
  // (up to 1 GB of G: cfg5's 1600 positions in one pair of launches)
  std::size_t pchunk = 1;
  if (pd) {
    const std::size_t gpos = sizeof(Cx<R>) * (std::size_t)pd->p1 * pd->r1 * pd->M2;
    pchunk = knobs().eval_pchunk > 0 ? (std::size_t)knobs().eval_pchunk : std::max<std::size_t>(1, (1ull << 30) / gpos);
    if (count > pchunk) pchunk = (count + (count + pchunk - 1) / pchunk - 1) / ((count + pchunk - 1) / pchunk);
    pchunk = std::min<std::size_t>(std::max<std::size_t>(count, 1), pchunk);
  }
  // q = 8, r = 9 complex64 plans: axis-2-first band chain (eval_band.cu); either
  // kernel can be swapped for the batched one (same G layout) with PFTG_EVAL_BAND_OLD
  bool eb_rows = false, eb_cols = false;
  if constexpr (sizeof(R) == 4) {
    if (pd) {
      const bool al = (reinterpret_cast<uintptr_t>(dcrop) & 15) == 0 && (reinterpret_cast<uintptr_t>(frame) & 7) == 0 &&
                      (reinterpret_cast<uintptr_t>(probe) & 7) == 0;
      eb_rows = al && eval_band_rows_ok(*pd) && !(knobs().eval_band_old & 1);
      eb_cols = al && eval_band_cols_ok(*pd) && !(knobs().eval_band_old & 2);
    }
  }
  if (pd) {
    G.reset(new Scratch(sizeof(Cx<R>) * (std::size_t)pd->p1 * pd->r1 * pd->M2 * pchunk, st));
    bstrips = eb_cols ? pd->M2 / 8 : cols_strips<R>(*pd);
    bpart.reset(new Scratch(sizeof(double) * bstrips * std::max<std::size_t>(count, 1), st));
  }
  // The full-FFT residual and the PFT band residual are independent: the band
  // chain runs on a side stream (forked / joined with events) so its kernels
  // fill the SMs the FFT kernels leave idle at chunk boundaries.
  cudaStream_t sb = st;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (pd && count && !knobs().eval_one_stream && !capturing(st)) {
    sb = side_stream();
    PFTG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    PFTG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    PFTG_CUDA(cudaEventRecord(ev_fork, st));
    PFTG_CUDA(cudaStreamWaitEvent(sb, ev_fork, 0));
  }
  for (std::size_t c0 = 0; c0 < count; c0 += chunk) {
    const int nb = (int)std::min(chunk, count - c0);
    const long long* o = doffs.as<long long>() + c0;
    // full-FFT objective: rows (natural input, bitrev-gather + DIT) ...
    RowSrc<R> src{static_cast<const Cx<R>*>(frame), (long long)fc, 0, o, static_cast<const Cx<R>*>(probe)};
    RowEpiArgs ep{};
    if constexpr (sizeof(R) == 4) {
      if (fast512) {
        const float2* tw = fft_twiddles<float>(512);
        {
          ProfScope prof(st, K_FFT_ROWS);
          // rows per 64-thread group: 8 (4: 4.58 ms, 8 / 16: 4.56 ms, 2: 4.68, 32: 4.94 per 1600 positions)
          ke_rows512<8><<<dim3(512 / (4 * 8), nb), 256, 0, st>>>(static_cast<const float2*>(frame), (long long)fc, o,
                                                                 static_cast<const float2*>(probe), tw,
                                                                 X.as<float2>());
          PFTG_LAUNCH_CHECK();
        }
        {
          ProfScope prof(st, K_FFT_COLS);
          ke_cols512_eval<<<dim3(64, nb), 512, 0, st>>>(X.as<float2>(), static_cast<const float*>(d) + (pb + c0) * n,
                                                        tw, part.as<double>() + c0 * nstrips);
          PFTG_LAUNCH_CHECK();
        }
      }
    }
    if (!fast512) {
      // natural-order spectrum (bit-reversed gathers stay on-chip) so the measured
      // magnitudes are read as coalesced strips
      launch_fft_rows<R>(ROW_DIT_NATURAL, EPI_STORE, n1, n2, src, X.as<Cx<R>>(), n, -1, 1.0, ep, nb, st);
      launch_fft_cols<R>(COL_EVAL_NAT, n1, n2, X.as<Cx<R>>(), n, static_cast<const R*>(d) + (pb + c0) * n, n,
                         nullptr, 0, -1, part.as<double>() + c0 * nstrips, nb, st);
    }
  }
  for (std::size_t c0 = 0; pd && c0 < count; c0 += pchunk) {
    const int nb = (int)std::min(pchunk, count - c0);
    const long long* o = doffs.as<long long>() + c0;
    bool evec = vec_ok(frame, (long long)fc, 0) && vec_ok(probe, n2, 0);
    for (std::size_t j = c0; j < c0 + nb; ++j) evec = evec && (offs[j] % 2 == 0);
    Src<R> s2{static_cast<const Cx<R>*>(frame), (long long)fc, 0, o, static_cast<const Cx<R>*>(probe), evec};
    const long long mb = (long long)pd->M1 * pd->M2;
    const R* dcp = static_cast<const R*>(dcrop) + (pb + c0) * mb;
    double* bp = bpart->as<double>() + c0 * bstrips;
    if constexpr (sizeof(R) == 4) {
      if (eb_rows)
        launch_eval_band_rows(*pd, static_cast<const float2*>(frame), (long long)fc, 0, o,
                              static_cast<const float2*>(probe), G->as<float2>(), nb, sb);
    }
    if (!eb_rows) launch_fwd_rows<R>(*pd, s2, G->as<Cx<R>>(), nb, sb);
    if constexpr (sizeof(R) == 4) {
      if (eb_cols) launch_eval_band_cols(*pd, 8, G->as<float2>(), nullptr, dcp, mb, nullptr, bp, nb, sb);
    }
    if (!eb_cols) launch_fwd_cols<R>(*pd, 2, G->as<Cx<R>>(), nullptr, dcp, mb, nullptr, bp, nb, sb);
  }
  if (ev_fork) {
    PFTG_CUDA(cudaEventRecord(ev_join, sb));
    PFTG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));  // scratch frees and the D2H below are ordered after the band chain
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
  }
  // per-position sums of the strip partials on the device (fixed strip order), so
  // only 2 x count doubles cross PCIe instead of the ~1 MB of per-strip partials
  Scratch psum(sizeof(double) * 2 * std::max<std::size_t>(count, 1), st);
  if (count) {
    k_sum_strips<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(part.as<double>(), nstrips, (int)count,
                                                                 psum.as<double>());
    if (pd)
      k_sum_strips<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(bpart->as<double>(), bstrips, (int)count,
                                                                   psum.as<double>() + count);
    PFTG_LAUNCH_CHECK();
  }
  std::vector<double> h(2 * count);
  if (count)
    PFTG_CUDA(cudaMemcpyAsync(h.data(), psum.p, sizeof(double) * (pd ? 2 : 1) * count, cudaMemcpyDeviceToHost, st));
  PFTG_CUDA(cudaStreamSynchronize(st));
  // (1/n) sum_k (|X_k| - d_k)^2 = ||x - P_M(x)||^2 by Parseval (solver.cpp:89-102)
  double s = 0.0;
  for (std::size_t j = 0; j < count; ++j) s += h[j] / static_cast<double>(n);
  *fft_sum = s;
  if (pd && band_sum) {
    double sb = 0.0;
    for (std::size_t j = 0; j < count; ++j) sb += h[count + j];
    *band_sum = sb;
  }
}

}  // namespace
}  // namespace pftg

pftg_plan::~pftg_plan() {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  for (auto& e : dev32) {
    cudaSetDevice(e.first);
    pftg::free_tables(e.second->t);
  }
  for (auto& e : dev64) {
    cudaSetDevice(e.first);
    pftg::free_tables(e.second->t);
  }
  cudaSetDevice(cur);
}

// ------------------------------------------------------------------ C ABI
using namespace pftg;

namespace {

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

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void check_dtype(int dtype) {
  if (dtype != PFTG_C64 && dtype != PFTG_C128) throw std::invalid_argument("pftg: dtype must be PFTG_C64 or PFTG_C128");
}

void check_plan(const pftg_plan* p) {
  if (!p) throw std::invalid_argument("pftg: null plan");
}

}  // namespace

extern "C" {

int pftg_version(void) { return 2; }

int pftg_profile_begin(void) {
  return guarded([&] {
    ProfState& p = prof();
    std::lock_guard<std::mutex> lock(p.mu);
    for (auto& e : p.ev) {
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    p.ev.clear();
    std::fill(p.launches, p.launches + K_NUM, 0);
    p.on = true;
  });
}

int pftg_profile_mode(int mode) {
  return guarded([&] {
    if (mode < 0 || mode > 2) throw std::invalid_argument("pftg_profile_mode: mode must be 0, 1 or 2");
    ProfState& p = prof();
    std::lock_guard<std::mutex> lock(p.mu);
    p.mode = mode;
  });
}

int pftg_profile_end(double* ms, int* count, int* launches) {
  return guarded([&] {
    ProfState& p = prof();
    std::lock_guard<std::mutex> lock(p.mu);
    p.on = false;
    for (int k = 0; k < K_NUM; ++k) {
      ms[k] = 0.0;
      count[k] = 0;
      if (launches) launches[k] = p.launches[k];
    }
    for (auto& e : p.ev) {
      PFTG_CUDA(cudaEventSynchronize(e.second.second));
      float t = 0.f;
      PFTG_CUDA(cudaEventElapsedTime(&t, e.second.first, e.second.second));
      ms[e.first] += t;
      count[e.first] += 1;
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    p.ev.clear();
  });
}
const char* pftg_last_error(void) { return g_err.c_str(); }

int pftg_device_ok(void) {
  try {
    ensure_device();
    return 1;
  } catch (...) {
    return 0;
  }
}

int pftg_table_load(const char* path, pftg_table** out) {
  return guarded([&] {
    auto t = std::make_unique<pftg_table>();
    t->t = table_load(path);
    *out = t.release();
  });
}

void pftg_table_free(pftg_table* t) { delete t; }

int pftg_table_min_degree(const pftg_table* t, double eps, double target, int* r_out) {
  return guarded([&] { *r_out = table_min_degree(t->t, eps, target); });
}

int pftg_best_approx(int r, double xi, double* coeff, double* achieved) {
  return guarded([&] {
    if (!coeff) throw std::invalid_argument("pftg_best_approx: null output");
    double e = 0.0;
    const std::vector<cd> w = best_approx_own(r, xi, &e);
    std::memcpy(coeff, w.data(), w.size() * sizeof(cd));
    if (achieved) *achieved = e;
  });
}

int pftg_table_compute(const double* eps, int neps, int max_r, pftg_table** out) {
  return guarded([&] {
    if (!out || (neps > 0 && !eps)) throw std::invalid_argument("pftg_table_compute: null argument");
    auto t = std::make_unique<pftg_table>();
    t->t = table_compute(std::vector<double>(eps, eps + std::max(neps, 0)), max_r);
    *out = t.release();
  });
}

int pftg_table_save(const pftg_table* t, const char* path) {
  return guarded([&] {
    if (!t || !path) throw std::invalid_argument("pftg_table_save: null argument");
    table_save(t->t, path);
  });
}

int pftg_table_info(const pftg_table* t, int* nrec, int* max_r) {
  return guarded([&] {
    if (!t) throw std::invalid_argument("pftg_table_info: null table");
    if (nrec) *nrec = (int)t->t.records.size();
    if (max_r) *max_r = t->t.max_r;
  });
}

int pftg_table_record(const pftg_table* t, int i, double* eps, int* r, double* xi, double* achieved,
                      double* coeff) {
  return guarded([&] {
    if (!t) throw std::invalid_argument("pftg_table_record: null table");
    if (i < 0 || i >= (int)t->t.records.size()) throw std::out_of_range("pftg_table_record: index out of range");
    const Record& rec = t->t.records[i];
    if (eps) *eps = rec.eps;
    if (r) *r = rec.r;
    if (xi) *xi = rec.xi;
    if (achieved) *achieved = rec.achieved_error;
    if (coeff) std::memcpy(coeff, rec.coeff.data(), rec.coeff.size() * sizeof(cd));
  });
}

int pftg_measurements_save(const char* dir, size_t count, size_t rows, size_t cols, const double* d, size_t mt1,
                           size_t mt2, const double* dcrop, double noise_scale, uint64_t noise_seed) {
  return guarded([&] {
    if (!dir || (count && !d)) throw std::invalid_argument("pftg_measurements_save: null argument");
    MeasMeta m;
    m.count = count;
    m.rows = rows;
    m.cols = cols;
    m.mt1 = dcrop ? mt1 : 0;
    m.mt2 = dcrop ? mt2 : 0;
    m.noise_scale = noise_scale;
    m.noise_seed = noise_seed;
    meas_save(dir, m, d, dcrop);
  });
}

int pftg_measurements_info(const char* dir, int64_t* info, double* noise_scale, uint64_t* noise_seed) {
  return guarded([&] {
    if (!dir || !info) throw std::invalid_argument("pftg_measurements_info: null argument");
    const MeasMeta m = meas_info(dir);
    info[0] = (int64_t)m.count;
    info[1] = (int64_t)m.rows;
    info[2] = (int64_t)m.cols;
    info[3] = (int64_t)m.mt1;
    info[4] = (int64_t)m.mt2;
    if (noise_scale) *noise_scale = m.noise_scale;
    if (noise_seed) *noise_seed = m.noise_seed;
  });
}

int pftg_measurements_read(const char* dir, int dtype, void* d, void* dcrop) {
  return guarded([&] {
    check_dtype(dtype);
    if (!dir || !d) throw std::invalid_argument("pftg_measurements_read: null argument");
    const MeasMeta m = meas_info(dir);
    if (dtype == PFTG_C64) meas_read<float>(dir, m, static_cast<float*>(d), static_cast<float*>(dcrop));
    else meas_read<double>(dir, m, static_cast<double*>(d), static_cast<double*>(dcrop));
  });
}

int pftg_plan_2d(const pftg_table* t, size_t n1, size_t n2, size_t mt1, size_t mt2, size_t p1, size_t p2,
                 double eps, pftg_plan** out) {
  return guarded([&] {
    if (!t) throw std::invalid_argument("pftg_plan_2d: null scope table");
    auto p = std::make_unique<pftg_plan>();
    p->a1 = plan_1d(n1, mt1, p1, eps, t->t);
    p->a2 = plan_1d(n2, mt2, p2, eps, t->t);
    *out = p.release();
  });
}

int pftg_plan_from_tables(size_t n1, size_t p1, size_t mt1, int r1, const double* B1, const double* W1, size_t n2,
                          size_t p2, size_t mt2, int r2, const double* B2, const double* W2, double eps,
                          pftg_plan** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("pftg_plan_from_tables: null output");
    auto axis = [eps](size_t n, size_t p, size_t mt, int r, const double* B, const double* W) {
      // pft_plan_1d's domain (pft.cpp:35-40)
      if (p < 2 || p > n || n % p != 0) throw std::invalid_argument("pft_plan_1d: p must divide n, 2 <= p <= n");
      if (n / p < 2) throw std::invalid_argument("pft_plan_1d: need q = n/p >= 2");
      if (mt < 1 || 2 * mt > n) throw std::invalid_argument("pft_plan_1d: need 1 <= mt and 2*mt <= n");
      if (r < 1) throw std::invalid_argument("pft_plan_1d: need r >= 1");
      if (!B || !W) throw std::invalid_argument("pftg_plan_from_tables: null table");
      Axis a;
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
      return a;
    };
    auto p = std::make_unique<pftg_plan>();
    p->a1 = axis(n1, p1, mt1, r1, B1, W1);
    p->a2 = axis(n2, p2, mt2, r2, B2, W2);
    *out = p.release();
  });
}

int pftg_plan_load(const char* path, pftg_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<pftg_plan>();
    plan_load(p->a1, p->a2, path);
    *out = p.release();
  });
}

int pftg_plan_save(const pftg_plan* plan, const char* path) {
  return guarded([&] {
    check_plan(plan);
    plan_save(plan->a1, plan->a2, path);
  });
}

void pftg_plan_free(pftg_plan* plan) { delete plan; }

int pftg_plan_info(const pftg_plan* plan, int64_t* info) {
  return guarded([&] {
    check_plan(plan);
    const Axis* ax[2] = {&plan->a1, &plan->a2};
    for (int a = 0; a < 2; ++a) {
      info[5 * a + 0] = (int64_t)ax[a]->n;
      info[5 * a + 1] = (int64_t)ax[a]->p;
      info[5 * a + 2] = (int64_t)ax[a]->q;
      info[5 * a + 3] = (int64_t)ax[a]->mt;
      info[5 * a + 4] = ax[a]->r;
    }
  });
}

int pftg_plan_tables(const pftg_plan* plan, int axis, double* B, double* W) {
  return guarded([&] {
    check_plan(plan);
    if (axis != 1 && axis != 2) throw std::invalid_argument("pftg_plan_tables: axis must be 1 or 2");
    const Axis& a = axis == 1 ? plan->a1 : plan->a2;
    std::memcpy(B, a.B.data(), a.B.size() * sizeof(cd));
    std::memcpy(W, a.W.data(), a.W.size() * sizeof(cd));
  });
}

int pftg_apply_2d_dev(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (batch == 0) return;
    if (dtype == PFTG_C64) apply_dev<float>(plan, z, band, batch, S(stream));
    else apply_dev<double>(plan, z, band, batch, S(stream));
  });
}

int pftg_adjoint_2d_dev(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (batch == 0) return;
    if (dtype == PFTG_C64) adjoint_dev<float>(plan, band, z, batch, S(stream));
    else adjoint_dev<double>(plan, band, z, batch, S(stream));
  });
}

extern "C++" int apply_2d_host_impl(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch,
                                    size_t total) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (batch == 0) return;
    ensure_device();
    const std::size_t nz = plan->a1.n * plan->a2.n, nb = 4 * plan->a1.mt * plan->a2.mt;
    auto run = [&](auto tag) {
      using R = decltype(tag);
      const std::size_t chunk = host_chunk(batch, sizeof(Cx<R>) * nz);
      host_pipeline<R>(batch, nz, nb, z, band, chunk, [&](Cx<R>* din, Cx<R>* dout, std::size_t nbat, cudaStream_t s) {
        apply_dev<R>(plan, din, dout, nbat, s, total);
      });
    };
    if (dtype == PFTG_C64) run(float{});
    else run(double{});
  });
}

extern "C++" int adjoint_2d_host_impl(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch,
                                      size_t total) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (batch == 0) return;
    ensure_device();
    const std::size_t nz = plan->a1.n * plan->a2.n, nb = 4 * plan->a1.mt * plan->a2.mt;
    auto run = [&](auto tag) {
      using R = decltype(tag);
      const std::size_t chunk = host_chunk(batch, sizeof(Cx<R>) * nz);
      host_pipeline<R>(batch, nb, nz, band, z, chunk, [&](Cx<R>* din, Cx<R>* dout, std::size_t nbat, cudaStream_t s) {
        adjoint_dev<R>(plan, din, dout, nbat, s, total);
      });
    };
    if (dtype == PFTG_C64) run(float{});
    else run(double{});
  });
}

// BASELINE configs[1] as one streamed call: forward, then the adjoint of the
// forward output, per chunk of fields. Chunks alternate between two streams,
// so the H2D copy of chunk k+1 runs while chunk k's results (band and
// back-projection) travel D2H (streams round robin): both PCIe directions are busy at once, which
// the two separate calls (H2D-bound apply, D2H-bound adjoint) cannot do.
extern "C++" int fwd_adj_2d_host_impl(const pftg_plan* plan, int dtype, const void* z, void* band, void* back,
                                      size_t batch, size_t total) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (!z || !band || !back) throw std::invalid_argument("pftg_fwd_adj_2d_host: null buffer");
    if (batch == 0) return;
    ensure_device();
    const std::size_t nz = plan->a1.n * plan->a2.n, nb = 4 * plan->a1.mt * plan->a2.mt;
    auto run = [&](auto tag) {
      using R = decltype(tag);
      using C = Cx<R>;
      const std::size_t chunk = host_chunk(batch, sizeof(C) * nz);
      HostRing& r = host_ring();
      {
        std::vector<std::unique_ptr<Scratch>> bufs;
        C *zi[NSLOT], *bo[NSLOT], *zo[NSLOT];
        for (int k = 0; k < NSLOT; ++k) {
          bufs.emplace_back(new Scratch(sizeof(C) * nz * chunk, r.s[1]));
          zi[k] = bufs.back()->as<C>();
          bufs.emplace_back(new Scratch(sizeof(C) * nb * chunk, r.s[1]));
          bo[k] = bufs.back()->as<C>();
          bufs.emplace_back(new Scratch(sizeof(C) * nz * chunk, r.s[1]));
          zo[k] = bufs.back()->as<C>();
        }
        host_ring_run(
            batch, chunk,
            [&](int k, std::size_t b0, std::size_t m, cudaStream_t s) {
              PFTG_CUDA(cudaMemcpyAsync(zi[k], static_cast<const C*>(z) + b0 * nz, sizeof(C) * nz * m,
                                        cudaMemcpyHostToDevice, s));
            },
            [&](int k, std::size_t m, cudaStream_t s) {
              apply_dev<R>(plan, zi[k], bo[k], m, s, total);
              adjoint_dev<R>(plan, bo[k], zo[k], m, s, total);
            },
            [&](int k, std::size_t b0, std::size_t m, cudaStream_t s) {
              PFTG_CUDA(cudaMemcpyAsync(static_cast<C*>(back) + b0 * nz, zo[k], sizeof(C) * nz * m,
                                        cudaMemcpyDeviceToHost, s));
              PFTG_CUDA(cudaMemcpyAsync(static_cast<C*>(band) + b0 * nb, bo[k], sizeof(C) * nb * m,
                                        cudaMemcpyDeviceToHost, s));
            });
      }
      PFTG_CUDA(cudaStreamSynchronize(r.s[1]));
    };
    if (dtype == PFTG_C64) run(float{});
    else run(double{});
  });
}

// `total` = the caller's whole batch: the kernel path (tile / streaming) is chosen on it, so
// a block of a multi-device call runs the same arithmetic as the single-device call
int pftg_apply_2d_host(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch) {
  return apply_2d_host_impl(plan, dtype, z, band, batch, batch);
}
int pftg_adjoint_2d_host(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch) {
  return adjoint_2d_host_impl(plan, dtype, band, z, batch, batch);
}
int pftg_fwd_adj_2d_host(const pftg_plan* plan, int dtype, const void* z, void* band, void* back, size_t batch) {
  return fwd_adj_2d_host_impl(plan, dtype, z, band, back, batch, batch);
}

extern "C++" {
namespace {
// Contiguous blocks of the batch over devices[0 .. ndev), one host thread per block;
// call(b0, m) runs a single-device host-buffer entry point on fields [b0, b0 + m).
template <class F>
int run_multi(const pftg_plan* plan, int dtype, std::size_t batch, const int* devices, int ndev, F&& call) {
  int rc0 = guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (!devices || ndev < 1) throw std::invalid_argument("pftg: multi-device call needs ndev >= 1 devices");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw cuda_error("pftg: no CUDA device available (this library has no CPU fallback)");
    }
    for (int i = 0; i < ndev; ++i)
      if (devices[i] < 0 || devices[i] >= n) throw std::out_of_range("pftg: device index out of range");
  });
  if (rc0 != PFTG_OK) return rc0;
  std::vector<int> rc(ndev, PFTG_OK);
  std::vector<std::string> msg(ndev);
  std::vector<std::thread> th;
  const std::size_t base = batch / ndev, rem = batch % ndev;
  for (int i = 0; i < ndev; ++i) {
    const std::size_t b0 = i * base + std::min<std::size_t>(i, rem), m = base + ((std::size_t)i < rem ? 1 : 0);
    th.emplace_back([&, i, b0, m] {
      if (m == 0) return;
      if (cudaSetDevice(devices[i]) != cudaSuccess) {
        rc[i] = PFTG_ECUDA;
        msg[i] = "pftg: cudaSetDevice failed";
        return;
      }
      rc[i] = call(b0, m);
      if (rc[i] != PFTG_OK) msg[i] = pftg_last_error();  // thread-local message of the worker
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < ndev; ++i)
    if (rc[i] != PFTG_OK) {
      set_error(msg[i]);
      return rc[i];
    }
  return PFTG_OK;
}
}  // namespace
}  // extern "C++"

int pftg_apply_2d_host_multi(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch,
                             const int* devices, int ndev) {
  if (!plan) return pftg_apply_2d_host(plan, dtype, z, band, batch);  // reports the error
  const std::size_t es = dtype == PFTG_C64 ? 8 : 16;
  const std::size_t nz = plan->a1.n * plan->a2.n * es, nb = 4 * plan->a1.mt * plan->a2.mt * es;
  return run_multi(plan, dtype, batch, devices, ndev, [&](std::size_t b0, std::size_t m) {
    return apply_2d_host_impl(plan, dtype, static_cast<const char*>(z) + b0 * nz, static_cast<char*>(band) + b0 * nb, m,
                              batch);
  });
}

int pftg_adjoint_2d_host_multi(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch,
                               const int* devices, int ndev) {
  if (!plan) return pftg_adjoint_2d_host(plan, dtype, band, z, batch);
  const std::size_t es = dtype == PFTG_C64 ? 8 : 16;
  const std::size_t nz = plan->a1.n * plan->a2.n * es, nb = 4 * plan->a1.mt * plan->a2.mt * es;
  return run_multi(plan, dtype, batch, devices, ndev, [&](std::size_t b0, std::size_t m) {
    return adjoint_2d_host_impl(plan, dtype, static_cast<const char*>(band) + b0 * nb, static_cast<char*>(z) + b0 * nz,
                                m, batch);
  });
}

int pftg_fwd_adj_2d_host_multi(const pftg_plan* plan, int dtype, const void* z, void* band, void* back,
                               size_t batch, const int* devices, int ndev) {
  if (!plan) return pftg_fwd_adj_2d_host(plan, dtype, z, band, back, batch);
  const std::size_t es = dtype == PFTG_C64 ? 8 : 16;
  const std::size_t nz = plan->a1.n * plan->a2.n * es, nb = 4 * plan->a1.mt * plan->a2.mt * es;
  return run_multi(plan, dtype, batch, devices, ndev, [&](std::size_t b0, std::size_t m) {
    return fwd_adj_2d_host_impl(plan, dtype, static_cast<const char*>(z) + b0 * nz, static_cast<char*>(band) + b0 * nb,
                                static_cast<char*>(back) + b0 * nz, m, batch);
  });
}

int pftg_band_residual_dev(const pftg_plan* plan, int dtype, const void* exit_wave, const void* dcrop, void* out,
                           size_t batch, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_dtype(dtype);
    if (batch == 0) return;
    if (dtype == PFTG_C64) band_residual_dev<float>(plan, exit_wave, dcrop, out, batch, S(stream));
    else band_residual_dev<double>(plan, exit_wave, dcrop, out, batch, S(stream));
  });
}

int pftg_fft2_dev(int dtype, const void* z, void* out, size_t rows, size_t cols, size_t batch, int inverse,
                  void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (rows == 0 || cols == 0) throw std::invalid_argument("fast_fft2: empty field");
    if (batch == 0) return;
    ensure_device();
    if (dtype == PFTG_C64) fft2_dev<float>(z, out, rows, cols, batch, inverse, S(stream));
    else fft2_dev<double>(z, out, rows, cols, batch, inverse, S(stream));
  });
}

int pftg_fft2_host(int dtype, const void* z, void* out, size_t rows, size_t cols, size_t batch, int inverse) {
  return guarded([&] {
    check_dtype(dtype);
    if (rows == 0 || cols == 0) throw std::invalid_argument("fast_fft2: empty field");
    check_fft_len(rows);
    check_fft_len(cols);
    if (batch == 0) return;
    ensure_device();
    const std::size_t n = rows * cols;
    auto run = [&](auto tag) {
      using R = decltype(tag);
      const std::size_t chunk = host_chunk(batch, sizeof(Cx<R>) * n);
      host_pipeline<R>(batch, n, n, z, out, chunk, [&](Cx<R>* din, Cx<R>* dout, std::size_t nbat, cudaStream_t s) {
        fft2_dev<R>(din, dout, rows, cols, nbat, inverse, s);
      });
    };
    if (dtype == PFTG_C64) run(float{});
    else run(double{});
  });
}

int pftg_project_modulus_dev(int dtype, const void* exit_wave, const void* d, void* out, size_t rows, size_t cols,
                             size_t batch, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (batch == 0) return;
    ensure_device();
    if (dtype == PFTG_C64) project_modulus_dev<float>(exit_wave, d, out, rows, cols, batch, S(stream));
    else project_modulus_dev<double>(exit_wave, d, out, rows, cols, batch, S(stream));
  });
}

int pftg_crop_centered_dev(int dtype, const void* spectrum, void* out, size_t rows, size_t cols, size_t mt1,
                           size_t mt2, size_t batch, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (mt1 == 0 || mt2 == 0) throw std::invalid_argument("crop_centered: mt must be >= 1");
    if (2 * mt1 > rows || 2 * mt2 > cols) throw std::invalid_argument("crop_centered: band exceeds spectrum shape");
    if (batch == 0) return;
    ensure_device();
    const long long tot = 4LL * mt1 * mt2 * batch;
    if (dtype == PFTG_C64)
      k_crop<float><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<const float*>(spectrum), static_cast<float*>(out),
                                                          (int)rows, (int)cols, (int)mt1, (int)mt2, (long long)batch);
    else
      k_crop<double><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<const double*>(spectrum),
                                                           static_cast<double*>(out), (int)rows, (int)cols, (int)mt1,
                                                           (int)mt2, (long long)batch);
    PFTG_LAUNCH_CHECK();
  });
}

int pftg_window_slice_dev(int dtype, const void* frame, size_t fr, size_t fc, void* patches, size_t wr, size_t wc,
                          const int64_t* offsets, size_t npos, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (npos == 0) return;
    ensure_device();
    std::vector<long long> offs(npos);
    for (size_t j = 0; j < npos; ++j) {
      check_window(offsets[2 * j], offsets[2 * j + 1], wr, wc, fr, fc);
      offs[j] = offsets[2 * j] * (long long)fc + offsets[2 * j + 1];
    }
    Scratch d(sizeof(long long) * npos, S(stream));
    PFTG_CUDA(cudaMemcpyAsync(d.p, offs.data(), sizeof(long long) * npos, cudaMemcpyHostToDevice, S(stream)));
    const long long tot = (long long)wr * wc * npos;
    if (dtype == PFTG_C64)
      k_window_slice<float2><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<const float2*>(frame), (long long)fc,
                                                                   static_cast<float2*>(patches), (int)wr, (int)wc,
                                                                   d.as<long long>(), (int)npos);
    else
      k_window_slice<double2><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<const double2*>(frame),
                                                                    (long long)fc, static_cast<double2*>(patches),
                                                                    (int)wr, (int)wc, d.as<long long>(), (int)npos);
    PFTG_LAUNCH_CHECK();
    // keep the offsets alive until the kernel has consumed them
    PFTG_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int pftg_set_window_dev(int dtype, void* frame, size_t fr, size_t fc, const void* patch, size_t wr, size_t wc,
                        int64_t r0, int64_t c0, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    check_window(r0, c0, wr, wc, fr, fc);
    ensure_device();
    const long long off = r0 * (long long)fc + c0;
    const long long tot = (long long)wr * wc;
    if (dtype == PFTG_C64)
      k_set_window<float2><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<float2*>(frame), (long long)fc,
                                                                 static_cast<const float2*>(patch), (int)wr, (int)wc,
                                                                 off);
    else
      k_set_window<double2><<<grid_for(tot), 256, 0, S(stream)>>>(static_cast<double2*>(frame), (long long)fc,
                                                                  static_cast<const double2*>(patch), (int)wr,
                                                                  (int)wc, off);
    PFTG_LAUNCH_CHECK();
  });
}

int pftg_pie_object_update_dev(int dtype, void* zj, const void* probe, const void* proj, size_t n, double beta,
                               void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    ensure_device();
    if (dtype == PFTG_C64)
      k_update<float2><<<grid_for(n), 256, 0, S(stream)>>>(static_cast<float2*>(zj), static_cast<const float2*>(probe),
                                                           static_cast<const float2*>(proj), (long long)n, beta, 0);
    else
      k_update<double2><<<grid_for(n), 256, 0, S(stream)>>>(static_cast<double2*>(zj),
                                                            static_cast<const double2*>(probe),
                                                            static_cast<const double2*>(proj), (long long)n, beta, 0);
    PFTG_LAUNCH_CHECK();
  });
}

int pftg_epie_probe_update_dev(int dtype, void* probe, const void* zj, const void* proj, size_t n, double gamma,
                               int blind, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (!blind) throw std::logic_error("epie_probe_update: probe updates need blind mode");
    ensure_device();
    if (dtype == PFTG_C64)
      k_update<float2><<<grid_for(n), 256, 0, S(stream)>>>(static_cast<float2*>(probe), static_cast<const float2*>(zj),
                                                           static_cast<const float2*>(proj), (long long)n, gamma, 1);
    else
      k_update<double2><<<grid_for(n), 256, 0, S(stream)>>>(static_cast<double2*>(probe),
                                                            static_cast<const double2*>(zj),
                                                            static_cast<const double2*>(proj), (long long)n, gamma, 1);
    PFTG_LAUNCH_CHECK();
  });
}

int pftg_evaluate_dev(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr, size_t wc,
                      const int64_t* offsets, size_t npos, size_t pos_begin, size_t pos_end, const void* d,
                      const pftg_plan* plan, const void* dcrop, double* fft_sum, double* band_sum, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    ensure_device();
    if (dtype == PFTG_C64)
      evaluate_dev<float>(frame, fr, fc, probe, wr, wc, offsets, npos, pos_begin, pos_end, d, plan, dcrop, fft_sum,
                          band_sum, S(stream));
    else
      evaluate_dev<double>(frame, fr, fc, probe, wr, wc, offsets, npos, pos_begin, pos_end, d, plan, dcrop, fft_sum,
                           band_sum, S(stream));
  });
}

}  // extern "C"
