// C++ façade: the reference's own operator signatures backed by libpftg.
//
// A reference maintainer adds this one translation unit to proj/core and links
// -lpftg; it REPLACES the online phase of src/pft.cpp and the fast transforms of
// src/fft.cpp:
//
//   ptycho::pft::pft_apply_2d   (pft.hpp:53, pft.cpp:119-172)
//   ptycho::pft::pft_adjoint_2d (pft.hpp:57, pft.cpp:174-226)
//   ptycho::pft::pft_apply_1d   (pft.hpp:38, pft.cpp:78-101)
//   ptycho::fast_fft2           (fft.hpp:18, fft.cpp:175-178)
//   ptycho::fast_ifft2          (fft.hpp:19, fft.cpp:180-183)
//
// Everything else -- plans (pft_plan_2d, load/save), solver.cpp (project_modulus,
// band_residual, hybrid_solve, ...), scan.cpp, simulate.cpp -- compiles
// unmodified and now runs on the GPU transforms: same signatures, same value
// semantics (inputs by const&, fresh 64-byte aligned outputs), same exception
// types (std::invalid_argument for shape/plan mismatch, ...). This per-call form
// is correct but copy-bound (host <-> device per call); whole solves belong on
// the device-resident pftg_solver_* API.
//
// Plans: the reference's PftPlan2D (host B/W tables) is mirrored into an
// immutable pftg plan by pftg_plan_from_tables (no file round trip), cached per
// plan identity (the plan's shared slice-FFT handle; copies of a plan share it)
// and dropped when the last copy of the plan is gone. Thread-safe.
//
// Build (oracle/Makefile's facade target does exactly this against the
// verbatim reference sources): compile with -I<proj/core>/include
// -I<repo>/include, and compile the reference's pft.cpp / fft.cpp with
// -Dpft_apply_2d=cpu_pft_apply_2d -Dpft_adjoint_2d=cpu_pft_adjoint_2d
// -Dpft_apply_1d=cpu_pft_apply_1d
// -Dfast_fft2=cpu_fast_fft2 -Dfast_ifft2=cpu_fast_ifft2 (or delete those five
// definitions) so this file's definitions are the ones linked.
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "pftg.h"
#include "ptycho/fft.hpp"
#include "ptycho/pft.hpp"

namespace ptycho {
namespace {

// pftg status -> the reference's exception types (include/pftg.h)
void check(int rc) {
  if (rc == PFTG_OK) return;
  const std::string msg = pftg_last_error();
  switch (rc) {
    case PFTG_EINVAL: throw std::invalid_argument(msg);
    case PFTG_ELOGIC: throw std::logic_error(msg);
    case PFTG_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

using GpuPlan = std::shared_ptr<pftg_plan>;

GpuPlan make_gpu_plan(const pft::PftPlan2D& p) {
  const auto& a = p.axis1;
  const auto& b = p.axis2;
  pftg_plan* h = nullptr;
  check(pftg_plan_from_tables(a.n, a.p, a.mt, a.r, reinterpret_cast<const double*>(a.B.data()),
                              reinterpret_cast<const double*>(a.W.data()), b.n, b.p, b.mt, b.r,
                              reinterpret_cast<const double*>(b.B.data()),
                              reinterpret_cast<const double*>(b.W.data()), a.eps, &h));
  return GpuPlan(h, pftg_plan_free);
}

struct CacheEntry {
  std::weak_ptr<const detail::SliceBatchFft2> owner;  // expires with the last copy of the plan
  GpuPlan gpu;
};

GpuPlan gpu_plan(const pft::PftPlan2D& p) {
  if (!p.slice_fft) return make_gpu_plan(p);  // hand-assembled plan: no identity to cache on
  static std::mutex mu;
  static std::map<const void*, CacheEntry> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto it = cache.begin(); it != cache.end();)  // drop plans whose owners are gone
    it = it->second.owner.expired() ? cache.erase(it) : std::next(it);
  auto& e = cache[p.slice_fft.get()];
  if (!e.gpu) {
    e.owner = p.slice_fft;
    e.gpu = make_gpu_plan(p);
  }
  return e.gpu;
}

ComplexField fft2_host(const ComplexField& z, int inverse) {
  ComplexField out(z.rows(), z.cols());
  check(pftg_fft2_host(PFTG_C128, z.data(), out.data(), z.rows(), z.cols(), 1, inverse));
  return out;
}

}  // namespace

namespace pft {

ComplexField pft_apply_2d(const PftPlan2D& plan, const ComplexField& z) {
  if (z.rows() != plan.axis1.n || z.cols() != plan.axis2.n)
    throw std::invalid_argument("pft_apply_2d: z shape must match the plan");  // pft.cpp:122-123
  ComplexField out(2 * plan.axis1.mt, 2 * plan.axis2.mt);
  const GpuPlan g = gpu_plan(plan);
  check(pftg_apply_2d_host(g.get(), PFTG_C128, z.data(), out.data(), 1));
  return out;
}

ComplexField pft_adjoint_2d(const PftPlan2D& plan, const ComplexField& band) {
  if (band.rows() != 2 * plan.axis1.mt || band.cols() != 2 * plan.axis2.mt)
    throw std::invalid_argument("pft_adjoint_2d: band shape must match the plan");  // pft.cpp:178-179
  ComplexField out(plan.axis1.n, plan.axis2.n);
  const GpuPlan g = gpu_plan(plan);
  check(pftg_adjoint_2d_host(g.get(), PFTG_C128, band.data(), out.data(), 1));
  return out;
}

ComplexField pft_apply_1d(const PftPlan1D& plan, const ComplexField& z) {
  if (!z.is_vector() || z.rows() != plan.n)
    throw std::invalid_argument("pft_apply_1d: z must be an n-vector matching the plan");  // pft.cpp:79-80
  // PftPlan1D has no shared identity to cache on: the GPU plan lives for this call
  pftg_plan1d* h = nullptr;
  check(pftg_plan1d_from_tables(plan.n, plan.p, plan.mt, plan.r, reinterpret_cast<const double*>(plan.B.data()),
                                reinterpret_cast<const double*>(plan.W.data()), plan.eps, &h));
  std::unique_ptr<pftg_plan1d, void (*)(pftg_plan1d*)> g(h, pftg_plan1d_free);
  ComplexField out(2 * plan.mt + 1, 1);
  check(pftg_apply_1d_host(g.get(), PFTG_C128, z.data(), out.data(), 1));
  return out;
}

}  // namespace pft

ComplexField fast_fft2(const ComplexField& z) { return fft2_host(z, 0); }

ComplexField fast_ifft2(const ComplexField& z) { return fft2_host(z, 1); }

}  // namespace ptycho
