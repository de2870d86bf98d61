// TEST INFRASTRUCTURE ONLY -- not product code.
//
// extern "C" shim over the UNMODIFIED reference library (proj/core compiled
// verbatim from /root/reference by oracle/Makefile, with the Eigen/FFTW shims
// under oracle/shim/). Lets pytest (ctypes + numpy), golden-fixture generation
// and bench.py's reference arm call the reference's own operators:
//   ptycho::pft::{pft_plan_2d, pft_apply_2d, pft_adjoint_2d, save_plan, load_plan_2d}
//   ptycho::{fast_fft2, fast_ifft2, naive_dft2, crop_centered}
//   ptycho::{band_residual, project_modulus, objective_value, hybrid_solve}
//   ptycho::minimax::{best_approx, ScopeTable}
//   ptycho::{relative_error, relative_error_aligned, ssim, psnr, dynamic_range} (fill_metrics set)
// Complex arrays cross the boundary as interleaved (re, im) float64, row-major,
// exactly the ComplexField layout (field.hpp:37-65).
#include <Eigen/Dense>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ptycho/fft.hpp"
#include "ptycho/field.hpp"
#include "ptycho/metrics.hpp"
#include "ptycho/minimax.hpp"
#include "ptycho/pft.hpp"
#include "ptycho/scan.hpp"
#include "ptycho/simulate.hpp"
#include "ptycho/solver.hpp"

using namespace ptycho;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 3;
  }
}

ComplexField to_field(const double* z, std::size_t rows, std::size_t cols) {
  ComplexField f(rows, cols);
  std::memcpy(static_cast<void*>(f.data()), z, rows * cols * sizeof(cdouble));
  return f;
}

RealField to_real(const double* d, std::size_t rows, std::size_t cols) {
  RealField f(rows, cols);
  std::memcpy(f.data(), d, rows * cols * sizeof(double));
  return f;
}

void from_field(const ComplexField& f, double* out) {
  std::memcpy(out, static_cast<const void*>(f.data()), f.size() * sizeof(cdouble));
}

struct PlanHandle {
  pft::PftPlan2D plan;
};

ScanPattern make_pattern(std::size_t fr, std::size_t fc, std::size_t wr, std::size_t wc,
                         const std::int64_t* offsets, std::size_t npos) {
  ScanPattern sp;
  sp.object_rows = sp.frame_rows = fr;
  sp.object_cols = sp.frame_cols = fc;
  sp.window_rows = wr;
  sp.window_cols = wc;
  sp.mask = RealField(wr, wc, 1.0);
  for (std::size_t j = 0; j < npos; ++j)
    sp.offsets.emplace_back(static_cast<std::size_t>(offsets[2 * j]),
                            static_cast<std::size_t>(offsets[2 * j + 1]));
  return sp;
}

MeasurementSet make_ms(std::size_t wr, std::size_t wc, const double* d, std::size_t npos) {
  MeasurementSet ms;
  ms.window_rows = wr;
  ms.window_cols = wc;
  for (std::size_t j = 0; j < npos; ++j) ms.d.push_back(to_real(d + j * wr * wc, wr, wc));
  return ms;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- minimax (minimax.hpp:28,45-70) ----
int ref_best_approx(int r, double xi, double* coeff_out, double* achieved, int* converged) {
  return guarded([&] {
    const auto p = minimax::best_approx(r, xi);
    for (int j = 0; j < r; ++j) {
      coeff_out[2 * j] = p.coeff[j].real();
      coeff_out[2 * j + 1] = p.coeff[j].imag();
    }
    *achieved = p.achieved_error;
    *converged = p.exchange_converged ? 1 : 0;
  });
}

int ref_scope_table_compute(const char* path, const double* eps, int neps, int max_r) {
  return guarded([&] {
    const auto t = minimax::ScopeTable::compute(std::vector<double>(eps, eps + neps), max_r);
    t.save(path);
  });
}

// One-record table (eps, r) certified on |x| <= xi: how the literal BASELINE
// plans (xi = mt/p = 4) are expressed through the reference's own table format.
int ref_scope_table_single(const char* path, double eps, int r, double xi) {
  return guarded([&] {
    const auto p = minimax::best_approx(r, xi);
    std::FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error("cannot open table path");
    std::fprintf(f, "pft-scope-table v1\n");
    std::fprintf(f, "# record <eps> <r> <xi> <achieved_error> <w0.re> <w0.im> ... (r pairs)\n");
    std::fprintf(f, "record %.6e %d %.17g %.17g", eps, r, xi, p.achieved_error);
    for (const auto& c : p.coeff) std::fprintf(f, " %.17g %.17g", c.real(), c.imag());
    std::fprintf(f, "\n");
    std::fclose(f);
  });
}

int ref_min_degree(const char* table_path, double eps, double target, int* r_out) {
  return guarded([&] {
    const auto t = minimax::ScopeTable::load(table_path);
    *r_out = t.min_degree(eps, target);
  });
}

// ---- plans (pft.hpp:44-63) ----
void* ref_plan_create(const char* table_path, std::size_t n1, std::size_t n2, std::size_t mt1,
                      std::size_t mt2, std::size_t p1, std::size_t p2, double eps) {
  PlanHandle* h = nullptr;
  const int rc = guarded([&] {
    const auto t = minimax::ScopeTable::load(table_path);
    auto hp = std::make_unique<PlanHandle>();
    hp->plan = pft::pft_plan_2d(n1, n2, mt1, mt2, p1, p2, eps, t);
    h = hp.release();
  });
  return rc == 0 ? h : nullptr;
}

void* ref_plan_load(const char* plan_path) {
  PlanHandle* h = nullptr;
  const int rc = guarded([&] {
    auto hp = std::make_unique<PlanHandle>();
    hp->plan = pft::load_plan_2d(plan_path);
    h = hp.release();
  });
  return rc == 0 ? h : nullptr;
}

int ref_plan_save(void* h, const char* plan_path) {
  return guarded([&] { pft::save_plan(plan_path, static_cast<PlanHandle*>(h)->plan); });
}

void ref_plan_free(void* h) { delete static_cast<PlanHandle*>(h); }

// info[10] = n1 p1 q1 mt1 r1 n2 p2 q2 mt2 r2
void ref_plan_info(void* h, std::int64_t* info) {
  const auto& pl = static_cast<PlanHandle*>(h)->plan;
  const pft::PftPlan1D* ax[2] = {&pl.axis1, &pl.axis2};
  for (int a = 0; a < 2; ++a) {
    info[5 * a + 0] = static_cast<std::int64_t>(ax[a]->n);
    info[5 * a + 1] = static_cast<std::int64_t>(ax[a]->p);
    info[5 * a + 2] = static_cast<std::int64_t>(ax[a]->q);
    info[5 * a + 3] = static_cast<std::int64_t>(ax[a]->mt);
    info[5 * a + 4] = ax[a]->r;
  }
}

// B (q x r) and W ((2mt+1) x r) of one axis, interleaved complex.
void ref_plan_tables(void* h, int axis, double* B, double* W) {
  const auto& pl = static_cast<PlanHandle*>(h)->plan;
  const pft::PftPlan1D& a = axis == 1 ? pl.axis1 : pl.axis2;
  from_field(a.B, B);
  from_field(a.W, W);
}

int ref_pft_apply_2d(void* h, const double* z, std::size_t n1, std::size_t n2, double* out) {
  return guarded([&] {
    const auto band = pft::pft_apply_2d(static_cast<PlanHandle*>(h)->plan, to_field(z, n1, n2));
    from_field(band, out);
  });
}

int ref_pft_adjoint_2d(void* h, const double* band, std::size_t m1, std::size_t m2, double* out) {
  return guarded([&] {
    const auto z = pft::pft_adjoint_2d(static_cast<PlanHandle*>(h)->plan, to_field(band, m1, m2));
    from_field(z, out);
  });
}

// Batched forward+adjoint over independent fields on T threads (one field per
// thread; apply/adjoint are reentrant). Used as the CPU arm.
int ref_pft_fwd_adj_batch(void* h, const double* z, std::size_t batch, std::size_t n1,
                          std::size_t n2, double* band_out, double* z_out, int threads);

// ---- 1-D plans and apply (pft.hpp:25-38, 60-63) ----
struct Plan1DHandle {
  pft::PftPlan1D plan;
};

void* ref_plan1d_create(const char* table_path, std::size_t n, std::size_t mt, std::size_t p, double eps) {
  Plan1DHandle* h = nullptr;
  const int rc = guarded([&] {
    const auto t = minimax::ScopeTable::load(table_path);
    auto hp = std::make_unique<Plan1DHandle>();
    hp->plan = pft::pft_plan_1d(n, mt, p, eps, t);
    h = hp.release();
  });
  return rc == 0 ? h : nullptr;
}

void* ref_plan1d_load(const char* plan_path) {
  Plan1DHandle* h = nullptr;
  const int rc = guarded([&] {
    auto hp = std::make_unique<Plan1DHandle>();
    hp->plan = pft::load_plan_1d(plan_path);
    h = hp.release();
  });
  return rc == 0 ? h : nullptr;
}

int ref_plan1d_save(void* h, const char* plan_path) {
  return guarded([&] { pft::save_plan(plan_path, static_cast<Plan1DHandle*>(h)->plan); });
}

void ref_plan1d_free(void* h) { delete static_cast<Plan1DHandle*>(h); }

// info[5] = n p q mt r
void ref_plan1d_info(void* h, std::int64_t* info) {
  const auto& a = static_cast<Plan1DHandle*>(h)->plan;
  info[0] = static_cast<std::int64_t>(a.n);
  info[1] = static_cast<std::int64_t>(a.p);
  info[2] = static_cast<std::int64_t>(a.q);
  info[3] = static_cast<std::int64_t>(a.mt);
  info[4] = a.r;
}

void ref_plan1d_tables(void* h, double* B, double* W) {
  const auto& a = static_cast<Plan1DHandle*>(h)->plan;
  from_field(a.B, B);
  from_field(a.W, W);
}

int ref_pft_apply_1d(void* h, const double* z, std::size_t n, double* out) {
  return guarded([&] {
    const auto band = pft::pft_apply_1d(static_cast<Plan1DHandle*>(h)->plan, to_field(z, n, 1));
    from_field(band, out);
  });
}

// ---- transforms (fft.hpp:9-30) ----
int ref_fast_fft2(const double* z, std::size_t r, std::size_t c, double* out) {
  return guarded([&] { from_field(fast_fft2(to_field(z, r, c)), out); });
}
int ref_fast_ifft2(const double* z, std::size_t r, std::size_t c, double* out) {
  return guarded([&] { from_field(fast_ifft2(to_field(z, r, c)), out); });
}
int ref_naive_dft2(const double* z, std::size_t r, std::size_t c, double* out) {
  return guarded([&] { from_field(naive_dft2(to_field(z, r, c)), out); });
}
int ref_naive_idft2(const double* z, std::size_t r, std::size_t c, double* out) {
  return guarded([&] { from_field(naive_idft2(to_field(z, r, c)), out); });
}
int ref_crop_centered_real(const double* d, std::size_t r, std::size_t c, std::size_t mt1,
                           std::size_t mt2, double* out) {
  return guarded([&] {
    const RealField o = crop_centered(to_real(d, r, c), mt1, mt2);
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

// ---- solver building blocks (solver.hpp:51-71) ----
int ref_project_modulus(const double* exit, const double* d, std::size_t r, std::size_t c,
                        double* out) {
  return guarded([&] { from_field(project_modulus(to_field(exit, r, c), to_real(d, r, c)), out); });
}

int ref_band_residual(void* h, const double* exit, std::size_t wr, std::size_t wc,
                      const double* dcrop, std::size_t m1, std::size_t m2, double* out) {
  return guarded([&] {
    from_field(band_residual(static_cast<PlanHandle*>(h)->plan, to_field(exit, wr, wc),
                             to_real(dcrop, m1, m2)),
               out);
  });
}

int ref_pie_object_update(double* zj, const double* probe, const double* proj, std::size_t r,
                          std::size_t c, double beta) {
  return guarded([&] {
    ComplexField z = to_field(zj, r, c);
    pie_object_update(z, to_field(probe, r, c), to_field(proj, r, c), beta);
    from_field(z, zj);
  });
}

int ref_epie_probe_update(double* probe, const double* zj, const double* proj, std::size_t r,
                          std::size_t c, double gamma, int blind) {
  return guarded([&] {
    ComplexField p = to_field(probe, r, c);
    epie_probe_update(p, to_field(zj, r, c), to_field(proj, r, c), gamma, blind != 0);
    from_field(p, probe);
  });
}

int ref_objective_value(const double* frame, std::size_t fr, std::size_t fc, const double* probe,
                        std::size_t wr, std::size_t wc, const std::int64_t* offsets,
                        std::size_t npos, const double* d, double* out) {
  return guarded([&] {
    const ScanPattern sp = make_pattern(fr, fc, wr, wc, offsets, npos);
    const MeasurementSet ms = make_ms(wr, wc, d, npos);
    *out = objective_value(to_field(frame, fr, fc), to_field(probe, wr, wc), sp, ms);
  });
}

int ref_simulate(const double* frame, std::size_t fr, std::size_t fc, const double* probe,
                 std::size_t wr, std::size_t wc, const std::int64_t* offsets, std::size_t npos,
                 double* d_out) {
  return guarded([&] {
    const ScanPattern sp = make_pattern(fr, fc, wr, wc, offsets, npos);
    const MeasurementSet ms = simulate(to_field(frame, fr, fc), to_field(probe, wr, wc), sp);
    for (std::size_t j = 0; j < npos; ++j)
      std::memcpy(d_out + j * wr * wc, ms.d[j].data(), wr * wc * sizeof(double));
  });
}

// save_measurements (simulate.cpp:91-127) of d [npos][wr][wc]; build_cropped
// first when mt1 > 0; the noise fields are recorded as given.
int ref_save_measurements(const char* dir, const double* d, std::size_t npos, std::size_t wr, std::size_t wc,
                          std::size_t mt1, std::size_t mt2, double noise_scale, std::uint64_t noise_seed) {
  return guarded([&] {
    MeasurementSet ms;
    ms.window_rows = wr;
    ms.window_cols = wc;
    for (std::size_t j = 0; j < npos; ++j) {
      RealField x(wr, wc);
      std::memcpy(x.data(), d + j * wr * wc, wr * wc * sizeof(double));
      ms.d.push_back(std::move(x));
    }
    if (mt1 > 0) build_cropped(ms, mt1, mt2);
    ms.noise_scale = noise_scale;
    ms.noise_seed = noise_seed;
    save_measurements(dir, ms);
  });
}

// load_measurements (simulate.cpp:129-164): info[5] = count rows cols mt1 mt2;
// d / dcrop filled when non-null.
int ref_load_measurements(const char* dir, std::int64_t* info, double* noise, double* d, double* dcrop) {
  return guarded([&] {
    const MeasurementSet ms = load_measurements(dir);
    info[0] = static_cast<std::int64_t>(ms.count());
    info[1] = static_cast<std::int64_t>(ms.window_rows);
    info[2] = static_cast<std::int64_t>(ms.window_cols);
    info[3] = static_cast<std::int64_t>(ms.mt1);
    info[4] = static_cast<std::int64_t>(ms.mt2);
    noise[0] = ms.noise_scale;
    noise[1] = static_cast<double>(ms.noise_seed);
    const std::size_t wn = ms.window_rows * ms.window_cols, cn = 4 * ms.mt1 * ms.mt2;
    for (std::size_t j = 0; j < ms.count(); ++j) {
      if (d) std::memcpy(d + j * wn, ms.d[j].data(), wn * sizeof(double));
      if (dcrop && j < ms.d_crop.size()) std::memcpy(dcrop + j * cn, ms.d_crop[j].data(), cn * sizeof(double));
    }
  });
}

int ref_add_poisson_noise(double* d, std::size_t wr, std::size_t wc, std::size_t npos,
                          double scale, std::uint64_t seed) {
  return guarded([&] {
    MeasurementSet ms = make_ms(wr, wc, d, npos);
    add_poisson_noise(ms, scale, seed);
    for (std::size_t j = 0; j < npos; ++j)
      std::memcpy(d + j * wr * wc, ms.d[j].data(), wr * wc * sizeof(double));
  });
}

// ---- driver (solver.hpp:87-90) ----
// cfg_d[8] = beta gamma beta_pft gamma_pft eps_pft tol tv_mag tv_phase
// cfg_i[9] = pft_sweeps fft_sweeps mt1 mt2 p1 p2 blind shuffled seed
// trace_out[2 * (pft+fft sweeps)] = (objective, wall_s) per sweep
int ref_hybrid_solve(double* frame, std::size_t fr, std::size_t fc, double* probe, std::size_t wr,
                     std::size_t wc, const std::int64_t* offsets, std::size_t npos,
                     const double* d, const double* cfg_d, const std::int64_t* cfg_i,
                     const char* table_path, double* trace_out, int* sweeps_run, int* flags) {
  return guarded([&] {
    const ScanPattern sp = make_pattern(fr, fc, wr, wc, offsets, npos);
    const MeasurementSet ms = make_ms(wr, wc, d, npos);
    SolverConfig cfg;
    cfg.beta = cfg_d[0];
    cfg.gamma = cfg_d[1];
    cfg.beta_pft = cfg_d[2];
    cfg.gamma_pft = cfg_d[3];
    cfg.eps_pft = cfg_d[4];
    cfg.tol = cfg_d[5];
    cfg.tv_lambda_mag = cfg_d[6];
    cfg.tv_lambda_phase = cfg_d[7];
    cfg.pft_sweeps = static_cast<int>(cfg_i[0]);
    cfg.fft_sweeps = static_cast<int>(cfg_i[1]);
    cfg.mt1 = static_cast<std::size_t>(cfg_i[2]);
    cfg.mt2 = static_cast<std::size_t>(cfg_i[3]);
    cfg.p1 = static_cast<std::size_t>(cfg_i[4]);
    cfg.p2 = static_cast<std::size_t>(cfg_i[5]);
    cfg.blind = cfg_i[6] != 0;
    cfg.order = cfg_i[7] != 0 ? VisitOrder::shuffled : VisitOrder::sequential;
    cfg.seed = static_cast<std::uint64_t>(cfg_i[8]);
    std::unique_ptr<minimax::ScopeTable> table;
    if (table_path && *table_path)
      table = std::make_unique<minimax::ScopeTable>(minimax::ScopeTable::load(table_path));
    const ReconResult res = hybrid_solve(ms, sp, to_field(probe, wr, wc), to_field(frame, fr, fc),
                                         cfg, table.get(), nullptr);
    from_field(res.frame, frame);
    from_field(res.probe, probe);
    const auto& rows = res.trace.rows();
    for (std::size_t i = 0; i < rows.size(); ++i) {
      trace_out[2 * i] = rows[i].objective;
      trace_out[2 * i + 1] = rows[i].wall_s;
    }
    *sweeps_run = res.sweeps_run;
    *flags = (res.diverged ? 1 : 0) | (res.stopped_early ? 2 : 0);
  });
}

}  // extern "C"

#include <thread>

extern "C" int ref_pft_fwd_adj_batch(void* h, const double* z, std::size_t batch, std::size_t n1,
                                     std::size_t n2, double* band_out, double* z_out,
                                     int threads) {
  return guarded([&] {
    const auto& plan = static_cast<PlanHandle*>(h)->plan;
    const std::size_t m1 = 2 * plan.axis1.mt, m2 = 2 * plan.axis2.mt;
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<std::size_t>(threads));
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (std::size_t b = static_cast<std::size_t>(t); b < batch;
               b += static_cast<std::size_t>(threads)) {
            const auto band = pft::pft_apply_2d(plan, to_field(z + 2 * b * n1 * n2, n1, n2));
            const auto back = pft::pft_adjoint_2d(plan, band);
            if (band_out) from_field(band, band_out + 2 * b * m1 * m2);
            if (z_out) from_field(back, z_out + 2 * b * n1 * n2);
          }
        } catch (const std::exception& e) {
          errs[static_cast<std::size_t>(t)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// The per-sweep metrics row of hybrid_solve's trace (fill_metrics,
// solver.cpp:141-160) for reconstruction x vs truth t (both rows x cols):
// out = rel_err, rel_err_aligned, rel_err_mag, rel_err_phase, ssim_mag,
// ssim_phase, psnr_mag, psnr_phase.
extern "C" int ref_fill_metrics(const double* x, const double* t, std::size_t rows, std::size_t cols,
                                double* out) {
  return guarded([&] {
    const ComplexField xf = to_field(x, rows, cols), tf = to_field(t, rows, cols);
    const RealField xm = magnitude(xf), xp = phase(xf), tm = magnitude(tf), tp = phase(tf);
    const double rm = dynamic_range(tm), rp = dynamic_range(tp);
    out[0] = relative_error(xf, tf);
    out[1] = relative_error_aligned(xf, tf);
    out[2] = relative_error(xm, tm);
    out[3] = relative_error(xp, tp);
    out[4] = ssim(xm, tm, rm);
    out[5] = ssim(xp, tp, rp);
    out[6] = psnr(xm, tm, rm);
    out[7] = psnr(xp, tp, rp);
  });
}

// Throughput of the Eigen shim's complex GEMM (oracle/shim/Eigen/Dense) on an
// m x k x n product -- reported beside the CPU baseline so the reader can
// judge the shim against a real Eigen build (the reference's stage A is
// B1^T (r x q) * Z_blk (q x n): m = r, k = q).
extern "C" int ref_shim_gemm_gflops(int m, int k, int n, int reps, double* gflops) {
  return guarded([&] {
    using RowMat = Eigen::Matrix<cdouble, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
    RowMat A(k, m), B(k, n), T(m, n);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < m; ++j) A(i, j) = cdouble(0.5 + 0.01 * i, -0.25 + 0.02 * j);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < n; ++j) B(i, j) = cdouble(0.001 * j, 0.003 * i);
    T.noalias() = A.transpose() * B;
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) T.noalias() = A.transpose() * B;
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *gflops = 8.0 * m * k * n * reps / s / 1e9;
  });
}
