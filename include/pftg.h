/* pftg -- B200-native (sm_100a) fast Partial Fourier Transform and
 * PFT-warm-started ePIE, C-ABI boundary.
 *
 * Every entry point replaces one operator of the reference C++ library
 * /root/reference/proj/core (namespace ptycho); the reference interface it
 * stands in for is cited as header:line. Plain pointers and sizes only.
 *
 * Conventions (identical to the reference):
 *  - complex arrays are interleaved (re, im), row-major, element (i, j) at
 *    i*cols + j  (field.hpp:37-65); a batch is `batch` such arrays back to back;
 *  - dtype PFTG_C64 = complex64 (float re, im; real arrays are float),
 *    dtype PFTG_C128 = complex128 (double; real arrays are double);
 *  - forward DFTs unnormalized, inverse carries 1/n (fft.hpp:14-15);
 *  - the PFT band is 2mt1 x 2mt2, DC at (mt1, mt2), +mt edge dropped
 *    (pft.hpp:40-43, fft.hpp:26-29);
 *  - *_dev functions take DEVICE pointers and a cudaStream_t (as void*, NULL =
 *    default stream) and are stream-ordered (they return before the work
 *    finishes); *_host functions take HOST pointers and return after the result
 *    is in host memory.
 *
 * Errors: every function returns PFTG_OK or an error code; the message is in
 * pftg_last_error() (thread-local). The codes map onto the reference's
 * exception types: PFTG_EINVAL <-> std::invalid_argument (shape/plan mismatch,
 * infeasible degree), PFTG_ELOGIC <-> std::logic_error (probe update without
 * blind), PFTG_ERANGE <-> std::out_of_range (scan position), PFTG_ERUNTIME <->
 * std::runtime_error (I/O, malformed files), PFTG_ECUDA = CUDA failure (no GPU,
 * launch error). There is no CPU fallback: without a usable sm_100 device every
 * compute entry point fails with PFTG_ECUDA.
 */
#ifndef PFTG_H_
#define PFTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFTG_OK 0
#define PFTG_EINVAL 1
#define PFTG_ELOGIC 2
#define PFTG_ERANGE 3
#define PFTG_ERUNTIME 4
#define PFTG_ECUDA 5

#define PFTG_C64 0
#define PFTG_C128 1

typedef struct pftg_table pftg_table; /* minimax::ScopeTable (minimax.hpp:45-70) */
typedef struct pftg_plan pftg_plan;   /* pft::PftPlan2D (pft.hpp:44-47) */
typedef struct pftg_solver pftg_solver; /* device-resident hybrid_solve state (solver.hpp:87-90) */

int pftg_version(void);
const char* pftg_last_error(void);
/* 1 if a CUDA device of compute capability 10.x is usable. */
int pftg_device_ok(void);

/* Per-kernel timing hook (no reference counterpart; used by bench.py for the
 * roofline of the dominant kernel). While on, every kernel launch outside a
 * graph capture is bracketed by CUDA events on its own stream. profile_end
 * fills, per kernel id (0 pft rows fwd, 1 pft cols fwd, 2 pft cols adj,
 * 3 pft rows adj, 4 fft rows, 5 fft cols): summed milliseconds, timed launch
 * count and the number of launches issued since profile_begin, graph replays
 * included (arrays of 6). */
int pftg_profile_begin(void);
int pftg_profile_end(double* ms, int* count, int* launches);
/* Profiling mode for the next begin/end window: 0 = CUDA events around every
 * launch; 1 = the same, each launch preceded by a ~30 us device spin so its
 * events time the kernel rather than host-side submission gaps (replays only:
 * the spins lengthen the stream); 2 = launch counts only (no events: for
 * counting the launches of a timed region). */
int pftg_profile_mode(int mode);

/* ---- offline phase: scope table + plans (host) ---------------------------- */
/* ScopeTable::load (minimax.hpp:50, format minimax.cpp:470-522). */
int pftg_table_load(const char* path, pftg_table** out);
void pftg_table_free(pftg_table* t);
/* ScopeTable::min_degree (minimax.hpp:59). */
int pftg_table_min_degree(const pftg_table* t, double eps, double target_scope, int* r_out);

/* pft_plan_2d (pft.hpp:49-51): r = min_degree(eps, mt/p) per axis;
 * B[l,j] = w_j (1-2l/q)^j, W[t,j] = (t/p)^j e^{-i pi t/p}  (pft.cpp:33-76). */
/* ---- offline scope-table pipeline (minimax.hpp:28-70) ----
 * Own near-minimax solver (csrc/minimax.cpp), certified like the reference
 * (4097-point a-posteriori error); coefficients are near- (not bit-) identical. */
/* best_approx (minimax.hpp:28): coeff = r interleaved complex, achieved = certified error */
int pftg_best_approx(int r, double xi, double* coeff, double* achieved);
/* ScopeTable::compute (minimax.hpp:48-49); eps list (default 1e-1 .. 1e-7), r = 1..max_r */
int pftg_table_compute(const double* eps, int neps, int max_r, pftg_table** out);
int pftg_table_save(const pftg_table* t, const char* path); /* ScopeTable::save (minimax.hpp:51) */
int pftg_table_info(const pftg_table* t, int* nrec, int* max_r);
/* record i (eps-major, r ascending): coeff = r interleaved complex */
int pftg_table_record(const pftg_table* t, int i, double* eps, int* r, double* xi, double* achieved,
                      double* coeff);

/* ---- measurement-set directory (simulate.hpp:40-43, raw_io.hpp:10-27) ----
 * d [count][rows][cols], dcrop [count][2mt1][2mt2] (NULL: none, mt = 0). */
int pftg_measurements_save(const char* dir, size_t count, size_t rows, size_t cols, const double* d, size_t mt1,
                           size_t mt2, const double* dcrop, double noise_scale, uint64_t noise_seed);
/* verifies the manifest; info = count rows cols mt1 mt2 */
int pftg_measurements_info(const char* dir, int64_t* info, double* noise_scale, uint64_t* noise_seed);
/* host buffers in the GPU path's precision: float (PFTG_C64) or double (PFTG_C128); dcrop may be NULL */
int pftg_measurements_read(const char* dir, int dtype, void* d, void* dcrop);

int pftg_plan_2d(const pftg_table* t, size_t n1, size_t n2, size_t mt1, size_t mt2, size_t p1,
                 size_t p2, double eps, pftg_plan** out);
/* PftPlan2D from in-memory tables (pft.hpp:25-47): per axis n, p, mt, r and
 * the B (q x r, q = n/p) and W ((2mt+1) x r) tables, complex128 interleaved,
 * row-major exactly as PftPlan1D::B / ::W store them. The tables are copied; the
 * plan is immutable. Lets a C++ host that already holds a
 * ptycho::pft::PftPlan2D (built by the reference's pft_plan_2d) mirror it with
 * no file round trip. Shape rules as pft_plan_1d
 * (pft.cpp:35-40): PFTG_EINVAL otherwise. */
int pftg_plan_from_tables(size_t n1, size_t p1, size_t mt1, int r1, const double* B1, const double* W1,
                          size_t n2, size_t p2, size_t mt2, int r2, const double* B2, const double* W2,
                          double eps, pftg_plan** out);
/* load_plan_2d / save_plan (pft.hpp:60-63), "pft-plan-2d v1" + PTYC blocks. */
int pftg_plan_load(const char* path, pftg_plan** out);
int pftg_plan_save(const pftg_plan* plan, const char* path);
void pftg_plan_free(pftg_plan* plan);
/* info[10] = n1 p1 q1 mt1 r1 n2 p2 q2 mt2 r2 */
int pftg_plan_info(const pftg_plan* plan, int64_t* info);
/* Host copies of one axis' tables (axis 1 or 2): B (q x r), W ((2mt+1) x r),
 * complex128 interleaved. */
int pftg_plan_tables(const pftg_plan* plan, int axis, double* B, double* W);

/* ---- online phase: PFT operators -------------------------------------------- */
/* pft_apply_2d (pft.hpp:53): z [batch][n1][n2] -> band [batch][2mt1][2mt2]. */
int pftg_apply_2d_dev(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch,
                      void* stream);
/* pft_adjoint_2d (pft.hpp:57): band [batch][2mt1][2mt2] -> z [batch][n1][n2]. */
int pftg_adjoint_2d_dev(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch,
                        void* stream);
/* Host-buffer variants: copies are pipelined with compute over chunks of the
 * batch (pinned host memory recommended). */
int pftg_apply_2d_host(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch);
int pftg_adjoint_2d_host(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch);
/* BASELINE configs[1] in one streamed call: band = pft_apply_2d(z) and
 * back = pft_adjoint_2d(band) per field, host buffers, chunks pipelined on two
 * streams so H2D and D2H copies overlap (full-duplex PCIe). Results are
 * bit-identical to the two separate calls. */
int pftg_fwd_adj_2d_host(const pftg_plan* plan, int dtype, const void* z, void* band, void* back, size_t batch);
/* Multi-device forms of the three host-buffer calls for a C / C++ host that drives
 * several GPUs from ONE process (BASELINE configs[1]: "batch 64 ... sharded across
 * 1/2/4/8 GPUs"; fields are independent, pft.cpp:119-226): the batch is
 * split in contiguous blocks of batch / ndev fields (sizes differ by <= 1, the same
 * split as paper_2408_03532_b200.dist.shard_range) over devices[0 .. ndev), one host
 * thread per block running the streamed single-device call on its device. No
 * data-path collective; the union of the blocks is bit-identical to the
 * single-device result. A device may be listed more than once. The caller's
 * current device is unchanged. */
int pftg_apply_2d_host_multi(const pftg_plan* plan, int dtype, const void* z, void* band, size_t batch,
                             const int* devices, int ndev);
int pftg_adjoint_2d_host_multi(const pftg_plan* plan, int dtype, const void* band, void* z, size_t batch,
                               const int* devices, int ndev);
int pftg_fwd_adj_2d_host_multi(const pftg_plan* plan, int dtype, const void* z, void* band, void* back,
                               size_t batch, const int* devices, int ndev);

/* band_residual (solver.hpp:63): A*(A x - dcrop .* exp(i arg(A x))), batched;
 * dcrop is real [batch][2mt1][2mt2]. */
int pftg_band_residual_dev(const pftg_plan* plan, int dtype, const void* exit_wave, const void* dcrop,
                           void* out, size_t batch, void* stream);

/* ---- full transforms and modulus projection -------------------------------- */
/* fast_fft2 / fast_ifft2 (fft.hpp:18-19): power-of-two rows, cols in [2, 1024]. */
int pftg_fft2_dev(int dtype, const void* z, void* out, size_t rows, size_t cols, size_t batch,
                  int inverse, void* stream);
/* Host-buffer fast_fft2 / fast_ifft2 (copies pipelined with compute over
 * chunks of the batch), for hosts that keep fields in host memory (the C++
 * façade of INTEGRATION.md). */
int pftg_fft2_host(int dtype, const void* z, void* out, size_t rows, size_t cols, size_t batch, int inverse);
/* project_modulus (solver.hpp:51): F^-1[d .* exp(i arg(F x))], phase 1 where F x == 0. */
int pftg_project_modulus_dev(int dtype, const void* exit_wave, const void* d, void* out, size_t rows,
                             size_t cols, size_t batch, void* stream);
/* crop_centered(RealField) (fft.hpp:30). */
int pftg_crop_centered_dev(int dtype, const void* spectrum, void* out, size_t rows, size_t cols,
                           size_t mt1, size_t mt2, size_t batch, void* stream);

/* ---- scan geometry and updates ---------------------------------------------- */
/* window_slice / set_window (scan.hpp:40-42): patches [batch][wr][wc] at
 * (offsets[2k], offsets[2k+1]) of a fr x fc frame. offsets are HOST int64
 * pairs. Unlike the reference (scan.cpp:14-22, unchecked) every window is
 * bounds-checked: PFTG_ERANGE if it leaves the frame (a device-side overrun
 * would leave the CUDA context unusable). */
int pftg_window_slice_dev(int dtype, const void* frame, size_t fr, size_t fc, void* patches,
                          size_t wr, size_t wc, const int64_t* offsets, size_t npos, void* stream);
int pftg_set_window_dev(int dtype, void* frame, size_t fr, size_t fc, const void* patch, size_t wr,
                        size_t wc, int64_t r0, int64_t c0, void* stream);
/* pie_object_update (solver.hpp:54): zj <- zj - beta conj(P) (P zj - proj). */
int pftg_pie_object_update_dev(int dtype, void* zj, const void* probe, const void* proj, size_t n,
                               double beta, void* stream);
/* epie_probe_update (solver.hpp:59): P <- P - gamma conj(zj) (P zj - proj);
 * PFTG_ELOGIC unless blind. */
int pftg_epie_probe_update_dev(int dtype, void* probe, const void* zj, const void* proj, size_t n,
                               double gamma, int blind, void* stream);

/* ---- forward model / residual evaluator ------------------------------------- */
/* objective_value (solver.hpp:70) restricted to positions [pos_begin, pos_end):
 * returns sum_j ||P z_j - P_M(P z_j)||^2 (NOT divided by N; the caller divides
 * by the global N after summing over shards). d: [npos][wr][wc] real, device.
 * offsets: HOST int64 pairs for all npos positions. If plan != NULL also
 * returns band_sum = sum_j || |PFT(P z_j)| - dcrop_j ||^2 (dcrop device,
 * [npos][2mt1][2mt2]); otherwise band_sum is untouched.
 * Synchronizes the stream. */
int pftg_evaluate_dev(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr,
                      size_t wc, const int64_t* offsets, size_t npos, size_t pos_begin, size_t pos_end,
                      const void* d, const pftg_plan* plan, const void* dcrop, double* fft_sum,
                      double* band_sum, void* stream);

/* ---- measurement simulator (simulate.hpp:33-42) ------------------------------ */
/* simulate (simulate.cpp:48-65): d[j] = |FFT2(probe .* window_j)| for the npos
 * windows at HOST int64 offsets (r0, c0) of the fr x fc frame; d is real
 * [npos][wr][wc] (float for PFTG_C64, double for PFTG_C128). Windows are
 * bounds-checked (PFTG_ERANGE). Synchronizes the stream. build_cropped
 * (simulate.cpp:81-89) is pftg_crop_centered_dev over the same d. */
int pftg_simulate_dev(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr, size_t wc,
                      const int64_t* offsets, size_t npos, void* d, void* stream);
/* add_poisson_noise (simulate.cpp:67-79): d <- sqrt(Poisson(scale d^2) / scale)
 * over n real elements, in place. Same law as the reference; the random stream
 * is counter-based (Philox-4x32-10 keyed by seed, counter = element index;
 * inversion for lambda < 10, Hoermann PTRS above), not libstdc++'s: results
 * are reproducible for a given seed and independent of the launch shape.
 * PFTG_EINVAL unless scale > 0. */
int pftg_add_poisson_noise_dev(int dtype, void* d, size_t n, double scale, uint64_t seed, void* stream);

/* ---- per-sweep reconstruction metrics (metrics.hpp:11-34) -------------------- */
/* fill_metrics (solver.cpp:141-160) of a reconstruction x against the truth ref,
 * both rows x cols complex regions with leading dimensions ld_x / ld_ref
 * (elements; e.g. the object region inside a frame): out[8] = relative_error,
 * relative_error_aligned, relative_error(|x|), relative_error(arg x),
 * ssim(|x|), ssim(arg x), psnr(|x|), psnr(arg x), ranges = dynamic_range of
 * the truth (metrics.cpp:60-143). FP64 accumulation, deterministic.
 * Synchronizes the stream. PFTG_EINVAL for regions under 11 x 11 (ssim). */
int pftg_fill_metrics_dev(int dtype, const void* x, size_t ld_x, const void* ref, size_t ld_ref, size_t rows,
                          size_t cols, double* out, void* stream);

/* ---- 1-D PFT (pft.hpp:25-38, 60-63; pft.cpp:33-101, 266-334) ---------------- */
typedef struct pftg_plan1d pftg_plan1d; /* pft::PftPlan1D (pft.hpp:25-31) */
/* pft::pft_plan_1d (pft.hpp:33-34): r = min_degree(eps, mt/p), same tables and errors. */
int pftg_plan_1d(const pftg_table* t, size_t n, size_t mt, size_t p, double eps, pftg_plan1d** out);
/* In-memory PftPlan1D (B: q x r, W: (2mt+1) x r, interleaved complex128). */
int pftg_plan1d_from_tables(size_t n, size_t p, size_t mt, int r, const double* B, const double* W, double eps,
                            pftg_plan1d** out);
int pftg_plan1d_load(const char* path, pftg_plan1d** out);        /* load_plan_1d (pft.hpp:62) */
int pftg_plan1d_save(const pftg_plan1d* plan, const char* path);  /* save_plan (pft.hpp:60) */
int pftg_plan1d_info(const pftg_plan1d* plan, int64_t* info);     /* n p q mt r */
int pftg_plan1d_tables(const pftg_plan1d* plan, double* B, double* W);
void pftg_plan1d_free(pftg_plan1d* plan);
/* pft::pft_apply_1d (pft.hpp:38): z [batch][n] -> out [batch][2mt+1], DC at index mt
 * (the +mt edge is kept in 1-D). Device buffers, stream-ordered. */
int pftg_apply_1d_dev(const pftg_plan1d* plan, int dtype, const void* z, void* out, size_t batch, void* stream);
/* The same from host buffers (synchronous). */
int pftg_apply_1d_host(const pftg_plan1d* plan, int dtype, const void* z, void* out, size_t batch);

/* ---- device-resident hybrid_solve (solver.hpp:87-90) ------------------------ */
typedef struct pftg_solver_config {
  int pft_sweeps, fft_sweeps;      /* SolverConfig (solver.hpp:21-37) */
  double beta, gamma, beta_pft, gamma_pft, eps_pft, tol;
  int64_t mt1, mt2, p1, p2;        /* 0 -> window/8 and mt (solver.cpp:195-198) */
  int blind;
  int shuffled;                    /* VisitOrder::shuffled */
  uint64_t seed;
  int objective_every;             /* evaluate objective every k sweeps (1 = reference) */
  double tv_lambda_mag, tv_lambda_phase; /* per-sweep TV step on |z| / arg z (solver.cpp:264-279) */
} pftg_solver_config;

/* Copies the HOST inputs to the device: frame [fr][fc], probe [wr][wc],
 * offsets int64 pairs [npos][2] (visit order), d [npos][wr][wc] real.
 * table may be NULL when pft_sweeps == 0 (solver.cpp:199). */
int pftg_solver_create(int dtype, const void* frame, size_t fr, size_t fc, const void* probe, size_t wr,
                       size_t wc, const int64_t* offsets, size_t npos, const void* d,
                       const pftg_solver_config* cfg, const pftg_table* table, pftg_solver** out);
/* Runs all remaining sweeps (or at most max_sweeps if > 0). */
int pftg_solver_run(pftg_solver* s, int max_sweeps);
/* Per completed sweep: objective and cumulative device seconds. */
int pftg_solver_trace(const pftg_solver* s, double* objective, double* wall_s, int* sweeps_run,
                      int* flags /* 1 diverged, 2 stopped early */);
int pftg_solver_result(const pftg_solver* s, void* frame, void* probe); /* host copies */
/* Device pointers to the live frame / probe (for device-side consumers). */
int pftg_solver_device_state(const pftg_solver* s, void** frame, void** probe);
void pftg_solver_free(pftg_solver* s);

#ifdef __cplusplus
}
#endif

#endif /* PFTG_H_ */
