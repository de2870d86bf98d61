"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the reference library.

Loads ``oracle/_ref/libptycho_ref.so``: the UNMODIFIED reference ``proj/core``
TUs compiled from /root/reference by ``oracle/Makefile`` (Eigen/FFTW replaced by
the shims in ``oracle/shim``), plus ``oracle/ref_capi.cpp``. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s reference / cpu_baseline legs may
import this module; the product never does.

Every wrapper names the reference function it calls (file:line into
/root/reference/proj/core).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libptycho_ref.so"
# The same verbatim reference library with pft_apply_2d / pft_adjoint_2d /
# fast_fft2 / fast_ifft2 provided by the C++ façade over libpftg
# (paper_2408_03532_b200/facade/pft_gpu.cpp; oracle/Makefile): the drop-in
# demonstration. Selected with ``with ref.facade(): ...``.
FACADE_PATH = HERE / "_ref" / "libptycho_facade.so"

_libs = {}
_active = [LIB_PATH]


def available() -> bool:
    return LIB_PATH.exists()


class facade:
    """Context manager: route every wrapper below through libptycho_facade.so."""

    def __enter__(self):
        if not FACADE_PATH.exists():
            raise RuntimeError(f"façade build missing: {FACADE_PATH} (run make -C oracle)")
        _active.append(FACADE_PATH)
        return self

    def __exit__(self, *exc):
        _active.pop()
        return False


def lib():
    path = _active[-1]
    if path not in _libs:
        if not path.exists():
            raise RuntimeError(f"reference oracle not built: {path} (run make -C oracle)")
        L = C.CDLL(str(path))
        vp, dp, szt, i64p = C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_int64)
        L.ref_last_error.restype = C.c_char_p
        L.ref_plan_create.restype = vp
        L.ref_plan_create.argtypes = [C.c_char_p, szt, szt, szt, szt, szt, szt, C.c_double]
        L.ref_plan_load.restype = vp
        L.ref_plan_load.argtypes = [C.c_char_p]
        L.ref_plan_save.argtypes = [vp, C.c_char_p]
        L.ref_plan_free.argtypes = [vp]
        L.ref_plan_info.argtypes = [vp, i64p]
        L.ref_plan_tables.argtypes = [vp, C.c_int, dp, dp]
        L.ref_pft_apply_2d.argtypes = [vp, dp, szt, szt, dp]
        L.ref_plan1d_create.restype = vp
        L.ref_plan1d_create.argtypes = [C.c_char_p, szt, szt, szt, C.c_double]
        L.ref_plan1d_load.restype = vp
        L.ref_plan1d_load.argtypes = [C.c_char_p]
        L.ref_plan1d_save.argtypes = [vp, C.c_char_p]
        L.ref_plan1d_free.argtypes = [vp]
        L.ref_plan1d_info.argtypes = [vp, i64p]
        L.ref_plan1d_tables.argtypes = [vp, dp, dp]
        L.ref_pft_apply_1d.argtypes = [vp, dp, szt, dp]
        L.ref_pft_adjoint_2d.argtypes = [vp, dp, szt, szt, dp]
        L.ref_pft_fwd_adj_batch.argtypes = [vp, dp, szt, szt, szt, dp, dp, C.c_int]
        for f in ("ref_fast_fft2", "ref_fast_ifft2", "ref_naive_dft2", "ref_naive_idft2"):
            getattr(L, f).argtypes = [dp, szt, szt, dp]
        L.ref_crop_centered_real.argtypes = [dp, szt, szt, szt, szt, dp]
        L.ref_project_modulus.argtypes = [dp, dp, szt, szt, dp]
        L.ref_band_residual.argtypes = [vp, dp, szt, szt, dp, szt, szt, dp]
        L.ref_pie_object_update.argtypes = [dp, dp, dp, szt, szt, C.c_double]
        L.ref_epie_probe_update.argtypes = [dp, dp, dp, szt, szt, C.c_double, C.c_int]
        L.ref_objective_value.argtypes = [dp, szt, szt, dp, szt, szt, i64p, szt, dp, dp]
        L.ref_simulate.argtypes = [dp, szt, szt, dp, szt, szt, i64p, szt, dp]
        L.ref_save_measurements.argtypes = [C.c_char_p, dp, szt, szt, szt, szt, szt, C.c_double, C.c_uint64]
        L.ref_load_measurements.argtypes = [C.c_char_p, i64p, dp, dp, dp]
        L.ref_add_poisson_noise.argtypes = [dp, szt, szt, szt, C.c_double, C.c_uint64]
        L.ref_hybrid_solve.argtypes = [dp, szt, szt, dp, szt, szt, i64p, szt, dp, dp, i64p,
                                       C.c_char_p, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_best_approx.argtypes = [C.c_int, C.c_double, dp, dp, C.POINTER(C.c_int)]
        L.ref_scope_table_compute.argtypes = [C.c_char_p, dp, C.c_int, C.c_int]
        L.ref_scope_table_single.argtypes = [C.c_char_p, C.c_double, C.c_int, C.c_double]
        L.ref_min_degree.argtypes = [C.c_char_p, C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.ref_fill_metrics.argtypes = [dp, dp, szt, szt, dp]
        L.ref_shim_gemm_gflops.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp]
        _libs[path] = L
    return _libs[path]


class RefError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        if msg.startswith("invalid_argument"):
            raise ValueError(msg)
        raise RefError(msg)


def _cptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _c128(z) -> np.ndarray:
    return np.ascontiguousarray(z, dtype=np.complex128)


def _f64(d) -> np.ndarray:
    return np.ascontiguousarray(d, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


class RefPlan:
    """Handle on a reference ``PftPlan2D`` (pft.hpp:44-47)."""

    def __init__(self, handle):
        if not handle:
            _check(1)
        self._L = lib()  # the library that owns the handle (reference or façade build)
        self.h = C.c_void_p(handle)
        info = np.zeros(10, np.int64)
        self._L.ref_plan_info(self.h, info.ctypes.data_as(C.POINTER(C.c_int64)))
        (self.n1, self.p1, self.q1, self.mt1, self.r1,
         self.n2, self.p2, self.q2, self.mt2, self.r2) = (int(v) for v in info)

    @classmethod
    def create(cls, table_path, n1, n2, mt1, mt2, p1, p2, eps):
        """pft_plan_2d (pft.cpp:103-112)."""
        return cls(lib().ref_plan_create(str(table_path).encode(), n1, n2, mt1, mt2, p1, p2, eps))

    @classmethod
    def load(cls, plan_path):
        """load_plan_2d (pft.cpp:336-366)."""
        return cls(lib().ref_plan_load(str(plan_path).encode()))

    def save(self, plan_path):
        """save_plan (pft.cpp:277-289)."""
        _check(self._L.ref_plan_save(self.h, str(plan_path).encode()))

    def tables(self, axis: int):
        q, r, mt = (self.q1, self.r1, self.mt1) if axis == 1 else (self.q2, self.r2, self.mt2)
        B = np.zeros((q, r), np.complex128)
        W = np.zeros((2 * mt + 1, r), np.complex128)
        self._L.ref_plan_tables(self.h, axis, _cptr(B), _cptr(W))
        return B, W

    def __del__(self):
        try:
            self._L.ref_plan_free(self.h)
        except Exception:
            pass

    def apply(self, z):
        """pft_apply_2d (pft.cpp:119-172)."""
        z = _c128(z)
        out = np.zeros((2 * self.mt1, 2 * self.mt2), np.complex128)
        _check(self._L.ref_pft_apply_2d(self.h, _cptr(z), z.shape[0], z.shape[1], _cptr(out)))
        return out

    def adjoint(self, band):
        """pft_adjoint_2d (pft.cpp:174-226)."""
        band = _c128(band)
        out = np.zeros((self.n1, self.n2), np.complex128)
        _check(self._L.ref_pft_adjoint_2d(self.h, _cptr(band), band.shape[0], band.shape[1],
                                        _cptr(out)))
        return out

    def fwd_adj_batch(self, z, threads=1, want=True):
        z = _c128(z)
        b = z.shape[0]
        band = np.zeros((b, 2 * self.mt1, 2 * self.mt2), np.complex128) if want else None
        back = np.zeros_like(z) if want else None
        _check(self._L.ref_pft_fwd_adj_batch(
            self.h, _cptr(z), b, self.n1, self.n2,
            _cptr(band) if want else None, _cptr(back) if want else None, threads))
        return band, back

    def band_residual(self, exit_wave, dcrop):
        """band_residual (solver.cpp:61-69)."""
        e, d = _c128(exit_wave), _f64(dcrop)
        out = np.zeros_like(e)
        _check(self._L.ref_band_residual(self.h, _cptr(e), e.shape[0], e.shape[1], _cptr(d),
                                       d.shape[0], d.shape[1], _cptr(out)))
        return out


class RefPlan1D:
    """Handle on a reference ``PftPlan1D`` (pft.hpp:25-31)."""

    def __init__(self, handle):
        if not handle:
            _check(1)
        self._L = lib()
        self.h = C.c_void_p(handle)
        info = np.zeros(5, np.int64)
        self._L.ref_plan1d_info(self.h, info.ctypes.data_as(C.POINTER(C.c_int64)))
        self.n, self.p, self.q, self.mt, self.r = (int(v) for v in info)

    @classmethod
    def create(cls, table_path, n, mt, p, eps):
        """pft_plan_1d (pft.cpp:33-76)."""
        return cls(lib().ref_plan1d_create(str(table_path).encode(), n, mt, p, eps))

    @classmethod
    def load(cls, plan_path):
        """load_plan_1d (pft.cpp:310-334)."""
        return cls(lib().ref_plan1d_load(str(plan_path).encode()))

    def save(self, plan_path):
        """save_plan(PftPlan1D) (pft.cpp:266-275)."""
        _check(self._L.ref_plan1d_save(self.h, str(plan_path).encode()))

    def tables(self):
        B = np.zeros((self.q, self.r), np.complex128)
        W = np.zeros((2 * self.mt + 1, self.r), np.complex128)
        self._L.ref_plan1d_tables(self.h, _cptr(B), _cptr(W))
        return B, W

    def __del__(self):
        try:
            self._L.ref_plan1d_free(self.h)
        except Exception:
            pass

    def apply(self, z):
        """pft_apply_1d (pft.cpp:78-101): 2mt+1 band entries, DC at index mt."""
        z = _c128(z).reshape(-1)
        out = np.zeros(2 * self.mt + 1, np.complex128)
        _check(self._L.ref_pft_apply_1d(self.h, _cptr(z), z.shape[0], _cptr(out)))
        return out


def _unary(fname, z):
    z = _c128(z)
    out = np.zeros_like(z)
    _check(getattr(lib(), fname)(_cptr(z), z.shape[0], z.shape[1], _cptr(out)))
    return out


def fast_fft2(z):
    """fast_fft2 (fft.cpp:175-178), FFTW replaced by oracle/shim."""
    return _unary("ref_fast_fft2", z)


def fast_ifft2(z):
    """fast_ifft2 (fft.cpp:180-183)."""
    return _unary("ref_fast_ifft2", z)


def naive_dft2(z):
    """naive_dft2 (fft.cpp:132-146): exact-phase O(n^2) oracle."""
    return _unary("ref_naive_dft2", z)


def naive_idft2(z):
    return _unary("ref_naive_idft2", z)


def crop_centered(d, mt1, mt2):
    """crop_centered(RealField) (fft.cpp:206-232)."""
    d = _f64(d)
    out = np.zeros((2 * mt1, 2 * mt2))
    _check(lib().ref_crop_centered_real(_cptr(d), d.shape[0], d.shape[1], mt1, mt2, _cptr(out)))
    return out


def project_modulus(exit_wave, d):
    """project_modulus (solver.cpp:35-42)."""
    e, d = _c128(exit_wave), _f64(d)
    out = np.zeros_like(e)
    _check(lib().ref_project_modulus(_cptr(e), _cptr(d), e.shape[0], e.shape[1], _cptr(out)))
    return out


def pie_object_update(zj, probe, proj, beta):
    """pie_object_update (solver.cpp:44-50); returns the updated patch."""
    z = _c128(zj).copy()
    p, q = _c128(probe), _c128(proj)
    _check(lib().ref_pie_object_update(_cptr(z), _cptr(p), _cptr(q), z.shape[0], z.shape[1], beta))
    return z


def epie_probe_update(probe, zj, proj, gamma, blind=True):
    """epie_probe_update (solver.cpp:52-59); returns the updated probe."""
    p = _c128(probe).copy()
    z, q = _c128(zj), _c128(proj)
    _check(lib().ref_epie_probe_update(_cptr(p), _cptr(z), _cptr(q), p.shape[0], p.shape[1],
                                       gamma, int(blind)))
    return p


def objective_value(frame, probe, offsets, d):
    """objective_value (solver.cpp:89-102)."""
    f, p, o, d = _c128(frame), _c128(probe), _i64(offsets), _f64(d)
    out = np.zeros(1)
    _check(lib().ref_objective_value(_cptr(f), f.shape[0], f.shape[1], _cptr(p), p.shape[0],
                                     p.shape[1], o.ctypes.data_as(C.POINTER(C.c_int64)), len(o),
                                     _cptr(d), _cptr(out)))
    return float(out[0])


def simulate(frame, probe, offsets):
    """simulate (simulate.cpp:48-65): d_j = |fft2(probe * patch_j)|."""
    f, p, o = _c128(frame), _c128(probe), _i64(offsets)
    d = np.zeros((len(o), p.shape[0], p.shape[1]))
    _check(lib().ref_simulate(_cptr(f), f.shape[0], f.shape[1], _cptr(p), p.shape[0], p.shape[1],
                              o.ctypes.data_as(C.POINTER(C.c_int64)), len(o), _cptr(d)))
    return d


def save_measurements(path, d, mt=0, noise_scale=0.0, noise_seed=0):
    """save_measurements (simulate.cpp:91-127); build_cropped(mt) first when mt > 0."""
    d = _f64(d)
    _check(lib().ref_save_measurements(str(path).encode(), _cptr(d), d.shape[0], d.shape[1], d.shape[2],
                                       mt, mt, noise_scale, noise_seed))


def load_measurements(path):
    """load_measurements (simulate.cpp:129-164) -> (d, dcrop or None, (scale, seed))."""
    info = np.zeros(5, np.int64)
    noise = np.zeros(2)
    _check(lib().ref_load_measurements(str(path).encode(), info.ctypes.data_as(C.POINTER(C.c_int64)),
                                       _cptr(noise), None, None))
    cnt, r, c, m1, m2 = (int(v) for v in info)
    d = np.zeros((cnt, r, c))
    dc = np.zeros((cnt, 2 * m1, 2 * m2)) if m1 else None
    _check(lib().ref_load_measurements(str(path).encode(), info.ctypes.data_as(C.POINTER(C.c_int64)),
                                       _cptr(noise), _cptr(d), _cptr(dc) if dc is not None else None))
    return d, dc, (float(noise[0]), int(noise[1]))


def add_poisson_noise(d, scale, seed):
    """add_poisson_noise (simulate.cpp:67-79), libstdc++ poisson_distribution."""
    d = _f64(d).copy()
    _check(lib().ref_add_poisson_noise(_cptr(d), d.shape[1], d.shape[2], d.shape[0], scale,
                                       seed))
    return d


def hybrid_solve(frame, probe, offsets, d, *, pft_sweeps, fft_sweeps, beta=1.0, gamma=1.0,
                 beta_pft=1e-3, gamma_pft=1e-3, eps_pft=1e-3, tol=0.0, mt=0, p=0,
                 blind=False, shuffled=False, seed=0, table_path=None, tv_mag=0.0, tv_phase=0.0):
    """hybrid_solve (solver.cpp:173-302). Returns (frame, probe, objectives, walls, flags)."""
    f, pr = _c128(frame).copy(), _c128(probe).copy()
    o, d = _i64(offsets), _f64(d)
    cfg_d = np.array([beta, gamma, beta_pft, gamma_pft, eps_pft, tol, tv_mag, tv_phase])
    cfg_i = np.array([pft_sweeps, fft_sweeps, mt, mt, p, p, int(blind), int(shuffled), seed],
                     np.int64)
    total = pft_sweeps + fft_sweeps
    trace = np.zeros(2 * max(total, 1))
    sweeps, flags = C.c_int(0), C.c_int(0)
    _check(lib().ref_hybrid_solve(
        _cptr(f), f.shape[0], f.shape[1], _cptr(pr), pr.shape[0], pr.shape[1],
        o.ctypes.data_as(C.POINTER(C.c_int64)), len(o), _cptr(d), _cptr(cfg_d),
        cfg_i.ctypes.data_as(C.POINTER(C.c_int64)),
        (str(table_path).encode() if table_path else b""), _cptr(trace),
        C.byref(sweeps), C.byref(flags)))
    n = sweeps.value
    return f, pr, trace[0:2 * n:2].copy(), trace[1:2 * n:2].copy(), flags.value


def best_approx(r, xi):
    """minimax::best_approx (minimax.cpp:276-342)."""
    c = np.zeros(2 * r)
    ach = C.c_double(0)
    conv = C.c_int(0)
    _check(lib().ref_best_approx(r, xi, _cptr(c), C.byref(ach), C.byref(conv)))
    return c[0::2] + 1j * c[1::2], ach.value, bool(conv.value)


def scope_table_compute(path, eps_list=(1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7), max_r=25):
    """ScopeTable::compute + save (minimax.cpp:388-433, 470-493)."""
    e = np.asarray(eps_list, np.float64)
    _check(lib().ref_scope_table_compute(str(path).encode(), _cptr(e), len(e), max_r))


def scope_table_single(path, eps, r, xi):
    _check(lib().ref_scope_table_single(str(path).encode(), eps, r, xi))


def min_degree(table_path, eps, target):
    """ScopeTable::min_degree (minimax.cpp:455-468)."""
    r = C.c_int(0)
    _check(lib().ref_min_degree(str(table_path).encode(), eps, target, C.byref(r)))
    return r.value


def fill_metrics(x, truth):
    """fill_metrics (solver.cpp:141-160) via metrics.cpp:60-143: [rel_err,
    rel_err_aligned, rel_err_mag, rel_err_phase, ssim_mag, ssim_phase, psnr_mag,
    psnr_phase]."""
    x, t = _c128(x), _c128(truth)
    out = np.zeros(8)
    _check(lib().ref_fill_metrics(_cptr(x), _cptr(t), x.shape[0], x.shape[1], _cptr(out)))
    return out


def shim_gemm_gflops(m=10, k=32, n=1024, reps=200):
    """GFLOP/s of the Eigen shim's complex GEMM on the PFT stage-A shape."""
    g = C.c_double(0)
    _check(lib().ref_shim_gemm_gflops(m, k, n, reps, C.byref(g)))
    return g.value


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
