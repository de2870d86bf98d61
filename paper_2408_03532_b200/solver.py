"""Python mirror of the reference's solver building blocks and driver
(/root/reference/proj/core/include/ptycho/{solver,scan}.hpp) over libpftg.

=============================  ==================================================
reference                      here
=============================  ==================================================
project_modulus                ``project_modulus(exit, d)``          (solver.hpp:51)
pie_object_update              ``pie_object_update(zj, P, proj, b)`` (solver.hpp:54)
epie_probe_update              ``epie_probe_update(P, zj, proj, g, blind)`` (solver.hpp:59)
window_slice / set_window      ``window_slice`` / ``set_window``     (scan.hpp:40-42)
objective_value                ``objective_value(frame, probe, offsets, d)`` (solver.hpp:70)
SolverConfig / hybrid_solve    ``SolverConfig`` / ``hybrid_solve``   (solver.hpp:21-37, 87-90)
solve_pie / solve_epie         ``solve_pie`` / ``solve_epie``        (solver.hpp:93-98)
=============================  ==================================================

Scan positions are given as an (N, 2) int64 array of window top-left corners
in visit order (ScanPattern::offsets, scan.hpp:20), measurements ``d`` as an
(N, wr, wc) real array (MeasurementSet::d, simulate.hpp:17).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

import numpy as np
import torch

from ._lib import PFTG_C64, PFTG_C128, SolverConfigC, check, lib
from .pft import PftPlan2D, ScopeTable, _batch, _dev, _dtype_code, _ptr, _real_of, _stream


def _inplace(t, what):
    """In-place targets must be contiguous CUDA tensors (the kernels write raw memory)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what}: expected a CUDA torch tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what}: in-place target must be contiguous")
    return t


def _match(ref, what, *others):
    """Operands must share the reference tensor's dtype and device (no silent casts)."""
    for o in others:
        if not isinstance(o, torch.Tensor) or o.dtype != ref.dtype or o.device != ref.device:
            raise ValueError(f"{what}: operands must have dtype {ref.dtype} on {ref.device}")


def project_modulus(exit_wave, d):
    """F^-1[d .* exp(i arg(F x))]; zero spectrum bins keep phase 1 (solver.cpp:35-42)."""
    x = _dev(exit_wave)
    rows, cols = x.shape[-2:]
    dd = _dev(d).to(_real_of(x))
    if tuple(dd.shape) != tuple(x.shape):
        raise ValueError("project_modulus: shape mismatch")
    out = torch.empty_like(x)
    check(lib().pftg_project_modulus_dev(_dtype_code(x), _ptr(x), _ptr(dd), _ptr(out), rows, cols,
                                         _batch(x, (rows, cols)), _stream()))
    return out


def pie_object_update(zj, probe, projected, beta):
    """In place: zj -= beta conj(P) (P zj - proj) (solver.cpp:44-50)."""
    if zj.shape != probe.shape or zj.shape != projected.shape:
        raise ValueError("pie_object_update: shape mismatch")
    _inplace(zj, "pie_object_update")
    _match(zj, "pie_object_update", probe, projected)
    p, q = _dev(probe), _dev(projected)
    check(lib().pftg_pie_object_update_dev(_dtype_code(zj), _ptr(zj), _ptr(p), _ptr(q), zj.numel(),
                                           float(beta), _stream()))
    return zj


def epie_probe_update(probe, zj, projected, gamma, blind):
    """In place: P -= gamma conj(zj) (P zj - proj); needs blind (solver.cpp:52-59)."""
    if not blind:
        raise RuntimeError("epie_probe_update: probe updates need blind mode")
    if zj.shape != probe.shape or zj.shape != projected.shape:
        raise ValueError("epie_probe_update: shape mismatch")
    _inplace(probe, "epie_probe_update")
    _match(probe, "epie_probe_update", zj, projected)
    z, q = _dev(zj), _dev(projected)
    check(lib().pftg_epie_probe_update_dev(_dtype_code(probe), _ptr(probe), _ptr(z), _ptr(q),
                                           probe.numel(), float(gamma), int(blind), _stream()))
    return probe


def _offsets(offsets) -> np.ndarray:
    o = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64).reshape(-1, 2))
    return o


def window_slice(frame, offsets, wr, wc):
    """Patches of every listed position (scan.cpp:105-109), shape (N, wr, wc)."""
    f = _dev(frame)
    o = _offsets(offsets)
    out = torch.empty((len(o), wr, wc), dtype=f.dtype, device=f.device)
    check(lib().pftg_window_slice_dev(_dtype_code(f), _ptr(f), f.shape[0], f.shape[1], _ptr(out),
                                      wr, wc, o.ctypes.data_as(C.POINTER(C.c_int64)), len(o),
                                      _stream()))
    return out


def set_window(frame, offset, patch):
    """In place: frame[r0:r0+wr, c0:c0+wc] = patch (scan.cpp:111-121)."""
    _inplace(frame, "set_window")
    _match(frame, "set_window", patch)
    if frame.dim() != 2 or patch.dim() != 2:
        raise ValueError("set_window: frame and patch must be 2-D")
    p = _dev(patch)
    r0, c0 = (int(v) for v in offset)
    check(lib().pftg_set_window_dev(_dtype_code(frame), _ptr(frame), frame.shape[0], frame.shape[1],
                                    _ptr(p), p.shape[0], p.shape[1], r0, c0, _stream()))
    return frame


def evaluate(frame, probe, offsets, d, pos_range=None, plan: PftPlan2D | None = None,
             d_crop=None):
    """Forward-model / residual evaluator over positions [b, e).

    Returns (fft_sum, band_sum): fft_sum = sum_j ||P z_j - P_M(P z_j)||^2
    (objective_value numerator, solver.cpp:89-102) and, with a band plan,
    band_sum = sum_j || |PFT(P z_j)| - d_crop_j ||^2 (else None).
    """
    f, p = _dev(frame), _dev(probe)
    _match(f, "evaluate", p)
    o = _offsets(offsets)
    dd = _dev(d).to(_real_of(f))
    b, e = pos_range if pos_range is not None else (0, len(o))
    if not 0 <= b <= e <= len(o):
        raise IndexError("evaluate: position range outside the scan")
    wr, wc = p.shape[-2:]
    if dd.dim() != 3 or tuple(dd.shape[1:]) != (wr, wc) or dd.shape[0] < e:
        raise ValueError(f"evaluate: d must be (>= {e}, {wr}, {wc}), got {tuple(dd.shape)}")
    fs, bs = C.c_double(0.0), C.c_double(0.0)
    dc = None
    if plan is not None:
        dc = _dev(d_crop).to(_real_of(f))
        if dc.dim() != 3 or tuple(dc.shape[1:]) != plan.band_shape or dc.shape[0] < e:
            raise ValueError(f"evaluate: d_crop must be (>= {e}, {plan.band_shape[0]}, "
                             f"{plan.band_shape[1]}), got {tuple(dc.shape)}")
        if plan.field_shape != (wr, wc):
            raise ValueError("band_residual: plan does not match the window shape")
    check(lib().pftg_evaluate_dev(
        _dtype_code(f), _ptr(f), f.shape[0], f.shape[1], _ptr(p), p.shape[0], p.shape[1],
        o.ctypes.data_as(C.POINTER(C.c_int64)), len(o), b, e, _ptr(dd),
        plan._h if plan is not None else None, _ptr(dc) if dc is not None else None,
        C.byref(fs), C.byref(bs), _stream()))
    return fs.value, (bs.value if plan is not None else None)


def objective_value(frame, probe, offsets, d) -> float:
    """Phi = (1/N) sum_j ||P z_j - P_M(P z_j)||^2 (solver.hpp:70)."""
    o = _offsets(offsets)
    if len(o) != d.shape[0]:
        raise ValueError("objective_value: measurement/pattern count mismatch")
    s, _ = evaluate(frame, probe, o, d)
    return s / len(o)


@dataclasses.dataclass
class SolverConfig:
    """ptycho::SolverConfig (solver.hpp:21-37)."""
    pft_sweeps: int = 0
    fft_sweeps: int = 50
    beta: float = 1.0
    gamma: float = 1.0
    beta_pft: float = 1e-3
    gamma_pft: float = 1e-3
    eps_pft: float = 1e-3
    mt1: int = 0
    mt2: int = 0
    p1: int = 0
    p2: int = 0
    tol: float = 0.0
    tv_lambda_mag: float = 0.0
    tv_lambda_phase: float = 0.0
    blind: bool = False
    shuffled: bool = False
    seed: int = 0
    objective_every: int = 1


@dataclasses.dataclass
class ReconResult:
    """ptycho::ReconResult (solver.hpp:39-46); trace = per-sweep (objective, wall_s)."""
    frame: object
    probe: object
    objective: np.ndarray
    wall_s: np.ndarray
    sweeps_run: int
    stopped_early: bool
    diverged: bool


class Solver:
    """Device-resident hybrid_solve state; ``run()`` advances sweeps."""

    def __init__(self, d, offsets, probe_init, object_init, cfg: SolverConfig,
                 table: ScopeTable | None = None, dtype=np.complex64):
        cdt = np.dtype(dtype)
        rdt = np.float32 if cdt == np.complex64 else np.float64
        self.code = PFTG_C64 if cdt == np.complex64 else PFTG_C128
        self.cdt = cdt
        obj = np.ascontiguousarray(np.asarray(object_init), dtype=cdt)
        pr = np.ascontiguousarray(np.asarray(probe_init), dtype=cdt)
        dd = np.ascontiguousarray(np.asarray(d), dtype=rdt)
        o = _offsets(offsets)
        if dd.shape[0] != len(o):
            raise ValueError("hybrid_solve: measurement/pattern count mismatch")
        if dd.shape[1:] != pr.shape:
            raise ValueError("hybrid_solve: measurement window mismatch")
        if cfg.pft_sweeps > 0 and table is None:
            table = ScopeTable.load()
        self.cfg = cfg
        self.shapes = (obj.shape, pr.shape)
        c = SolverConfigC(cfg.pft_sweeps, cfg.fft_sweeps, cfg.beta, cfg.gamma, cfg.beta_pft,
                          cfg.gamma_pft, cfg.eps_pft, cfg.tol, cfg.mt1, cfg.mt2, cfg.p1, cfg.p2,
                          int(cfg.blind), int(cfg.shuffled), cfg.seed, cfg.objective_every,
                          cfg.tv_lambda_mag, cfg.tv_lambda_phase)
        h = C.c_void_p()
        check(lib().pftg_solver_create(self.code, obj.ctypes.data, obj.shape[0], obj.shape[1],
                                       pr.ctypes.data, pr.shape[0], pr.shape[1],
                                       o.ctypes.data_as(C.POINTER(C.c_int64)), len(o),
                                       dd.ctypes.data, C.byref(c),
                                       table._h if table is not None else None, C.byref(h)))
        self._h = h
        self._table = table

    def run(self, max_sweeps: int = 0):
        check(lib().pftg_solver_run(self._h, max_sweeps))
        return self

    def result(self) -> ReconResult:
        total = self.cfg.pft_sweeps + self.cfg.fft_sweeps
        obj = np.zeros(max(total, 1))
        wall = np.zeros(max(total, 1))
        n, fl = C.c_int(0), C.c_int(0)
        check(lib().pftg_solver_trace(self._h, obj.ctypes.data_as(C.POINTER(C.c_double)),
                                      wall.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n),
                                      C.byref(fl)))
        frame = np.zeros(self.shapes[0], self.cdt)
        probe = np.zeros(self.shapes[1], self.cdt)
        check(lib().pftg_solver_result(self._h, frame.ctypes.data, probe.ctypes.data))
        k = n.value
        return ReconResult(frame, probe, obj[:len(wall)][:k], wall[:k], k, bool(fl.value & 2),
                           bool(fl.value & 1))

    def metrics(self, truth):
        """fill_metrics (solver.cpp:141-160) of the live frame against ``truth``
        (a frame-shaped CUDA tensor of the solver's dtype), on the device, between
        sweeps: the per-sweep metric row of the reference's trace. Returns
        paper_2408_03532_b200.metrics.Metrics."""
        from .metrics import Metrics
        fptr, pptr = C.c_void_p(), C.c_void_p()
        check(lib().pftg_solver_device_state(self._h, C.byref(fptr), C.byref(pptr)))
        want = torch.complex64 if self.code == PFTG_C64 else torch.complex128
        if not isinstance(truth, torch.Tensor) or not truth.is_cuda or truth.dtype != want or \
                tuple(truth.shape) != tuple(self.shapes[0]) or not truth.is_contiguous():
            raise ValueError(f"metrics: truth must be a contiguous {want} CUDA tensor of shape {self.shapes[0]}")
        fr, fc = self.shapes[0]
        out = (C.c_double * 8)()
        check(lib().pftg_fill_metrics_dev(self.code, fptr, fc, _ptr(truth), fc, fr, fc, out, None))
        return Metrics(*[float(v) for v in out])

    def __del__(self):
        try:
            lib().pftg_solver_free(self._h)
        except Exception:
            pass


def hybrid_solve(d, offsets, probe_init, object_init, cfg: SolverConfig,
                 table: ScopeTable | None = None, dtype=np.complex64) -> ReconResult:
    """ptycho::hybrid_solve (solver.hpp:87-90; solver.cpp:173-302), on the GPU."""
    return Solver(d, offsets, probe_init, object_init, cfg, table, dtype).run().result()


def solve_pie(d, offsets, probe, object_init, cfg: SolverConfig, dtype=np.complex64):
    """solve_pie (solver.cpp:304-311): pft_sweeps forced to 0, non-blind."""
    c = dataclasses.replace(cfg, pft_sweeps=0, blind=False)
    return hybrid_solve(d, offsets, probe, object_init, c, None, dtype)


def solve_epie(d, offsets, probe_init, object_init, cfg: SolverConfig, dtype=np.complex64):
    """solve_epie (solver.cpp:313-320): pft_sweeps forced to 0, blind."""
    c = dataclasses.replace(cfg, pft_sweeps=0, blind=True)
    return hybrid_solve(d, offsets, probe_init, object_init, c, None, dtype)
