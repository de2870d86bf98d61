"""Python mirror of the reference's ``ptycho::pft`` / ``ptycho`` transform API
over libpftg (include/pftg.h).

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/ptycho/{pft,fft,minimax}.hpp:

=========================  ====================================================
reference                  here
=========================  ====================================================
minimax::ScopeTable::load  ``ScopeTable.load(path)``            (minimax.hpp:50)
ScopeTable::min_degree     ``ScopeTable.min_degree(eps, xi)``   (minimax.hpp:59)
pft::pft_plan_2d           ``pft_plan_2d(n1, n2, mt1, mt2, p1, p2, eps, table)`` (pft.hpp:49)
pft::load_plan_2d/save     ``PftPlan2D.load(path)`` / ``plan.save(path)`` (pft.hpp:60-63)
pft::pft_apply_2d          ``pft_apply_2d(plan, z)``            (pft.hpp:53)
pft::pft_adjoint_2d        ``pft_adjoint_2d(plan, band)``       (pft.hpp:57)
pft::pft_plan_1d           ``pft_plan_1d(n, mt, p, eps, table)`` (pft.hpp:33)
pft::pft_apply_1d          ``pft_apply_1d(plan, z)``            (pft.hpp:38)
pft::load_plan_1d/save     ``PftPlan1D.load(path)`` / ``plan.save(path)`` (pft.hpp:60-62)
fast_fft2 / fast_ifft2     ``fast_fft2(z)`` / ``fast_ifft2(z)`` (fft.hpp:18-19)
crop_centered              ``crop_centered(d, mt1, mt2)``       (fft.hpp:30)
=========================  ====================================================

Arrays are ``torch`` tensors on a CUDA device (complex64 or complex128; the
dtype selects the kernel precision) with optional leading batch dimensions;
``pft_apply_2d`` / ``pft_adjoint_2d`` additionally accept host numpy arrays
(routed through the pipelined host-buffer C-ABI entry points). Shape errors
raise ValueError, like the reference's std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._lib import PFTG_C64, PFTG_C128, check, lib

DATA = Path(__file__).resolve().parent / "data"
DEFAULT_TABLE = DATA / "scope_table_v1.txt"


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(t) -> int:
    if t.dtype in (torch.complex64, np.complex64):
        return PFTG_C64
    if t.dtype in (torch.complex128, np.complex128):
        return PFTG_C128
    raise TypeError(f"expected complex64 or complex128, got {t.dtype}")


def _real_of(t: torch.Tensor) -> torch.dtype:
    return torch.float32 if t.dtype == torch.complex64 else torch.float64


def _dev(t):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA torch tensor")
    return t.contiguous()


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


class ScopeTable:
    """minimax::ScopeTable loaded from the ``pft-scope-table v1`` text format."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    @classmethod
    def load(cls, path=DEFAULT_TABLE) -> "ScopeTable":
        h = C.c_void_p()
        check(lib().pftg_table_load(str(path).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def compute(cls, eps_list=(1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7), max_r: int = 25) -> "ScopeTable":
        """ScopeTable::compute (minimax.hpp:48-49): the own near-minimax solver
        (csrc/minimax.cpp) over eps x r = 1..max_r."""
        e = np.ascontiguousarray(eps_list, np.float64)
        h = C.c_void_p()
        check(lib().pftg_table_compute(e.ctypes.data_as(C.POINTER(C.c_double)), len(e), max_r, C.byref(h)))
        return cls(h.value)

    def save(self, path) -> None:
        """ScopeTable::save: the pft-scope-table v1 text format."""
        check(lib().pftg_table_save(self._h, str(path).encode()))

    def records(self):
        """[(eps, r, xi, achieved_error, coeff complex128[r]), ...], eps-major, r ascending."""
        n, mr = C.c_int(), C.c_int()
        check(lib().pftg_table_info(self._h, C.byref(n), C.byref(mr)))
        out = []
        for i in range(n.value):
            eps, xi, ach, r = C.c_double(), C.c_double(), C.c_double(), C.c_int()
            check(lib().pftg_table_record(self._h, i, C.byref(eps), C.byref(r), C.byref(xi), C.byref(ach), None))
            w = np.zeros(r.value, np.complex128)
            check(lib().pftg_table_record(self._h, i, None, None, None, None,
                                          w.ctypes.data_as(C.POINTER(C.c_double))))
            out.append((eps.value, r.value, xi.value, ach.value, w))
        return out

    def min_degree(self, eps: float, target_scope: float) -> int:
        r = C.c_int()
        check(lib().pftg_table_min_degree(self._h, eps, target_scope, C.byref(r)))
        return r.value

    def __del__(self):
        try:
            lib().pftg_table_free(self._h)
        except Exception:
            pass


class PftPlan2D:
    """pft::PftPlan2D: immutable plan; device tables are uploaded on first use."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        info = np.zeros(10, np.int64)
        check(lib().pftg_plan_info(self._h, info.ctypes.data_as(C.POINTER(C.c_int64))))
        (self.n1, self.p1, self.q1, self.mt1, self.r1,
         self.n2, self.p2, self.q2, self.mt2, self.r2) = (int(v) for v in info)

    @property
    def band_shape(self):
        return (2 * self.mt1, 2 * self.mt2)

    @property
    def field_shape(self):
        return (self.n1, self.n2)

    @classmethod
    def load(cls, path) -> "PftPlan2D":
        h = C.c_void_p()
        check(lib().pftg_plan_load(str(path).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_tables(cls, n1, p1, mt1, B1, W1, n2, p2, mt2, B2, W2, eps=0.0) -> "PftPlan2D":
        """Plan from in-memory PftPlan1D tables (B: q x r, W: (2mt+1) x r, complex128)."""
        def arr(a):
            return np.ascontiguousarray(a, np.complex128)
        B1, W1, B2, W2 = arr(B1), arr(W1), arr(B2), arr(W2)
        r1, r2 = B1.shape[1], B2.shape[1]
        if B1.shape != (n1 // p1, r1) or W1.shape != (2 * mt1 + 1, r1) or \
                B2.shape != (n2 // p2, r2) or W2.shape != (2 * mt2 + 1, r2):
            raise ValueError("pftg_plan_from_tables: table shapes do not match the plan")
        dp = C.POINTER(C.c_double)
        h = C.c_void_p()
        check(lib().pftg_plan_from_tables(n1, p1, mt1, r1, B1.ctypes.data_as(dp), W1.ctypes.data_as(dp),
                                          n2, p2, mt2, r2, B2.ctypes.data_as(dp), W2.ctypes.data_as(dp),
                                          eps, C.byref(h)))
        return cls(h.value)

    def save(self, path) -> None:
        check(lib().pftg_plan_save(self._h, str(path).encode()))

    def tables(self, axis: int):
        """(B, W) of one axis as complex128 numpy arrays (pft.hpp:29-30)."""
        q, r, mt = (self.q1, self.r1, self.mt1) if axis == 1 else (self.q2, self.r2, self.mt2)
        B = np.zeros((q, r), np.complex128)
        W = np.zeros((2 * mt + 1, r), np.complex128)
        check(lib().pftg_plan_tables(self._h, axis, B.ctypes.data_as(C.POINTER(C.c_double)),
                                     W.ctypes.data_as(C.POINTER(C.c_double))))
        return B, W

    def __del__(self):
        try:
            lib().pftg_plan_free(self._h)
        except Exception:
            pass


class PftPlan1D:
    """pft::PftPlan1D (pft.hpp:25-31): immutable 1-D plan."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        info = np.zeros(5, np.int64)
        check(lib().pftg_plan1d_info(self._h, info.ctypes.data_as(C.POINTER(C.c_int64))))
        self.n, self.p, self.q, self.mt, self.r = (int(v) for v in info)

    @property
    def band_len(self):
        return 2 * self.mt + 1

    @classmethod
    def load(cls, path) -> "PftPlan1D":
        h = C.c_void_p()
        check(lib().pftg_plan1d_load(str(path).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_tables(cls, n, p, mt, B, W, eps=0.0) -> "PftPlan1D":
        B = np.ascontiguousarray(B, np.complex128)
        W = np.ascontiguousarray(W, np.complex128)
        r = B.shape[1]
        if B.shape != (n // p, r) or W.shape != (2 * mt + 1, r):
            raise ValueError("pftg_plan1d_from_tables: table shapes do not match the plan")
        dp = C.POINTER(C.c_double)
        h = C.c_void_p()
        check(lib().pftg_plan1d_from_tables(n, p, mt, r, B.ctypes.data_as(dp), W.ctypes.data_as(dp), eps,
                                            C.byref(h)))
        return cls(h.value)

    def save(self, path) -> None:
        check(lib().pftg_plan1d_save(self._h, str(path).encode()))

    def tables(self):
        B = np.zeros((self.q, self.r), np.complex128)
        W = np.zeros((2 * self.mt + 1, self.r), np.complex128)
        check(lib().pftg_plan1d_tables(self._h, B.ctypes.data_as(C.POINTER(C.c_double)),
                                       W.ctypes.data_as(C.POINTER(C.c_double))))
        return B, W

    def __del__(self):
        try:
            lib().pftg_plan1d_free(self._h)
        except Exception:
            pass


def best_approx(r: int, xi: float):
    """minimax::best_approx (minimax.hpp:28): (coeff complex128[r], achieved_error)."""
    w = np.zeros(r, np.complex128)
    e = C.c_double()
    check(lib().pftg_best_approx(r, xi, w.ctypes.data_as(C.POINTER(C.c_double)), C.byref(e)))
    return w, e.value


def pft_plan_1d(n, mt, p, eps, table: ScopeTable | None = None) -> PftPlan1D:
    """pft::pft_plan_1d (pft.hpp:33-34; pft.cpp:33-76)."""
    table = table or ScopeTable.load()
    h = C.c_void_p()
    check(lib().pftg_plan_1d(table._h, n, mt, p, eps, C.byref(h)))
    return PftPlan1D(h.value)


def pft_apply_1d(plan: PftPlan1D, z):
    """pft::pft_apply_1d: the 2mt+1 centered band entries of the DFT of each
    n-vector (last axis), DC at index mt (pft.hpp:36-38)."""
    if isinstance(z, np.ndarray):
        if z.shape[-1] != plan.n:
            raise ValueError("pft_apply_1d: z must be an n-vector matching the plan")
        z = np.ascontiguousarray(z)
        b = int(np.prod(z.shape[:-1], dtype=np.int64))
        out = np.empty(z.shape[:-1] + (plan.band_len,), z.dtype)
        check(lib().pftg_apply_1d_host(plan._h, _dtype_code(z), z.ctypes.data, out.ctypes.data, b))
        return out
    z = _dev(z)
    if z.shape[-1] != plan.n:
        raise ValueError("pft_apply_1d: z must be an n-vector matching the plan")
    b = 1
    for s_ in z.shape[:-1]:
        b *= int(s_)
    out = torch.empty(z.shape[:-1] + (plan.band_len,), dtype=z.dtype, device=z.device)
    check(lib().pftg_apply_1d_dev(plan._h, _dtype_code(z), _ptr(z), _ptr(out), b, _stream()))
    return out


def pft_fwd_adj_2d(plan: "PftPlan2D", z, devices=None):
    """BASELINE configs[1] in one call: (band, back) = (pft_apply_2d(z),
    pft_adjoint_2d(band)). Host numpy input: one streamed C-ABI call
    (pftg_fwd_adj_2d_host, H2D and D2H overlapped); CUDA tensors: the two
    device calls. Bit-identical to calling the two operators in turn.
    devices (host input only): list of CUDA device indices; the batch is split in
    contiguous blocks over them inside the library (pftg_fwd_adj_2d_host_multi,
    one host thread per device, no collective)."""
    if isinstance(z, np.ndarray):
        if tuple(z.shape[-2:]) != plan.field_shape:
            raise ValueError("pft_apply_2d: z shape must match the plan")
        z = np.ascontiguousarray(z)
        b = _batch(z, plan.field_shape)
        band = np.empty(z.shape[:-2] + plan.band_shape, z.dtype)
        back = np.empty(z.shape, z.dtype)
        if devices is not None:
            dv = (C.c_int * len(devices))(*[int(d) for d in devices])
            check(lib().pftg_fwd_adj_2d_host_multi(plan._h, _dtype_code(z), z.ctypes.data, band.ctypes.data,
                                                   back.ctypes.data, b, dv, len(devices)))
            return band, back
        check(lib().pftg_fwd_adj_2d_host(plan._h, _dtype_code(z), z.ctypes.data, band.ctypes.data,
                                         back.ctypes.data, b))
        return band, back
    band = pft_apply_2d(plan, z)
    return band, pft_adjoint_2d(plan, band)


def pft_plan_2d(n1, n2, mt1, mt2, p1, p2, eps, table: ScopeTable | None = None) -> PftPlan2D:
    """pft::pft_plan_2d (pft.hpp:49-51; pft.cpp:33-76,103-112)."""
    table = table or ScopeTable.load()
    h = C.c_void_p()
    check(lib().pftg_plan_2d(table._h, n1, n2, mt1, mt2, p1, p2, eps, C.byref(h)))
    return PftPlan2D(h.value)


def _batch(x, tail):
    if tuple(x.shape[-2:]) != tuple(tail):
        raise ValueError(f"shape must end in {tuple(tail)}, got {tuple(x.shape)}")
    b = 1
    for s in x.shape[:-2]:
        b *= int(s)
    return b


def pft_apply_2d(plan: PftPlan2D, z):
    """pft::pft_apply_2d: band of the 2-D DFT, DC at (mt1, mt2) (pft.hpp:53)."""
    if isinstance(z, np.ndarray):
        if tuple(z.shape[-2:]) != plan.field_shape:
            raise ValueError("pft_apply_2d: z shape must match the plan")
        z = np.ascontiguousarray(z)
        b = _batch(z, plan.field_shape)
        out = np.empty(z.shape[:-2] + plan.band_shape, z.dtype)
        check(lib().pftg_apply_2d_host(plan._h, _dtype_code(z), z.ctypes.data, out.ctypes.data, b))
        return out
    z = _dev(z)
    if tuple(z.shape[-2:]) != plan.field_shape:
        raise ValueError("pft_apply_2d: z shape must match the plan")
    b = _batch(z, plan.field_shape)
    out = torch.empty(z.shape[:-2] + plan.band_shape, dtype=z.dtype, device=z.device)
    check(lib().pftg_apply_2d_dev(plan._h, _dtype_code(z), _ptr(z), _ptr(out), b, _stream()))
    return out


def pft_adjoint_2d(plan: PftPlan2D, band):
    """pft::pft_adjoint_2d: exact adjoint of pft_apply_2d (pft.hpp:57)."""
    if isinstance(band, np.ndarray):
        if tuple(band.shape[-2:]) != plan.band_shape:
            raise ValueError("pft_adjoint_2d: band shape must match the plan")
        band = np.ascontiguousarray(band)
        b = _batch(band, plan.band_shape)
        out = np.empty(band.shape[:-2] + plan.field_shape, band.dtype)
        check(lib().pftg_adjoint_2d_host(plan._h, _dtype_code(band), band.ctypes.data,
                                         out.ctypes.data, b))
        return out
    band = _dev(band)
    if tuple(band.shape[-2:]) != plan.band_shape:
        raise ValueError("pft_adjoint_2d: band shape must match the plan")
    b = _batch(band, plan.band_shape)
    out = torch.empty(band.shape[:-2] + plan.field_shape, dtype=band.dtype, device=band.device)
    check(lib().pftg_adjoint_2d_dev(plan._h, _dtype_code(band), _ptr(band), _ptr(out), b,
                                    _stream()))
    return out


def band_residual(plan: PftPlan2D, exit_wave, d_crop):
    """ptycho::band_residual (solver.hpp:63): A*(A x - d .* exp(i arg(A x)))."""
    x = _dev(exit_wave)
    if tuple(x.shape[-2:]) != plan.field_shape:
        raise ValueError("pft_apply_2d: z shape must match the plan")
    d = _dev(d_crop).to(_real_of(x))
    if tuple(d.shape[-2:]) != plan.band_shape or d.numel() // (4 * plan.mt1 * plan.mt2) != \
            _batch(x, plan.field_shape):
        raise ValueError("band_residual: cropped measurement shape mismatch")
    out = torch.empty_like(x)
    check(lib().pftg_band_residual_dev(plan._h, _dtype_code(x), _ptr(x), _ptr(d), _ptr(out),
                                       _batch(x, plan.field_shape), _stream()))
    return out


def _fft2(z, inverse):
    z = _dev(z)
    if z.dim() < 2 or z.numel() == 0:
        raise ValueError("fast_fft2: empty field")
    rows, cols = z.shape[-2:]
    out = torch.empty_like(z)
    check(lib().pftg_fft2_dev(_dtype_code(z), _ptr(z), _ptr(out), rows, cols,
                              _batch(z, (rows, cols)), int(inverse), _stream()))
    return out


def fast_fft2(z):
    """fast_fft2 (fft.hpp:18): unnormalized forward 2-D DFT."""
    return _fft2(z, False)


def fast_ifft2(z):
    """fast_ifft2 (fft.hpp:19): inverse 2-D DFT with the 1/n factor."""
    return _fft2(z, True)


def crop_centered(spectrum, mt1, mt2):
    """crop_centered(RealField) (fft.hpp:30; fft.cpp:206-232)."""
    s = _dev(spectrum)
    rows, cols = s.shape[-2:]
    out = torch.empty(s.shape[:-2] + (2 * mt1, 2 * mt2), dtype=s.dtype, device=s.device)
    code = PFTG_C64 if s.dtype == torch.float32 else PFTG_C128
    if s.dtype not in (torch.float32, torch.float64):
        raise TypeError("crop_centered: real float32/float64 spectrum expected")
    check(lib().pftg_crop_centered_dev(code, _ptr(s), _ptr(out), rows, cols, mt1, mt2,
                                       _batch(s, (rows, cols)), _stream()))
    return out
