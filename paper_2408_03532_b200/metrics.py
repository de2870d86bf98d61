"""Python mirror of the reference's reconstruction metrics
(/root/reference/proj/core/include/ptycho/metrics.hpp) over libpftg -- the
step after the hot path, on the GPU.

``fill_metrics(x, truth)`` computes the per-sweep metrics row of
hybrid_solve's trace (solver.cpp:141-160) in one device pass:
relative_error, relative_error_aligned, relative_error of magnitude and phase,
ssim and psnr of magnitude and phase, with the truth's dynamic_range
(metrics.cpp:60-143). ``relative_error_aligned`` / ``relative_error`` return
single entries of it.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import torch

from ._lib import check, lib
from .pft import _dtype_code, _ptr, _stream

FIELDS = ("rel_err", "rel_err_aligned", "rel_err_mag", "rel_err_phase", "ssim_mag", "ssim_phase",
          "psnr_mag", "psnr_phase")


@dataclasses.dataclass
class Metrics:
    rel_err: float
    rel_err_aligned: float
    rel_err_mag: float
    rel_err_phase: float
    ssim_mag: float
    ssim_phase: float
    psnr_mag: float
    psnr_phase: float


def _region(t):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dim() != 2:
        raise TypeError("metrics: expected a 2-D CUDA tensor")
    if t.stride(1) != 1:
        raise ValueError("metrics: rows must be contiguous (unit column stride)")
    return t.stride(0)


def fill_metrics(x, truth) -> Metrics:
    """Metrics of reconstruction x against the truth (same shape; views into a
    larger frame are fine: row strides are honoured)."""
    if x.shape != truth.shape:
        raise ValueError("relative_error: shape mismatch")
    if x.dtype != truth.dtype or x.device != truth.device:
        raise ValueError("metrics: x and truth must share dtype and device")
    ldx, ldr = _region(x), _region(truth)
    out = (C.c_double * 8)()
    check(lib().pftg_fill_metrics_dev(_dtype_code(x), _ptr(x), ldx, _ptr(truth), ldr, x.shape[0], x.shape[1],
                                      out, _stream()))
    return Metrics(*[float(v) for v in out])


def relative_error_aligned(x, truth) -> float:
    """relative_error_aligned (metrics.cpp:83-96)."""
    return fill_metrics(x, truth).rel_err_aligned


def relative_error(x, truth) -> float:
    """relative_error (metrics.cpp:60-70), complex fields."""
    return fill_metrics(x, truth).rel_err
