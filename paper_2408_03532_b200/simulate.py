"""Python mirror of the reference's measurement simulator
(/root/reference/proj/core/include/ptycho/simulate.hpp) over libpftg -- the
step before the hot path, on the GPU.

=================  ================================================  ==================
reference          here                                              reference lines
=================  ================================================  ==================
simulate           ``simulate(frame, probe, offsets)``               simulate.cpp:48-65
add_poisson_noise  ``add_poisson_noise(d, scale, seed)`` (in place)  simulate.cpp:67-79
build_cropped      ``build_cropped(d, mt1, mt2)``                    simulate.cpp:81-89
save_measurements  ``save_measurements(dir, d, dcrop, scale, seed)`` simulate.cpp:91-127
load_measurements  ``load_measurements(dir, dtype)``                 simulate.cpp:129-164
=================  ================================================  ==================

The Poisson law is the reference's; the random stream is counter-based
(Philox-4x32-10, include/pftg.h), so a given seed reproduces bit for bit on
any launch shape but does not reproduce libstdc++'s mt19937_64 stream.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import check, lib
from .pft import _dev, _dtype_code, _ptr, _stream, crop_centered


def simulate(frame, probe, offsets):
    """d_j = |FFT2(probe .* frame window j)|, shape (N, wr, wc), real."""
    f, p = _dev(frame), _dev(probe)
    if f.dtype != p.dtype or f.device != p.device:
        raise ValueError("simulate: frame and probe must share dtype and device")
    if f.dim() != 2 or p.dim() != 2:
        raise ValueError("simulate: frame and probe must be 2-D")
    o = np.ascontiguousarray(np.asarray(offsets, np.int64).reshape(-1, 2))
    wr, wc = p.shape
    real = torch.float32 if f.dtype == torch.complex64 else torch.float64
    d = torch.empty((len(o), wr, wc), dtype=real, device=f.device)
    check(lib().pftg_simulate_dev(_dtype_code(f), _ptr(f), f.shape[0], f.shape[1], _ptr(p), wr, wc,
                                  o.ctypes.data_as(C.POINTER(C.c_int64)), len(o), _ptr(d), _stream()))
    return d


def add_poisson_noise(d, scale: float, seed: int):
    """In place: d <- sqrt(Poisson(scale d^2) / scale) (simulate.cpp:67-79)."""
    if not isinstance(d, torch.Tensor) or not d.is_cuda or not d.is_contiguous():
        raise ValueError("add_poisson_noise: d must be a contiguous CUDA tensor")
    if d.dtype not in (torch.float32, torch.float64):
        raise TypeError("add_poisson_noise: real float32/float64 measurements expected")
    code = 0 if d.dtype == torch.float32 else 1
    check(lib().pftg_add_poisson_noise_dev(code, _ptr(d), d.numel(), float(scale), int(seed) & (2**64 - 1),
                                           _stream()))
    return d


def photon_scale(d, photons_per_pattern: float) -> float:
    """Global scale s with mean_j sum_k s d_jk^2 = photons."""
    return float(photons_per_pattern) / float((d.double() ** 2).sum(dim=(-2, -1)).mean())


def build_cropped(d, mt1: int, mt2: int):
    """Centered low-frequency band of every d_j (simulate.cpp:81-89)."""
    if mt1 == 0 or mt2 == 0 or 2 * mt1 > d.shape[-2] or 2 * mt2 > d.shape[-1]:
        raise ValueError("build_cropped: band must satisfy 0 < 2*mt <= window")
    return crop_centered(d, mt1, mt2)


def save_measurements(path, d, dcrop=None, noise_scale: float = 0.0, noise_seed: int = 0):
    """Write the reference's measurement directory (meta.txt, d_NNNN.ptyr,
    dcrop_NNNN.ptyr, FNV-1a manifest) from d [N][wr][wc] (and dcrop
    [N][2mt1][2mt2]); host or device arrays, stored as float64."""
    def host64(a):
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().numpy()
        return np.ascontiguousarray(a, np.float64)
    dd = host64(d)
    if dd.ndim != 3:
        raise ValueError("save_measurements: d must be [count, rows, cols]")
    dc = host64(dcrop) if dcrop is not None else None
    if dc is not None and (dc.ndim != 3 or dc.shape[0] != dd.shape[0] or dc.shape[1] % 2 or dc.shape[2] % 2):
        raise ValueError("save_measurements: dcrop must be [count, 2mt1, 2mt2]")
    dp = C.POINTER(C.c_double)
    mt1, mt2 = (dc.shape[1] // 2, dc.shape[2] // 2) if dc is not None else (0, 0)
    check(lib().pftg_measurements_save(str(path).encode(), dd.shape[0], dd.shape[1], dd.shape[2],
                                       dd.ctypes.data_as(dp), mt1, mt2,
                                       dc.ctypes.data_as(dp) if dc is not None else None,
                                       float(noise_scale), int(noise_seed)))


def load_measurements(path, dtype=np.float32, device=None):
    """Read a measurement directory (manifest verified, like the reference):
    returns (d, dcrop or None, noise_scale, noise_seed) as numpy arrays in
    ``dtype`` (float32 for the complex64 path, float64 for complex128), or
    CUDA tensors when ``device`` is given."""
    info = np.zeros(5, np.int64)
    scale, seed = C.c_double(), C.c_uint64()
    check(lib().pftg_measurements_info(str(path).encode(), info.ctypes.data_as(C.POINTER(C.c_int64)),
                                       C.byref(scale), C.byref(seed)))
    cnt, r, c, m1, m2 = (int(v) for v in info)
    dt = np.dtype(dtype)
    if dt not in (np.float32, np.float64):
        raise TypeError("load_measurements: dtype must be float32 or float64")
    d = np.empty((cnt, r, c), dt)
    dc = np.empty((cnt, 2 * m1, 2 * m2), dt) if m1 else None
    code = 0 if dt == np.float32 else 1
    check(lib().pftg_measurements_read(str(path).encode(), code, d.ctypes.data,
                                       dc.ctypes.data if dc is not None else None))
    if device is not None:
        d = torch.from_numpy(d).to(device)
        dc = torch.from_numpy(dc).to(device) if dc is not None else None
    return d, dc, scale.value, seed.value
