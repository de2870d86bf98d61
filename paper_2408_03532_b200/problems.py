"""Seeded synthetic ptychography problems with BASELINE.json's shapes (configs
[2]-[4]); the paper's test images are not available and not needed.

Decisions (stated in DESIGN.md):
  * object: amplitude U[0.5, 1]; phase = periodic Gaussian smoothing (sigma px)
    of U[-pi, pi], rescaled to span [-pi, pi] (unscaled smoothing would leave a
    ~0.06 rad phase);
  * probe: Gaussian amplitude (sigma px) times the reference's quadratic phase
    (pi/6) rho^2 / r_max^2 (simulate.cpp:26-46);
  * scan: K x K raster keeping n, w and the position count; offsets
    round(k (n - w - 2J) / (K - 1)) + J + seeded jitter in [-J, J] (J = 2 px),
    row-major visit order (the BASELINE overlaps cannot fit the frame, §9.2);
  * data: d = |FFT2(probe * patch)| (simulate.cpp:48-65) with Poisson noise at
    a global scale s = photons / mean_j sum_k d_jk^2 (add_poisson_noise,
    simulate.cpp:67-79): d <- sqrt(Poisson(s d^2) / s).
Object and probe are generated with torch on the GPU; the measurements come
from the package's own GPU simulator (paper_2408_03532_b200.simulate, F1) --
input generation, outside every timed region.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch


@dataclasses.dataclass
class Problem:
    obj: torch.Tensor      # truth frame (n x n) complex
    probe: torch.Tensor    # truth probe (w x w) complex
    offsets: np.ndarray    # (N, 2) int64, visit order
    d: torch.Tensor        # (N, w, w) measured magnitudes (real)
    photons: float


CONFIGS = {
    # name: (n, w, K, sigma_phase, sigma_probe, photons, pft_sweeps, fft_sweeps, mt)
    "cfg3": (1024, 256, 20, 8.0, 40.0, 1e6, 10, 20, 32),
    "cfg4": (4096, 512, 40, 16.0, 80.0, 1e7, 15, 15, 64),
}


def smoothed_phase(n, sigma, gen, device):
    u = (torch.rand((n, n), generator=gen, device=device, dtype=torch.float64) * 2 - 1) * math.pi
    f = torch.fft.fftfreq(n, device=device, dtype=torch.float64)
    g = torch.exp(-2 * (math.pi * sigma) ** 2 * (f[:, None] ** 2 + f[None, :] ** 2))
    ph = torch.fft.ifft2(torch.fft.fft2(u) * g).real
    return ph * (math.pi / ph.abs().max())


def make_object(n, sigma, gen, device, dtype=torch.complex64):
    amp = 0.5 + 0.5 * torch.rand((n, n), generator=gen, device=device, dtype=torch.float64)
    ph = smoothed_phase(n, sigma, gen, device)
    return torch.polar(amp, ph).to(dtype)


def make_probe(w, sigma, device, dtype=torch.complex64):
    c = (w - 1) / 2.0
    y, x = torch.meshgrid(torch.arange(w, device=device, dtype=torch.float64) - c,
                          torch.arange(w, device=device, dtype=torch.float64) - c, indexing="ij")
    rho2 = x * x + y * y
    rmax = c + 0.5
    amp = torch.exp(-rho2 / (2 * sigma * sigma))
    ph = (math.pi / 6.0) * rho2 / (rmax * rmax)
    return torch.polar(amp, ph).to(dtype)


def raster_offsets(n, w, K, jitter, seed):
    rng = np.random.default_rng(seed)
    base = [round(k * (n - w - 2 * jitter) / (K - 1)) + jitter for k in range(K)]
    offs = []
    for r in base:
        for c in base:
            jr, jc = rng.integers(-jitter, jitter + 1, size=2)
            offs.append((min(max(r + jr, 0), n - w), min(max(c + jc, 0), n - w)))
    return np.array(offs, np.int64)


def simulate(obj, probe, offsets, photons, seed):
    """Measurements through the package's own GPU simulator (F1): d = |FFT2(probe
    .* window)| in complex128 (simulate.cpp:48-65), then Poisson noise at the
    global photon scale (add_poisson_noise, simulate.cpp:67-79; counter-based
    stream, include/pftg.h)."""
    from .simulate import add_poisson_noise, photon_scale
    from .simulate import simulate as gpu_simulate
    d = gpu_simulate(obj.to(torch.complex128).contiguous(), probe.to(torch.complex128).contiguous(), offsets)
    if photons:
        add_poisson_noise(d, photon_scale(d, photons), seed)
    return d


def make_problem(name, device="cuda", seed=0, dtype=torch.complex64, npos=None) -> Problem:
    n, w, K, sph, spr, photons, *_ = CONFIGS[name]
    gen = torch.Generator(device=device).manual_seed(seed)
    obj = make_object(n, sph, gen, device, dtype)
    probe = make_probe(w, spr, device, dtype)
    offs = raster_offsets(n, w, K, 2, seed)
    if npos is not None:
        offs = offs[:npos]
    d = simulate(obj, probe, offs, photons, 0x5EED + seed)
    return Problem(obj, probe, offs, d.to(torch.float32 if dtype == torch.complex64 else torch.float64), photons)


def relative_error_aligned(x, ref):
    """relative_error_aligned (metrics.cpp:83-96): divide out the best global phase."""
    x = np.asarray(x, np.complex128).ravel()
    ref = np.asarray(ref, np.complex128).ravel()
    c = np.vdot(x, ref)
    ph = c / abs(c) if abs(c) > 0 else 1.0
    return float(np.linalg.norm(x * ph - ref) / np.linalg.norm(ref))
