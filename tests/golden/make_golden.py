"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py
Every array here is produced by the unmodified reference proj/core sources
(pft.cpp, fft.cpp, minimax.cpp, solver.cpp, scan.cpp, simulate.cpp) compiled
into oracle/_ref/libptycho_ref.so; only Eigen/FFTW are replaced by the shims in
oracle/shim (their published semantics: dense GEMM, unnormalized DFT, LU with
complete pivoting). Inputs are seeded numpy draws, stored alongside.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
DATA = ROOT / "paper_2408_03532_b200" / "data"


def cn(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def main():
    # 1. small PFT (n=64, m~=p=8, eps=1e-7 -> r=13): forward + adjoint
    rng = np.random.default_rng(100)
    rp = ref.RefPlan.create(DATA / "scope_table_v1.txt", 64, 64, 8, 8, 8, 8, 1e-7)
    z = cn(rng, (64, 64))
    y = cn(rng, (16, 16))
    B1, W1 = rp.tables(1)
    np.savez_compressed(OUT / "pft_small.npz", z=z, band=rp.apply(z), y=y, adj=rp.adjoint(y),
                        B=B1, W=W1, r=rp.r1)

    # 2. rectangular PFT with M < p on axis 1 (n1=128, mt1=4, p1=16; n2=64, mt2=8, p2=8)
    rng = np.random.default_rng(101)
    rp = ref.RefPlan.create(DATA / "scope_table_v1.txt", 128, 64, 4, 8, 16, 8, 1e-3)
    z = cn(rng, (128, 64))
    y = cn(rng, (8, 16))
    np.savez_compressed(OUT / "pft_rect.npz", z=z, band=rp.apply(z), y=y, adj=rp.adjoint(y),
                        r1=rp.r1, r2=rp.r2)

    # 3. BASELINE cfg1 literal plan (512^2, p=16, q=32, r=12, m~=64): band + sampled adjoint
    rng = np.random.default_rng(102)
    rp = ref.RefPlan.create(DATA / "scope_table_xi4_r12.txt", 512, 512, 64, 64, 16, 16, 1.0)
    z = cn(rng, (512, 512))
    band = rp.apply(z)
    adj = rp.adjoint(band)
    np.savez_compressed(OUT / "pft_cfg1_literal.npz", seed=102, band=band,
                        adj_sample=adj[::7, ::13], adj_norm=np.linalg.norm(adj))

    # 4. project_modulus / band_residual / objective on a tiny scan (64^2 window)
    rng = np.random.default_rng(103)
    n, w = 96, 64
    obj = (0.5 + 0.5 * rng.random((n, n))) * np.exp(1j * rng.uniform(-1, 1, (n, n)))
    yy, xx = np.mgrid[0:w, 0:w] - (w - 1) / 2
    probe = np.exp(-(xx ** 2 + yy ** 2) / (2 * 12.0 ** 2)) * np.exp(1j * 0.2 * (xx ** 2 + yy ** 2) / w ** 2)
    offs = np.array([[r, c] for r in (0, 16, 32) for c in (0, 16, 32)], np.int64)
    d = ref.simulate(obj, probe, offs)
    x = probe * obj[16:16 + w, 16:16 + w]
    dn = d[4] * 0.9
    pm = ref.project_modulus(x, dn)
    rpb = ref.RefPlan.create(DATA / "scope_table_v1.txt", w, w, 8, 8, 8, 8, 1e-3)
    dcrop = ref.crop_centered(dn, 8, 8)
    br = rpb.band_residual(x, dcrop)
    init = np.exp(1j * 0.1 * rng.standard_normal((n, n))) * 0.8
    phi0 = ref.objective_value(init, probe, offs, d)
    kw = dict(pft_sweeps=2, fft_sweeps=2, beta=1.0, gamma=1.0, beta_pft=1.0 / w ** 2,
              gamma_pft=1.0 / w ** 2, eps_pft=1e-3, blind=True)
    f, pr, objv, _, flags = ref.hybrid_solve(init, probe * 0.9, offs, d,
                                             table_path=DATA / "scope_table_v1.txt", **kw)
    np.savez_compressed(OUT / "solver_tiny.npz", obj=obj, probe=probe, offs=offs, d=d, x=x, dn=dn,
                        project_modulus=pm, dcrop=dcrop, band_residual=br, init=init, phi0=phi0,
                        hybrid_frame=f, hybrid_probe=pr, hybrid_objective=objv,
                        hybrid_cfg=np.array([2, 2, 1.0, 1.0, 1.0 / w ** 2, 1.0 / w ** 2, 1e-3, 1.0]))

    # 5. minimax: best_approx known answers and min_degree (SPEC ACC-3)
    recs = {}
    for r, xi in ((13, 1.0), (9, 1.0), (12, 4.0), (10, 4.0), (3, 0.1)):
        c, ach, conv = ref.best_approx(r, xi)
        recs[f"r{r}_xi{xi}"] = np.concatenate([[ach, float(conv)], c.real, c.imag])
    md = np.array([ref.min_degree(DATA / "scope_table_v1.txt", e, t)
                   for e, t in ((1e-7, 1.0), (1e-3, 1.0), (1e-1, 4.0), (1e-3, 4.0), (1e-5, 4.0))])
    np.savez_compressed(OUT / "minimax.npz", min_degree=md, **recs)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
