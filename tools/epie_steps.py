"""Step-size sweep for the blind hybrid ePIE (GPU, complex64): final
objective and phase-aligned relative error vs the truth for each setting.
usage: python tools/epie_steps.py [cfg3|cfg4]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import itertools  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_03532_b200 as P  # noqa: E402
from paper_2408_03532_b200 import problems as PR  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
_n, _w, _K, _sph, spr, _ph, pft_sweeps, fft_sweeps, mt = PR.CONFIGS[name]
prob = PR.make_problem(name, seed=0)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 1.2 * spr, "cuda").abs().to(torch.complex64).cpu().numpy()
d = prob.d.cpu().numpy()
truth = prob.obj.cpu().numpy()
grid = (((1.0, 0.5), (1.0, 0.2, 0.05), (1.0, 0.25)) if name == "cfg3" else
        ((0.5, 0.25, 0.1), (0.05, 0.01, 0.002), (0.25, 0.05)))
for beta, gamma, bp in itertools.product(*grid):
    cfg = P.SolverConfig(pft_sweeps=pft_sweeps, fft_sweeps=fft_sweeps, beta=beta, gamma=gamma,
                         beta_pft=bp / w ** 2, gamma_pft=bp * gamma / w ** 2, eps_pft=1e-3, mt1=mt, mt2=mt,
                         blind=True)
    res = P.hybrid_solve(d, prob.offsets, pinit, init, cfg)
    err = PR.relative_error_aligned(res.frame, truth) if not res.diverged else float("nan")
    print(f"beta={beta} gamma={gamma} bpft*w2={bp}: sweeps={res.sweeps_run} div={res.diverged} "
          f"obj[pft_end]={res.objective[min(pft_sweeps - 1, len(res.objective) - 1)]:.4g} obj_final={res.objective[-1]:.4g} "
          f"err={err:.4f}", flush=True)
