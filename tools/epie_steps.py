"""Step-size sweep for the cfg3 blind hybrid ePIE (GPU, complex64): final
objective and phase-aligned relative error vs the truth for each setting."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import itertools  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_03532_b200 as P  # noqa: E402
from paper_2408_03532_b200 import problems as PR  # noqa: E402

prob = PR.make_problem("cfg3", seed=0)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex64).cpu().numpy()
d = prob.d.cpu().numpy()
truth = prob.obj.cpu().numpy()
for beta, gamma, bp in itertools.product((1.0, 0.5), (1.0, 0.2, 0.05), (1.0, 0.25)):
    cfg = P.SolverConfig(pft_sweeps=10, fft_sweeps=20, beta=beta, gamma=gamma, beta_pft=bp / w ** 2,
                         gamma_pft=bp * gamma / w ** 2, eps_pft=1e-3, mt1=32, mt2=32, blind=True)
    res = P.hybrid_solve(d, prob.offsets, pinit, init, cfg)
    err = PR.relative_error_aligned(res.frame, truth) if not res.diverged else float("nan")
    print(f"beta={beta} gamma={gamma} bpft*w2={bp}: sweeps={res.sweeps_run} div={res.diverged} "
          f"obj[pft_end]={res.objective[min(9, len(res.objective) - 1)]:.4g} obj_final={res.objective[-1]:.4g} "
          f"err={err:.4f}", flush=True)
