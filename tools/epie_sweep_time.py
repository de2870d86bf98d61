"""Steady-state per-sweep wall time of the cfg3 ePIE (graph mode), band and FFT
stages, objective evaluated only on the last sweep."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200 import problems as PR
prob = PR.make_problem("cfg3", seed=0)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex64).cpu().numpy()
cfg = P.SolverConfig(pft_sweeps=4, fft_sweeps=4, beta=0.5, gamma=0.05, beta_pft=0.25 / w**2,
                     gamma_pft=0.0125 / w**2, eps_pft=1e-3, mt1=32, mt2=32, blind=True, objective_every=1000)
s = P.Solver(prob.d.cpu().numpy(), prob.offsets, pinit, init, cfg)
s.run()
r = s.result()
npos = len(prob.offsets)
dt = np.diff(np.concatenate([[0.0], r.wall_s]))
print("per-sweep ms:", np.round(dt * 1e3, 2))
print(f"band us/pos (steady): {1e6 * np.median(dt[1:4]) / npos:.1f}   fft us/pos (steady): {1e6 * np.median(dt[5:7]) / npos:.1f}")
print("objective", r.objective[-1], "err", PR.relative_error_aligned(r.frame, prob.obj.cpu().numpy()))
