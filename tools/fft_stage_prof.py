"""One full-FFT ePIE sweep over a few cfg3 positions (for ncu on the fused
sweep kernel). usage: python tools/fft_stage_prof.py [npos]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200 import problems as PR
npos = int(sys.argv[1]) if len(sys.argv) > 1 else 40
prob = PR.make_problem("cfg3", seed=0, npos=npos)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex64).cpu().numpy()
cfg = P.SolverConfig(pft_sweeps=0, fft_sweeps=1, beta=0.5, gamma=0.05, blind=True)
r = P.hybrid_solve(prob.d.cpu().numpy(), prob.offsets, pinit, init, cfg)
print("ok", r.objective, r.wall_s)
