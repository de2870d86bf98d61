"""Short band-stage ePIE run for the ncu launch list: cfgN problem, first npos
positions, 1 band sweep + 1 FFT sweep. usage: python tools/prof_band.py [cfg3|cfg4] [npos]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2408_03532_b200 as P  # noqa: E402
from paper_2408_03532_b200 import problems as PR  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
npos = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n, w, K, sph, spr, ph, pft, fft, mt = PR.CONFIGS[name]
prob = PR.make_problem(name, seed=0, npos=npos)
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 1.2 * spr, "cuda").abs().to(torch.complex64).cpu().numpy()
cfg = P.SolverConfig(pft_sweeps=1, fft_sweeps=1, beta=0.5, gamma=0.01, beta_pft=0.25 / w ** 2,
                     gamma_pft=0.0025 / w ** 2, eps_pft=1e-3, mt1=mt, mt2=mt, blind=True)
res = P.hybrid_solve(prob.d.cpu().numpy(), prob.offsets, pinit, init, cfg)
print("ok", res.objective)
