"""Compare the GPU hybrid_solve (c64, c128) with the reference on the cfg3
problem for a few sweeps; prints objectives and relative differences."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_03532_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2408_03532_b200 import problems as PR  # noqa: E402

npos = int(sys.argv[1]) if len(sys.argv) > 1 else 400
pft, fft = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1, 1)
bscale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
beta = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
gamma = float(sys.argv[6]) if len(sys.argv) > 6 else 1.0
prob = PR.make_problem("cfg3", seed=0, npos=npos)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2))
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex128).cpu().numpy()
d = prob.d.cpu().numpy().astype(np.float64)
kw = dict(pft_sweeps=pft, fft_sweeps=fft, beta=beta, gamma=gamma, beta_pft=bscale / w ** 2,
          gamma_pft=bscale * gamma / w ** 2, eps_pft=1e-3, blind=True)
t0 = time.time()
fr, pr, objr, _, flags = ref.hybrid_solve(init, pinit, prob.offsets, d, mt=32, table_path=P.DEFAULT_TABLE, **kw)
print("ref", time.time() - t0, "s, objective", objr, "flags", flags)
for dt in (np.complex128, np.complex64):
    res = P.hybrid_solve(d, prob.offsets, pinit, init, P.SolverConfig(mt1=32, mt2=32, **kw), dtype=dt)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    print(dt.__name__, "objective", res.objective, "frame rel", rel(res.frame, fr), "probe rel",
          rel(res.probe, pr), "diverged", res.diverged)
