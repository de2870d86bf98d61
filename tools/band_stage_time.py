"""Per-kernel CUDA-event times of one band sweep + one FFT sweep of the cfg3
ePIE (shuffled order -> no graph, so launches are timed individually)."""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200 import problems as PR
from paper_2408_03532_b200._lib import KernelProfile
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
prob = PR.make_problem(name, seed=0)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)).astype(np.complex64)
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex64).cpu().numpy()
for shuffled in (True, False):
    cfg = P.SolverConfig(pft_sweeps=1, fft_sweeps=1, beta=0.5, gamma=0.05, beta_pft=0.25 / w**2,
                         gamma_pft=0.0125 / w**2, eps_pft=1e-3, mt1=w // 8, mt2=w // 8, blind=True, shuffled=shuffled)
    s = P.Solver(prob.d.cpu().numpy(), prob.offsets, pinit, init, cfg)
    with KernelProfile() as prof:
        torch.cuda.synchronize(); t0 = time.perf_counter(); s.run(1); torch.cuda.synchronize(); t1 = time.perf_counter()
        s.run(); torch.cuda.synchronize(); t2 = time.perf_counter()
    npos = len(prob.offsets)
    print(f"shuffled={shuffled} band sweep {1e3*(t1-t0):.1f} ms ({1e6*(t1-t0)/npos:.1f} us/pos), fft sweep {1e3*(t2-t1):.1f} ms ({1e6*(t2-t1)/npos:.1f} us/pos)")
    print({k: (round(v * 1e3 / max(prof.count[k], 1), 2), prof.count[k]) for k, v in prof.ms.items() if prof.count[k]})
