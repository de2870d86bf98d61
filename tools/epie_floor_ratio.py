"""cfg3 problem, 1 band + 1 FFT sweep (tests/test_ops_gpu.py::test_cfg3_full_problem_one_band_one_fft_sweep):
deviation of the complex64 GPU solve from the double reference over the oracle<float> floor."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200 import problems as PR
from oracle import ref
import test_ops_gpu as T
prob = PR.make_problem("cfg3", seed=0)
n, w = prob.obj.shape[0], prob.probe.shape[0]
rng = np.random.default_rng(1)
init = rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)
pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex128).cpu().numpy()
d = prob.d.cpu().numpy().astype(np.float64)
kw = dict(pft_sweeps=1, fft_sweeps=1, beta=0.5, gamma=0.05, beta_pft=0.25 / w ** 2, gamma_pft=0.25 * 0.05 / w ** 2, eps_pft=1e-3, blind=True)
cache = Path("/tmp/epie_floor_ref.npz")
if cache.exists():
    z = np.load(cache); fr, pr, ff, fp = z["fr"], z["pr"], float(z["ff"]), float(z["fp"])
else:
    fr, pr, objr, _, flags = ref.hybrid_solve(init, pinit, prob.offsets, d, mt=32, table_path=T.DATA / "scope_table_v1.txt", **kw)
    ff, fp = T._epie_float_floor(init, pinit, prob.offsets, d, fr, pr, mt=32, **kw)
    np.savez(cache, fr=fr, pr=pr, ff=ff, fp=fp)
r64 = P.hybrid_solve(d, prob.offsets, pinit, init, P.SolverConfig(mt1=32, mt2=32, **kw))
ef, ep = T.rel_l2(r64.frame, fr), T.rel_l2(r64.probe, pr)
print(sys.argv[1:], "frame %.3e (%.2f x floor %.3e)  probe %.3e (%.2f x floor %.3e)" % (ef, ef / ff, ff, ep, ep / fp, fp))
