"""Short evaluator run for ncu (cfg5: cfg4 problem, 1600 positions of 512^2 c64,
PFT M=128 + full FFT). Usage: python tools/prof_eval.py [npos]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2408_03532_b200 as P  # noqa: E402
from paper_2408_03532_b200 import problems as PR  # noqa: E402
from paper_2408_03532_b200.solver import evaluate  # noqa: E402

npos = int(sys.argv[1]) if len(sys.argv) > 1 else 64
prob = PR.make_problem("cfg4", seed=0, npos=npos)
w = prob.probe.shape[0]
plan = P.pft_plan_2d(w, w, 64, 64, 64, 64, 1e-3)
dcrop = P.crop_centered(prob.d.cuda(), 64, 64)
for _ in range(2):
    r = evaluate(prob.obj, prob.probe, prob.offsets, prob.d, (0, npos), plan, dcrop)
torch.cuda.synchronize()
print("ok", r)
