"""Short cfg1 run for ncu launch lists (single 512^2 complex128 field, literal
plan p = 16, q = 32, r = 12): 5 forward + adjoint pairs."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2408_03532_b200 as P  # noqa: E402
from paper_2408_03532_b200.dist import make_fields  # noqa: E402

plan = P.pft_plan_2d(512, 512, 64, 64, 16, 16, 1.0, P.ScopeTable.load(ROOT / "paper_2408_03532_b200/data/scope_table_xi4_r12.txt"))
z = make_fields(1000, 0, 1, 512, 512, torch.complex128, "cuda")
for _ in range(5):
    b = P.pft_apply_2d(plan, z)
    y = P.pft_adjoint_2d(plan, b)
torch.cuda.synchronize()
print("ok")
