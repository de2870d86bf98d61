"""Short PFT run for ncu: cfg2 batched fwd+adj (64 x 1024^2 c64), 1 warm-up
step + 1 profiled step. Usage: python tools/prof_pft.py [workload]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2408_03532_b200 as P  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if wl == "cfg2":
    table, n, mt, p, cdt, batch, eps = "scope_table_xi4_r10.txt", 1024, 128, 32, torch.complex64, 64, 1.0
elif wl == "cfg2c":  # scope-1 companion
    table, n, mt, p, cdt, batch, eps = "scope_table_v1.txt", 1024, 128, 128, torch.complex64, 64, 1e-7
else:
    table, n, mt, p, cdt, batch, eps = "scope_table_xi4_r12.txt", 512, 64, 16, torch.complex128, 1, 1.0
plan = P.pft_plan_2d(n, n, mt, mt, p, p, eps, P.ScopeTable.load(ROOT / "paper_2408_03532_b200/data" / table))
z = torch.randn((batch, n, n), dtype=cdt, device="cuda")
for _ in range(2):
    band = P.pft_apply_2d(plan, z)
    zb = P.pft_adjoint_2d(plan, band)
torch.cuda.synchronize()
print("ok", float(zb.abs().mean()))
