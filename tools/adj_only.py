"""Time the adjoint PFT alone (cfg2: 64 fields, 256^2 band -> 1024^2, c64)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200._lib import KernelProfile
plan = P.pft_plan_2d(1024, 1024, 128, 128, 32, 32, 1.0, P.ScopeTable.load(ROOT / "paper_2408_03532_b200/data/scope_table_xi4_r10.txt"))
y = torch.randn((64, 256, 256), dtype=torch.complex64, device="cuda")
for _ in range(3):
    P.pft_adjoint_2d(plan, y)
torch.cuda.synchronize()
with KernelProfile() as prof:
    for _ in range(10):
        P.pft_adjoint_2d(plan, y)
    torch.cuda.synchronize()
rows = prof.ms["pft_rows_adj"] / prof.count["pft_rows_adj"]
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} rows_adj launch {rows*1e3:.1f} us -> {32*8*2**20/rows/1e6:.0f} GB/s; cols_adj {prof.ms['pft_cols_adj']/prof.count['pft_cols_adj']*1e3:.1f} us")
