"""Time the forward PFT alone (cfg2: 64 x 1024^2 c64) with CUDA events."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import paper_2408_03532_b200 as P
from paper_2408_03532_b200._lib import KernelProfile
plan = P.pft_plan_2d(1024, 1024, 128, 128, 32, 32, 1.0, P.ScopeTable.load(ROOT / "paper_2408_03532_b200/data/scope_table_xi4_r10.txt"))
z = torch.randn((64, 1024, 1024), dtype=torch.complex64, device="cuda")
for _ in range(3):
    P.pft_apply_2d(plan, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with KernelProfile() as prof:
    e0.record()
    for _ in range(10):
        P.pft_apply_2d(plan, z)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
rows = prof.ms["pft_rows_fwd"] / prof.count["pft_rows_fwd"]
cols = prof.ms["pft_cols_fwd"] / prof.count["pft_cols_fwd"]
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} fwd step {ms*1e3:.1f} us; rows launch {rows*1e3:.1f} us -> {32*8*2**20/rows/1e6:.0f} GB/s (per 32 fields); cols launch {cols*1e3:.1f} us")
