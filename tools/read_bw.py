"""Reference read/copy bandwidth on this GPU (torch kernels), for context."""
import torch
x = torch.randn(64 * 1024 * 1024 * 2, device="cuda")  # 512 MiB
y = torch.empty_like(x)
for _ in range(3):
    x.sum(); y.copy_(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    s = x.sum()
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f"read (sum) {x.numel()*4/t/1e6:.0f} GB/s")
e0.record()
for _ in range(10):
    y.copy_(x)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f"copy r+w {2*x.numel()*4/t/1e6:.0f} GB/s")
