"""Write-only HBM bandwidth (fill_ / memset of a 5.6 GB buffer), the ceiling for the reconstruction."""
import torch

n = 5624208000 // 4
x = torch.empty(n, dtype=torch.float32, device="cuda")
for name, f in [("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_()),
                ("copy 2.8GB->2.8GB", lambda: x[n // 2:].copy_(x[: n // 2]))]:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = n * 4
    print(f"{name}: {ms:.3f} ms, {nbytes / ms / 1e6:.0f} GB/s (counting {nbytes / 1e9:.2f} GB)")

# the reconstruction's DRAM pattern: 256-B column chunks of 8000-B rows, all rows per pass
y = x.view(-1, 2000)
def chunked(w):
    for c in range(0, 2000, w):
        y[:, c:c + w].fill_(1.0)
for w in (64, 128, 256, 500):
    chunked(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        chunked(w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"column chunks of {w * 4} B: {ms:.3f} ms, {n * 4 / ms / 1e6:.0f} GB/s")
