"""Pinned host -> device copy bandwidth for c2's A (268.5 MB), the floor of the host-buffer e2e."""
import time
import torch
n = 8192 * 4096
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D {n * 8 / 1e6:.1f} MB: {ms:.3f} ms = {n * 8 / ms / 1e6:.1f} GB/s")
