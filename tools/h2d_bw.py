"""Pinned host -> device copy bandwidth (the e2e path's PCIe bound), one and two streams."""
import torch
n = 256 * 256 * 256  # one step's images at R: 67 MB
src = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
dst = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("H2D pinned, 67.1 MB: %.3f ms  %.1f GB/s" % (ms, n * 4 / ms / 1e6))
back = torch.empty(n, dtype=torch.float32, pin_memory=True)
e0.record()
for _ in range(20):
    back.copy_(dst, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("D2H pinned, 67.1 MB: %.3f ms  %.1f GB/s" % (ms, n * 4 / ms / 1e6))
