"""H2D bandwidth on the box: copy-engine pinned copy of a 400 MB batch."""
import time, torch
n = 100_000_000
h = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("H2D copy engine: %.2f ms per 400 MB = %.1f GB/s" % (ms, 0.4 / ms * 1e3))
