"""H2D bandwidth stability: 12 timed 1.06 GB copies from pinned host memory (C5b input size)."""
import time
import torch

n = 1064928092 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
out = []
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    s.synchronize()
    out.append((time.perf_counter() - t0) * 1e3)
print("H2D 1.06 GB ms:", [round(x, 1) for x in out])
