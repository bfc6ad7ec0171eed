"""Pinned host <-> device copy bandwidth on this box (dev probe)."""
import torch
n = 400_000_000   # 3.2 GB of doubles
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {8 * n / ms / 1e6:.1f} GB/s ({ms:.1f} ms for {8 * n / 1e9:.1f} GB)")
