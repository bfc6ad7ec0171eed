"""In-place read-modify-write vs copy bandwidth on this GPU (dev probe)."""
import torch
n = 135_000_000
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.randn(n, dtype=torch.float64, device="cuda")
z = torch.randn(n // 4, dtype=torch.float64, device="cuda")
def t(fn, nbytes, name, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:28s} {ms:7.3f} ms  {nbytes / ms / 1e6:7.1f} GB/s")
t(lambda: y.copy_(x), 16 * n, "copy y=x")
t(lambda: x.mul_(1.0000001), 16 * n, "in-place x*=a")
t(lambda: x.add_(y), 24 * n, "in-place x+=y")
t(lambda: x.view(-1, 4).add_(z.view(-1, 1)), 16 * n + 8 * n // 4, "in-place x+=bcast(z)")
