"""wd_rhs / wd_recover_wind device time at Paper-scale (CUDA events, median of 20)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2101_08453_b200 as wd  # noqa: E402
import synth  # noqa: E402

p = synth.make(sys.argv[1] if len(sys.argv) > 1 else "paper", device="cuda")
ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
f = wd.wd_rhs(ctx, p.u0)
lam = torch.randn_like(f)
u = torch.empty_like(p.u0)
out = {}
for name, fn in (("rhs", lambda: wd.wd_rhs(ctx, p.u0, f)),
                 ("recover", lambda: wd.wd_recover_wind(ctx, lam, p.u0, u))):
    ts = []
    for _ in range(22):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    out[name] = ts[len(ts) // 2]
print(json.dumps(out))
