"""Setup kernels at Paper-scale through wd_bench_kernel: assembly and the
Galerkin products of every transition (CUDA events, ms per launch)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2101_08453_b200 as wd  # noqa: E402
import synth  # noqa: E402

p = synth.make(sys.argv[1] if len(sys.argv) > 1 else "paper", device="cuda")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
out = {"assemble": wd.wd_bench_kernel(ctx, "assemble", 0, reps)}
for l in range(ctx.num_levels() - 1):
    out[f"galerkin{l}"] = wd.wd_bench_kernel(ctx, "galerkin", l, reps)
out["galerkin_total"] = sum(v for k, v in out.items() if k.startswith("galerkin"))
print(json.dumps(out))
