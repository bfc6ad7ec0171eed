"""Cycles and solve time to 1e-8 for splits of the paper's four smoothing
steps per cycle between pre- and post-smoothing (dev study)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2101_08453_b200 as wd  # noqa: E402
import synth  # noqa: E402


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["small", "medium", "paper"]
    for cfg in cfgs:
        p = synth.make(cfg, device=torch.device("cuda:0"))
        for pre, post in [(2, 2), (1, 3), (3, 1), (0, 4), (4, 0)]:
            ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(pre_smooth=pre, post_smooth=post))
            f = wd.wd_rhs(ctx, p.u0)
            wd.wd_solve(ctx, f, rel_tol=1e-8, raise_on_noconv=False)   # warm-up (graph capture)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-8, raise_on_noconv=False)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"config": cfg, "pre": pre, "post": post, "cycles": rep["cycles"],
                              "rate": rep["rate"], "solve_ms": e0.elapsed_time(e1)}), flush=True)
            ctx.close()
        del p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
