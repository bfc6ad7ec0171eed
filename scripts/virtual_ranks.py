#!/usr/bin/env python
"""The slab decomposition's own cost, measured on ONE GPU with virtual ranks
(wd.h opt.rank = -1): R slabs of the same grid run one after the
other on one device with the same halo exchanges (as device copies) and the
same replicated coarse levels.  Per R: setup, the solve to 1e-8 from zero and
its V-cycle time, the gather level, and a bitwise check of lambda against
R = 1.  The serial time over R parts is R x (one rank's compute) + the
replicated coarse levels R times; it bounds the work, not the NCCL latency.

  python scripts/virtual_ranks.py --config paper --ranks 1,2,4,8 > profiles/r2_virtual_ranks.jsonl
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--overlap", default="1", help="wd_options.overlap_halo values to run, e.g. 0,1")
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd
    import synth
    dev = torch.device("cuda:0")
    p = synth.make(args.config, device=dev)
    ref = None
    runs = [(int(r), int(o)) for r in args.ranks.split(",") for o in args.overlap.split(",")
            if int(r) > 1 or o == args.overlap.split(",")[0]]
    for R, ov in runs:
        opt = wd.default_options(profile=1, nranks=R, rank=-1 if R > 1 else 0, overlap_halo=ov)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)   # warm
        f = wd.wd_rhs(ctx, p.u0)
        wd.wd_solve(ctx, f, rel_tol=1e-8)
        ctx.close()
        setup, solve, cyc = 0.0, 0.0, 0
        for _ in range(args.reps):
            e[0].record()
            ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)
            e[1].record()
            f = wd.wd_rhs(ctx, p.u0)
            lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-8)
            e[2].record()
            torch.cuda.synchronize()
            setup += e[0].elapsed_time(e[1])
            solve += e[1].elapsed_time(e[2])
            cyc += rep["cycles"]
            prof = wd.wd_profile_read(ctx)
            gl = wd.wd_gather_level(ctx)
            if ref is None:
                ref = lam.clone()
            same = bool(torch.equal(lam, ref))
            ctx.close()
        line = dict(config=args.config, ranks=R, overlap_halo=ov, setup_ms=setup / args.reps,
                    solve_ms=solve / args.reps, cycles=cyc / args.reps,
                    vcycle_ms=prof["vcycle_ms"] / max(prof["vcycles"], 1),
                    gather_level=gl, lambda_bitwise_equal_to_1_rank=same)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
