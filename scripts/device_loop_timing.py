#!/usr/bin/env python
"""wd_solve time with the cycle loop on the device (conditional WHILE graph,
the default) against the host-driven loop, per config (CUDA events around
wd_solve from the zero start to 1e-8; the two contexts alternate, N solves each).

  python scripts/device_loop_timing.py [--configs tiny,small,medium,paper] [--n 30]
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
    ap.add_argument("--configs", default="tiny,small,medium,paper")
    ap.add_argument("--n", type=int, default=30)
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd
    import synth
    dev = torch.device("cuda:0")
    for name in args.configs.split(","):
        p = synth.make(name, device=dev)
        ctxs = {dl: wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(device_loop=dl))
                for dl in (1, 0)}
        f = wd.wd_rhs(ctxs[1], p.u0)
        lam = torch.empty_like(f)
        ts = {1: [], 0: []}
        cyc = {}
        for it in range(args.n + 2):   # interleaved, 2 warm-up rounds
            for dl in (1, 0):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                torch.cuda.synchronize()
                e0.record()
                _, rep = wd.wd_solve(ctxs[dl], f, rel_tol=1e-8, lam=lam)
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    ts[dl].append(e0.elapsed_time(e1))
                cyc[dl] = rep["cycles"]
        out = {"config": name, "n": args.n}
        for dl, key in ((1, "device_loop"), (0, "host_loop")):
            t = sorted(ts[dl])
            out[key] = {"solve_ms_median": t[len(t) // 2], "solve_ms_min": t[0], "cycles": cyc[dl]}
        out["saved_us_per_cycle_median"] = 1e3 * (out["host_loop"]["solve_ms_median"] -
                                                  out["device_loop"]["solve_ms_median"]) / max(cyc[0], 1)
        print(json.dumps(out), flush=True)
        for c in ctxs.values():
            c.close()
        del f, lam
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
