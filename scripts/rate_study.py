#!/usr/bin/env python
"""Convergence-rate study: V-cycle convergence factor and
cycles to rel. residual 1e-8 over penalty a3, the coarsening-rule readings
(C1/C1b of DESIGN.md and the base method's full coarsening) and the
smoother (point GS of P:174-176 / vertical line relaxation).

  * S:539-style hill grids (64x64x16, dx 50 m, sigma 500 m, dz0 10 m, r 1.3;
    heights 100 m and 300 m), random RHS, 10 cycles: GPU and oracle side by side;
  * the BASELINE configs Small / Medium / Paper-scale with their physical RHS:
    GPU only (the oracle at Medium/Paper size takes minutes per solve).

Prints one JSON line per case.  Needs a GPU.
  python scripts/rate_study.py [--configs small,medium,paper] [--no-oracle]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

RULES = ["coupling_cur", "coupling_paper", "verbatim", "full"]
SMOOTHERS = {"gs": "fused", "line": "line"}


def work(ctx):
    """nodes of all levels / nodes of the fine level"""
    n = [np.prod(ctx.level_dims(l)) for l in range(ctx.num_levels())]
    return float(sum(n) / n[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="small,medium,paper")
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd
    import synth
    import oracle
    from brute import free_mask
    dev = torch.device("cuda:0")

    # hill grids, random RHS, fixed 10 cycles
    for height in (100.0, 300.0):
        for a3 in (1, 10, 100):
            p = synth.hill(height=height, a=(1, 1, a3))
            X, Y, Z, _ = p.numpy()
            g = p.to(dev)
            rng = np.random.default_rng(0)
            f = rng.standard_normal(X.shape) * free_mask(X.shape)
            for rule in RULES:
                for sm, gsm in SMOOTHERS.items():
                    opt = wd.default_options(coarsen_rule=rule, smoother=gsm, max_cycles=10)
                    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
                    _, rep = wd.wd_solve(ctx, torch.as_tensor(f, device=dev), rel_tol=1e-30,
                                         raise_on_noconv=False)
                    d = {"grid": f"hill h={height:g} 64x64x16", "a3": a3, "rule": rule,
                         "smoother": sm, "levels": ctx.num_levels(), "gpu_rate": rep["rate"],
                         "work": work(ctx)}
                    ctx.close()
                    if not args.no_oracle:
                        mg = oracle.MG(X, Y, Z, p.a, rule=rule, smoother=sm)
                        _, ro = mg.solve(f, tol=1e-30, max_cycles=10)
                        d["oracle_rate"] = ro["rate"]
                    print(json.dumps(d), flush=True)

    # configs with their physical RHS, solved to 1e-8 from zero
    for name in args.configs.split(","):
        if not name:
            continue
        p = synth.make(name, device=dev)
        for rule in RULES:
            for sm, gsm in SMOOTHERS.items():
                opt = wd.default_options(coarsen_rule=rule, smoother=gsm, max_cycles=60)
                t0 = time.time()
                ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)
                f = wd.wd_rhs(ctx, p.u0)
                torch.cuda.synchronize()
                t1 = time.time()
                _, rep = wd.wd_solve(ctx, f, rel_tol=1e-8, raise_on_noconv=False)
                torch.cuda.synchronize()
                t2 = time.time()
                print(json.dumps({"grid": name, "a3": p.a[2], "rule": rule, "smoother": sm,
                                  "levels": [list(ctx.level_dims(l)) for l in range(ctx.num_levels())],
                                  "work": work(ctx), "coarse_direct": rep["coarse_direct"],
                                  "cycles": rep["cycles"], "converged": rep["converged"],
                                  "rate": rep["rate"], "setup_s": t1 - t0, "solve_s": t2 - t1}),
                      flush=True)
                ctx.close()


if __name__ == "__main__":
    main()
