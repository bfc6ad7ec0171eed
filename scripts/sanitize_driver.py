#!/usr/bin/env python
"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck): one
pass of every kernel of the path on Tiny and on a ragged hill grid (37x22x5,
two tiles in x, a ragged tail), including both fused-sweep variants (plain and
residual-returning, k_gs_fused.cu and k_gs_fused2.cu), the TMA residual, the
transfers, the coarsest solve, RHS and recovery.  Run as

  compute-sanitizer --tool racecheck python scripts/sanitize_driver.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2101_08453_b200 as wd  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    grids = [synth.tiny(device=dev),
             synth.hill(nx=37, ny=22, nz=5, dx=40.0, height=120.0, sigma=300.0, dz0=8.0, r=1.3,
                        a=(1, 1, 3), device=dev)]
    for p in grids:
        for v2 in ("1", "0"):
            os.environ["WD_GS_V2"] = v2
            ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60,
                                                                         use_graph=0))
            f = wd.wd_rhs(ctx, p.u0)
            lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-6, raise_on_noconv=False)   # RES sweeps
            x = wd.wd_smooth(ctx, 0, lam.clone(), f, sweeps=2)
            wd.wd_apply(ctx, 0, x)
            wd.wd_residual_norm(ctx, x, f)
            wd.wd_recover_wind(ctx, lam, p.u0)
            torch.cuda.synchronize()
            print(p.name, "v2" if v2 == "1" else "v1", rep["cycles"], flush=True)
            ctx.close()
    os.environ.pop("WD_GS_V2", None)


if __name__ == "__main__":
    main()
