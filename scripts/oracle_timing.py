#!/usr/bin/env python
"""The oracle (test infrastructure, plain C + OpenMP) timed on the host cores
on whole BASELINE configs: RHS + hierarchy setup, one V-cycle, the solve to
rel. residual 1e-8 from zero, the recovery.  One JSON line per config.

  python scripts/oracle_timing.py tiny small medium > profiles/r2_oracle_timing.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from parity_full import host_info  # noqa: E402


def main():
    for name in sys.argv[1:] or ["tiny", "small", "medium"]:
        p = synth.make(name)
        X, Y, Z, u0 = p.numpy()
        n1, n2, n3 = p.dims
        t = time.perf_counter()
        f = oracle.rhs(X, Y, Z, u0)
        mg = oracle.MG(X, Y, Z, p.a)
        t_setup = time.perf_counter() - t
        t = time.perf_counter()
        mg.vcycle(np.zeros_like(f), f)
        t_vc = time.perf_counter() - t
        t = time.perf_counter()
        lam, rep = mg.solve(f, tol=1e-8)
        t_solve = time.perf_counter() - t
        t = time.perf_counter()
        oracle.recover(X, Y, Z, p.a, lam, u0)
        t_rec = time.perf_counter() - t
        nodes = n1 * n2 * n3
        print(json.dumps(dict(config=name, dims=[n1, n2, n3], host=host_info(),
                              levels=[list(d) for d in mg.dims], setup_s=t_setup,
                              vcycle_s=t_vc, cycles_to_1e8=rep["cycles"], rate=rep["rate"],
                              time_to_1e8_s=t_solve, recover_s=t_rec,
                              node_cycles_per_s=nodes * rep["cycles"] / t_solve if t_solve else None)),
              flush=True)
        del mg


if __name__ == "__main__":
    main()
