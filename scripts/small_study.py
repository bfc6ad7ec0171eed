#!/usr/bin/env python
"""Why BASELINE configs[1] (Small) converges slowly (the
paper's claim of rates <= ~0.28 over "a range of grids and penalty
coefficients"): the oracle's V-cycle convergence factor
(C10, cycles to rel. residual 1e-8 from zero, physical RHS) on Small and on
variants of it that change one thing at a time -- the smoother, the
coarsening rule, the penalty a3 and the terrain amplitude (Z scaled between
the flat variant and the real terrain).  The GPU reproduces the oracle's
factors (profiles/r1f_rate_study.jsonl, tests/test_gpu_parity.py), so the
study runs the oracle only (CPU, a few minutes).

  python scripts/small_study.py > profiles/r2_small_study.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth   # noqa: E402


def run(name, X, Y, Z, a, u0, **kw):
    sm = kw.pop("smoother", "gs")
    mg = oracle.MG(X, Y, Z, a, smoother=sm, **kw)
    f = oracle.rhs(X, Y, Z, u0)
    _, rep = mg.solve(f, tol=1e-8, max_cycles=60)
    print(f"{name:44s} a3={a[2]:<4g} levels={len(mg.dims)} cycles={rep['cycles']:3d} "
          f"rate={rep['rate']:.3f}", flush=True)


def main():
    p = synth.small()
    X, Y, Z, u0 = p.numpy()
    Zf = synth.flat_variant(p).numpy()[2]
    print("# Small (128x128x10, dx 50 m, hills up to 400 m, a = (1, 1, 10)), 2+2 sweeps unless noted")
    for rule in ("coupling_cur", "coupling_paper", "verbatim", "full"):
        for sm in ("gs", "line"):
            run(f"rule={rule} smoother={sm}", X, Y, Z, p.a, u0, rule=rule, smoother=sm)
    run("3+3 sweeps (outside P:202's four)", X, Y, Z, p.a, u0, pre=3, post=3)
    print("# the same grid with a3 = 1 (isotropic coefficient)")
    for sm in ("gs", "line"):
        run(f"a3=1 smoother={sm}", X, Y, Z, (1.0, 1.0, 1.0), u0, smoother=sm)
    print("# terrain amplitude: Z = Z_flat + s (Z - Z_flat), a3 = 10")
    for s in (0.0, 0.25, 0.5, 0.75, 1.0):
        Zs = Zf + s * (Z - Zf)
        for sm in ("gs", "line"):
            run(f"terrain scale {s} smoother={sm}", X, Y, Zs, p.a, u0, smoother=sm)


if __name__ == "__main__":
    main()
