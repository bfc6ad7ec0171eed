#!/usr/bin/env python
"""Per-kernel timing (CUDA events, through wd_bench_kernel) on a config, with
algorithmic bytes -> GB/s.  Development tool; prints one JSON line per kernel.

  python scripts/kbench.py [--config paper] [--reps 10] [--apply-variants 0,1,2,3]
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--apply-variants", default="")
    ap.add_argument("--only", default="", help="comma list of level-0 kernels; skip the rest")
    ap.add_argument("--breakdown", action="store_true",
                    help="sweep/apply/restrict/prolong at every level (V-cycle time per level)")
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd
    import synth
    dev = torch.device("cuda:0")
    p = synth.make(args.config, device=dev)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
    f = wd.wd_rhs(ctx, p.u0)
    if not args.only:
        lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-8)
    n1, n2, n3 = ctx.level_dims(0)
    free0 = (n1 - 2) * (n2 - 2) * (n3 - 1)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    alg = {"gs_sweep": 136 * free0, "gs_sweep_res": 136 * free0, "gs_sweep_phased": 264 * free0, "apply": 136 * free0, "residual_norm": 128 * free0,
           "prolong": 16 * free0, "restrict": 8 * free0 + 8 * free0 // 4}

    def report(name, level=0, extra=None):
        ms = wd.wd_bench_kernel(ctx, name, level, args.reps)
        d = {"kernel": name, "level": level, "ms": ms}
        if level == 0 and name in alg:
            gbs = alg[name] / (ms * 1e-3) / 1e9
            d.update(alg_GBps=gbs, frac=gbs / peak)
        if extra:
            d.update(extra)
        print(json.dumps(d), flush=True)

    if args.breakdown:
        tot = 0.0
        for l in range(ctx.num_levels() - 1):
            t = {k: wd.wd_bench_kernel(ctx, k, l, args.reps)
                 for k in ("gs_sweep", "apply", "restrict", "prolong")}
            est = 4 * t["gs_sweep"] + t["apply"] + t["restrict"] + t["prolong"]
            tot += est
            print(json.dumps({"level": l, "dims": ctx.level_dims(l), **t, "est_level_ms": est}),
                  flush=True)
        print(json.dumps({"vcycle_ms": wd.wd_bench_kernel(ctx, "vcycle", 0, args.reps),
                          "sum_levels_ms": tot}), flush=True)
        return
    if args.only:
        for name in args.only.split(","):
            report(name)
        return
    for name in ["gs_sweep", "gs_sweep_res", "gs_sweep_phased", "apply", "residual_norm", "restrict", "prolong", "vcycle"]:
        report(name)
    for l in range(1, ctx.num_levels() - 1):
        report("gs_sweep", l)
        report("gs_sweep_phased", l)
    report("assemble")
    for l in range(ctx.num_levels() - 1):
        report("galerkin", l)
    if args.apply_variants:
        tiny = synth.tiny(device=dev)
        for v in args.apply_variants.split(","):
            os.environ["WD_APPLY_VARIANT"] = v
            wd.wd_assemble(tiny.X, tiny.Y, tiny.Z, tiny.a).close()   # re-reads the knob
            report("apply", 0, {"variant": int(v)})
    print(json.dumps({"levels": [ctx.level_dims(l) for l in range(ctx.num_levels())],
                      "cycles": rep["cycles"], "device_bytes": ctx.device_bytes()}))


if __name__ == "__main__":
    main()
