#!/usr/bin/env python
"""Whole-solve GPU-vs-oracle parity at a full BASELINE size (tests/parity_full.py),
written as one JSON artifact:

  python scripts/parity_fullsize.py --config paper --warm 10 --out profiles/r2_parity_paper.json

The oracle (test infrastructure) runs on all host cores; host CPU model, core
count and memory are recorded with its timings.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    ap.add_argument("--warm", type=int, default=0)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd
    from parity_full import solve_parity
    # host-memory guard: the oracle holds ~310 B per fine node (27-coefficient
    # stencils on all levels + vectors), the script ~100 B more (inputs, outputs)
    n1, n2, n3 = {"tiny": (17, 17, 9), "small": (129, 129, 11), "medium": (1001, 1001, 16),
                  "paper": (3001, 3001, 16)}[args.config]
    need = 420 * n1 * n2 * n3
    avail = 0
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable"):
            avail = int(line.split()[1]) * 1024
    if avail < 1.3 * need:
        print(json.dumps({"skipped": f"host memory {avail / 1e9:.1f} GB available, "
                                     f"need ~{1.3 * need / 1e9:.1f} GB"}))
        return
    res = solve_parity(args.config, wd, torch.device("cuda:0"), tol=args.tol,
                       warm_steps=args.warm, log=lambda m: print(m, flush=True))
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res["compare"]))


if __name__ == "__main__":
    main()
