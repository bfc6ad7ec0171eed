#!/usr/bin/env python
"""End-to-end use of the library inside a model time loop:

  terrain  --wd_build_mesh-->  terrain-following mesh (reading C13)
  coarse "WRF" wind  --wd_interp_wind-->  u0 at element centres
  wd_assemble (once per mesh: operator, hierarchy, coarsest inverse)
  per time step: wd_downscale_step (RHS + warm-started solve + recovery)
                 wd_mass_consistency (diagnostics of Eq. (1))

All arrays stay on the GPU; every step of the computation runs in the
library's sm_100a kernels.  Synthetic inputs only (no DEM / WRF data here).

  python examples/downscale_demo.py [--nx 256 --ny 256 --nz 12 --steps 5]
"""
import argparse
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def terrain(nx, ny, dx, seed):
    """A few Gaussian hills on a (ny+1, nx+1) node grid (metres)."""
    rng = np.random.default_rng(seed)
    x = np.arange(nx + 1) * dx
    y = np.arange(ny + 1) * dx
    X, Y = np.meshgrid(x, y)
    z = np.zeros_like(X)
    for _ in range(5):
        h, s = rng.uniform(80, 300), rng.uniform(5, 15) * dx
        cx, cy = rng.uniform(0, x[-1]), rng.uniform(0, y[-1])
        z += h * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2 * s * s))
    return z


def coarse_wind(Lx, Ly, t, seed):
    """A 1 km "WRF" grid with 10 levels: log profile, direction turning in time."""
    nxc, nyc = int(Lx // 1000) + 2, int(Ly // 1000) + 2
    hc = np.array([2.0, 10, 30, 60, 100, 200, 400, 700, 1200, 2000])
    ang = 0.3 + 0.1 * t + 0.2 * np.sin(np.linspace(0, math.pi, nxc))[None, None, :]
    speed = 8.0 * np.log((hc + 0.1) / 0.1) / math.log(10.1 / 0.1)
    uc = np.zeros((3, hc.size, nyc, nxc))
    uc[0] = speed[:, None, None] * np.cos(ang)
    uc[1] = speed[:, None, None] * np.sin(ang)
    return uc, hc, -500.0, -500.0, 1000.0, 1000.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--ny", type=int, default=256)
    ap.add_argument("--nz", type=int, default=12)
    ap.add_argument("--dx", type=float, default=30.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--tol", type=float, default=1e-8)
    args = ap.parse_args()
    import paper_2101_08453_b200 as wd

    dev = torch.device("cuda:0")
    zs = terrain(args.nx, args.ny, args.dx, seed=1)
    zs -= zs.min()
    zeta = np.concatenate([[0.0], np.cumsum(10.0 * 1.25 ** np.arange(args.nz))])
    H = zs.max() + zeta[-1]
    X, Y, Z = wd.wd_build_mesh(torch.as_tensor(zs, device=dev), 0.0, 0.0, args.dx, args.dx,
                               zeta, H)
    t0 = time.time()
    ctx = wd.wd_assemble(X, Y, Z, (1.0, 1.0, 10.0))
    torch.cuda.synchronize()
    print(f"mesh {args.nx}x{args.ny}x{args.nz} elements, hierarchy "
          f"{[ctx.level_dims(l) for l in range(ctx.num_levels())]} in {time.time() - t0:.2f} s")
    lam = torch.zeros(ctx.node_shape, dtype=torch.float64, device=dev)
    Lx, Ly = args.nx * args.dx, args.ny * args.dx
    print(f"{'step':>4s} {'cycles':>6s} {'rel0':>9s} {'rel':>9s} {'|D1 u0|':>10s} {'|D1 u|':>10s} {'ms':>7s}")
    for t in range(args.steps):
        uc, hc, xc0, yc0, dxc, dyc = coarse_wind(Lx, Ly, t, seed=2)
        u0 = wd.wd_interp_wind(torch.as_tensor(uc, device=dev), xc0, yc0, dxc, dyc, hc, X, Y, Z)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u, rep = wd.wd_downscale_step(ctx, u0, lam, warm=t > 0, rel_tol=args.tol)
        e1.record()
        torch.cuda.synchronize()
        d0, _ = wd.wd_mass_consistency(ctx, u0)
        d1, _ = wd.wd_mass_consistency(ctx, u)
        print(f"{t:4d} {rep['cycles']:6d} {rep['rel_res0']:9.2e} {rep['rel_res_final']:9.2e} "
              f"{d0:10.3e} {d1:10.3e} {e0.elapsed_time(e1):7.2f}")
    ctx.close()


if __name__ == "__main__":
    main()
