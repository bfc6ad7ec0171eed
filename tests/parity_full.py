"""Whole-solve parity at BASELINE.json's full sizes: the GPU path against the
oracle's own multigrid solve on the same seeded inputs (north_star: "lambda
after both solves are converged to relative residual 1e-10 to <= 1e-8
relative L2; the V-cycle convergence factor within 10% of the oracle's").

Used by tests/test_gpu_fullparity.py (Medium, configs[2]) and by
scripts/parity_fullsize.py (Paper-scale configs[3] and the warm-start
sequence configs[4]; artifact profiles/r2_parity_*.json).  Test
infrastructure: it calls oracle/ and the product binding side by side.
"""
from __future__ import annotations

import os
import platform
import time

import numpy as np
import torch

import oracle
import synth

TOL_LAM = 1e-8    # lambda, u: relative l2 (north_star)
TOL_RATE = 0.10   # convergence factor: relative (north_star)
TOL_F = 1e-12     # RHS: relative max (north_star)


def host_info() -> dict:
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem = int(line.split()[1]) * 1024
    except OSError:
        pass
    return dict(cpu_model=model or platform.processor(), nproc=os.cpu_count(),
                oracle_threads=oracle.num_threads(), host_mem_bytes=mem)


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def cycles_to(hist, tol):
    """cycles of 'cycle, then test' to reach tol from the residual history"""
    for c, r in enumerate(hist):
        if r <= tol:
            return c
    return None


def solve_parity(name: str, wd, dev, tol=1e-10, warm_steps=0, log=print) -> dict:
    """GPU (bench.py's default options) and oracle on configs[name]: RHS, one
    V-cycle from zero, the solve to `tol` from zero, the recovered wind; and
    `warm_steps` steps of the warm-start sequence (configs[4]: each solve to
    1e-8 warm-started from the previous step's lambda, both sides from their
    own previous lambda), the last one then continued to `tol` on both sides."""
    out = dict(config=name, host=host_info(), rel_tol=tol)
    p = synth.make(name, device=dev)
    X, Y, Z, u0 = p.numpy()
    out["dims"] = list(p.dims)
    # ---- GPU
    t = time.time()
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
    f_g = wd.wd_rhs(ctx, p.u0)
    torch.cuda.synchronize()
    lam_g, rep_g = wd.wd_solve(ctx, f_g, rel_tol=tol)
    u_g = wd.wd_recover_wind(ctx, lam_g, p.u0)
    v1_g = torch.zeros_like(f_g)
    wd.wd_vcycle(ctx, v1_g, f_g, want_residual=False)
    torch.cuda.synchronize()
    out["gpu"] = dict(levels=rep_g["dims"], cycles=rep_g["cycles"], rate=rep_g["rate"],
                      hist=rep_g["hist"], cycles_to_1e8=cycles_to(rep_g["hist"], 1e-8),
                      wall_s=time.time() - t)
    log(f"[{name}] gpu: {rep_g['cycles']} cycles, rate {rep_g['rate']:.4f}")
    # ---- oracle
    t = time.time()
    f_o = oracle.rhs(X, Y, Z, u0)
    t_rhs = time.time() - t
    t = time.time()
    mg = oracle.MG(X, Y, Z, p.a)
    t_setup = time.time() - t
    log(f"[{name}] oracle setup {t_setup:.1f} s, levels {mg.dims}")
    t = time.time()
    v1_o = mg.vcycle(np.zeros_like(f_o), f_o)
    t_vc = time.time() - t
    t = time.time()
    lam_o, rep_o = mg.solve(f_o, tol=tol)
    t_solve = time.time() - t
    t = time.time()
    u_o = oracle.recover(X, Y, Z, p.a, lam_o, u0)
    t_rec = time.time() - t
    hist_o = rep_o["hist"].tolist()
    out["oracle"] = dict(levels=[list(d) for d in mg.dims], cycles=rep_o["cycles"],
                         rate=rep_o["rate"], hist=hist_o, status=rep_o["status"],
                         cycles_to_1e8=cycles_to(hist_o, 1e-8),
                         time_s=dict(rhs=t_rhs, setup=t_setup, vcycle=t_vc, solve=t_solve,
                                     recover=t_rec))
    log(f"[{name}] oracle: {rep_o['cycles']} cycles, rate {rep_o['rate']:.4f}, "
        f"solve {t_solve:.1f} s")
    # ---- comparisons
    fg = f_g.cpu().numpy()
    lg = lam_g.cpu().numpy()
    ug = u_g.cpu().numpy()
    cmp = dict(
        levels_equal=[list(d) for d in mg.dims] == [list(d) for d in rep_g["dims"]],
        rhs_rel_max=float(np.abs(fg - f_o).max() / np.abs(f_o).max()),
        vcycle1_rel_max=float(np.abs(v1_g.cpu().numpy() - v1_o).max() / np.abs(v1_o).max()),
        lam_rel_l2=_rel_l2(lg, lam_o), u_rel_l2=_rel_l2(ug, u_o),
        cycles_diff=rep_g["cycles"] - rep_o["cycles"],
        rate_rel_diff=abs(rep_g["rate"] - rep_o["rate"]) / rep_o["rate"],
        hist_rel_diff_max=max(abs(a - b) / b for a, b in zip(rep_g["hist"], hist_o) if b > 0),
    )
    out["compare"] = cmp
    log(f"[{name}] compare {cmp}")
    del fg, ug, v1_o, u_o
    # ---- warm-start sequence (configs[4]: successive u0 from seeds 4..)
    if warm_steps:
        steps = []
        # the sequence starts from the converged 1e-8 solution of step 0
        lam_gs, _ = wd.wd_solve(ctx, f_g, rel_tol=1e-8)
        lam_os, _ = mg.solve(f_o, tol=1e-8)
        seq = synth.warm_sequence(p, steps=warm_steps)
        for s, us in enumerate(seq, start=1):
            fs_g = wd.wd_rhs(ctx, us)
            lam_gn, rg = wd.wd_solve(ctx, fs_g, lam0=lam_gs, rel_tol=1e-8)
            torch.cuda.synchronize()
            us_np = us.cpu().numpy()
            fs_o = oracle.rhs(X, Y, Z, us_np)
            t = time.time()
            lam_on, ro = mg.solve(fs_o, lam0=lam_os, tol=1e-8)
            ts = time.time() - t
            st = dict(step=s, gpu_cycles=rg["cycles"], oracle_cycles=ro["cycles"],
                      gpu_rel_res0=rg["rel_res0"], oracle_rel_res0=float(ro["hist"][0]),
                      gpu_rate=rg["rate"], oracle_rate=ro["rate"],
                      lam_rel_l2=_rel_l2(lam_gn.cpu().numpy(), lam_on), oracle_solve_s=ts)
            if s == warm_steps:   # the last step continued to tol on both sides
                lam_gt, _ = wd.wd_solve(ctx, fs_g, lam0=lam_gn, rel_tol=tol)
                lam_ot, _ = mg.solve(fs_o, lam0=lam_on, tol=tol)
                st["lam_rel_l2_at_tol"] = _rel_l2(lam_gt.cpu().numpy(), lam_ot)
                ug = wd.wd_recover_wind(ctx, lam_gt, us).cpu().numpy()
                uo = oracle.recover(X, Y, Z, p.a, lam_ot, us_np)
                st["u_rel_l2_at_tol"] = _rel_l2(ug, uo)
                del ug, uo
            log(f"[{name}] warm step {st}")
            steps.append(st)
            lam_gs, lam_os = lam_gn, lam_on
        out["warm"] = steps
    ctx.close()
    del mg
    return out
