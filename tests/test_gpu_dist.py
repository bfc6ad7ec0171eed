"""Slab decomposition on one GPU through the virtual-rank mode:
the grid split into R slabs with the same halo exchanges and coarse gather
the NCCL path performs, done as device copies.  The iterates of the method
are partition invariant by construction (each node update sees identical
neighbour values, transfers are fixed-order gathers), so lambda after every
V-cycle, the RHS and the recovered wind must be BITWISE equal to the
single-GPU context."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _ctx(wd, p, nranks, gather, smoother="fused"):
    opt = wd.default_options(coarsest_max_free=200, nranks=nranks, rank=-1 if nranks > 1 else 0,
                             gather_below_nodes=gather, smoother=smoother)
    return wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)


PROBLEMS = {
    "small": lambda: synth.small(device=DEV),
    "ragged": lambda: synth.hill(nx=45, ny=38, nz=6, dx=40.0, height=120.0, sigma=300.0, dz0=8.0,
                                 r=1.3, a=(1, 1, 3), device=DEV),
}


@pytest.mark.parametrize("name", list(PROBLEMS))
@pytest.mark.parametrize("nranks,gather,smoother", [(2, 10 ** 9, "fused"), (3, 1000, "fused"),
                                                    (4, 1000, "fused"), (5, 50000, "fused"),
                                                    (3, 1000, "phased"), (3, 1000, "line")])
def test_virtual_ranks_bitwise(wd, name, nranks, gather, smoother):
    """Fused sweeps on slabs: one 2-row exchange per sweep, halo row recomputed;
    phased: exchanges after colours 1 and 3.  Both against one part (fused)."""
    p = PROBLEMS[name]()
    ref = _ctx(wd, p, 1, 0, "line" if smoother == "line" else "fused")
    ctx = _ctx(wd, p, nranks, gather, smoother)
    assert ctx.num_levels() == ref.num_levels()
    gl = wd.wd_gather_level(ctx)
    assert gl >= 1
    f1 = wd.wd_rhs(ref, p.u0)
    fR = wd.wd_rhs(ctx, p.u0)
    assert torch.equal(f1, fR)
    lam1 = synth.random_lambda(p, 4).to(DEV)
    lamR = lam1.clone()
    for c in range(3):
        r1 = wd.wd_vcycle(ref, lam1, f1)
        rR = wd.wd_vcycle(ctx, lamR, fR)
        assert torch.equal(lam1, lamR), (c, float((lam1 - lamR).abs().max()))
        assert abs(r1 - rR) <= 1e-12 * r1
    l1, rep1 = wd.wd_solve(ref, f1, rel_tol=1e-9)
    lR, repR = wd.wd_solve(ctx, fR, rel_tol=1e-9)
    assert rep1["cycles"] == repR["cycles"] and torch.equal(l1, lR)
    u1 = wd.wd_recover_wind(ref, l1, p.u0)
    uR = wd.wd_recover_wind(ctx, lR, p.u0)
    assert torch.equal(u1, uR)
    ctx.close()
    ref.close()


def test_virtual_ranks_partition_rules(wd):
    p = synth.tiny(device=DEV)
    with pytest.raises(wd.WDError) as e:         # 17 rows over 5 ranks: 3 rows < 4
        _ctx(wd, p, 5, 1000)
    assert e.value.code == wd.WD_E_INVAL
    ctx = _ctx(wd, p, 4, 10 ** 9)
    assert wd.wd_gather_level(ctx) == 1
    f = wd.wd_rhs(ctx, p.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
    assert rep["converged"]


def test_virtual_ranks_f4_entry_points(wd):
    """Diagnostics and the one-call time step on 3 slabs equal one part:
    wd_mass_consistency (norms summed in rank order) and wd_downscale_step."""
    p = PROBLEMS["ragged"]()
    ref = _ctx(wd, p, 1, 0)
    ctx = _ctx(wd, p, 3, 1000)
    a = wd.wd_mass_consistency(ref, p.u0)
    b = wd.wd_mass_consistency(ctx, p.u0)
    assert abs(a[0] - b[0]) <= 1e-12 * a[0] and a[1] == b[1]
    l1 = torch.zeros(ref.node_shape, dtype=torch.float64, device=DEV)
    lR = l1.clone()
    u1, r1 = wd.wd_downscale_step(ref, p.u0, l1, warm=False, rel_tol=1e-9)
    uR, rR = wd.wd_downscale_step(ctx, p.u0, lR, warm=False, rel_tol=1e-9)
    assert r1["cycles"] == rR["cycles"] and torch.equal(l1, lR) and torch.equal(u1, uR)
    ctx.close()
    ref.close()


def test_nccl_one_rank_bitwise(wd):
    """The NCCL code path on one GPU: libnccl found by dlopen, a one-rank
    communicator, empty exchange groups, rank sums through ncclAllGather
    (also inside the captured V-cycle graph).  Bitwise equal to the
    single-GPU context."""
    p = PROBLEMS["ragged"]()
    n2 = p.X.shape[1]
    comm = wd.wd_nccl_comm_init(wd.wd_nccl_unique_id(), 1, 0)
    ref = _ctx(wd, p, 1, 0)
    jb, je = wd.wd_partition_rows(n2, 1, 0)
    assert (jb, je) == (0, n2)
    opt = wd.default_options(coarsest_max_free=200, nranks=1, rank=0, nccl_comm=comm,
                             j_begin=jb, j_end=je)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)
    f1, fN = wd.wd_rhs(ref, p.u0), wd.wd_rhs(ctx, p.u0)
    assert torch.equal(f1, fN)
    l1, rep1 = wd.wd_solve(ref, f1, rel_tol=1e-9)
    lN, repN = wd.wd_solve(ctx, fN, rel_tol=1e-9)
    assert rep1["cycles"] == repN["cycles"]
    assert torch.equal(l1, lN)
    assert torch.equal(wd.wd_recover_wind(ref, l1, p.u0), wd.wd_recover_wind(ctx, lN, p.u0))
    ctx.close()
    ref.close()


@pytest.mark.parametrize("name", list(PROBLEMS))
@pytest.mark.parametrize("nranks,use_graph", [(2, 1), (3, 1), (4, 0), (6, 1)])
def test_boundary_first_overlap_bitwise(wd, name, nranks, use_graph):
    """Boundary-first sweeps (wd_options.overlap_halo = 1; off by default):
    each fused sweep on a distributed level runs the tile rows holding the
    first / last 2 owned rows, exchanges those rows on a second stream while
    the interior tile rows run, and skips the next sweep's leading exchange.
    Every V-cycle iterate, the solve and its history equal the serial order
    (overlap_halo = 0) and one part bit for bit."""
    p = PROBLEMS[name]()

    def mk(nr, ov):
        opt = wd.default_options(coarsest_max_free=200, nranks=nr, rank=-1 if nr > 1 else 0,
                                 gather_below_nodes=1000, overlap_halo=ov, use_graph=use_graph)
        return wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)

    ref, ser, ovl = mk(1, 0), mk(nranks, 0), mk(nranks, 1)
    try:
        f = wd.wd_rhs(ref, p.u0)
        lams = [synth.random_lambda(p, 6).to(DEV) for _ in range(3)]
        for c in range(3):
            for ctx, lam in zip((ref, ser, ovl), lams):
                wd.wd_vcycle(ctx, lam, f)
            assert torch.equal(lams[0], lams[1]) and torch.equal(lams[1], lams[2]), c
        out = [wd.wd_solve(ctx, f, rel_tol=1e-9) for ctx in (ref, ser, ovl)]
        assert torch.equal(out[0][0], out[2][0]) and torch.equal(out[1][0], out[2][0])
        assert out[0][1]["hist"] == out[2][1]["hist"] or all(
            abs(a - b) <= 1e-12 * b for a, b in zip(out[0][1]["hist"], out[2][1]["hist"]) if b)
        assert out[1][1]["hist"] == out[2][1]["hist"]
    finally:
        for ctx in (ref, ser, ovl):
            ctx.close()
    # longer runs of consecutive sweeps (4 pre, 3 post): each reuses the halo
    # rows the previous sweep's overlapped exchange brought
    opt = dict(coarsest_max_free=200, nranks=nranks, rank=-1, gather_below_nodes=1000,
               pre_smooth=4, post_smooth=3, use_graph=use_graph)
    a = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(overlap_halo=0, **opt))
    b = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(overlap_halo=1, **opt))
    try:
        x1, x2 = synth.random_lambda(p, 8).to(DEV), synth.random_lambda(p, 8).to(DEV)
        for _ in range(2):
            wd.wd_vcycle(a, x1, f)
            wd.wd_vcycle(b, x2, f)
        assert torch.equal(x1, x2)
    finally:
        a.close()
        b.close()
