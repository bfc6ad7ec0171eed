"""GPU steps either side of the solver against the oracle:
terrain-following mesh generation, coarse-wind interpolation to element
centres, mass-consistency diagnostics, and the one-call time step with the
persistent hierarchy.  Tolerances: mesh and interpolation <= 1e-13 relative
max (the GPU contracts to FMA), diagnostics <= 1e-12 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from brute import free_mask

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _levels(nz, dz0, r):
    return np.concatenate([[0.0], np.cumsum(dz0 * r ** np.arange(nz))])


@pytest.mark.parametrize("n1,n2,nz", [(17, 9, 8), (130, 67, 15)])
def test_build_mesh_parity(wd, n1, n2, nz):
    rng = np.random.default_rng(n1)
    zs = rng.uniform(0, 400, (n2, n1))
    zeta = _levels(nz, 10.0, 1.25)
    H = zs.max() + zeta[-1] + 5.0
    X, Y, Z = wd.wd_build_mesh(torch.as_tensor(zs, device=DEV), 100.0, -50.0, 33.0, 31.0, zeta, H)
    Xo, Yo, Zo = oracle.build_mesh(zs, 100.0, -50.0, 33.0, 31.0, zeta, H)
    for a, b in ((X, Xo), (Y, Yo), (Z, Zo)):
        a = a.cpu().numpy()
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    # host pointers through the same entry point
    Xh, Yh, Zh = wd.wd_build_mesh(torch.as_tensor(zs), 100.0, -50.0, 33.0, 31.0, zeta, H)
    assert torch.equal(Zh, Z.cpu())


def test_build_mesh_errors(wd):
    zs = torch.zeros((4, 5), dtype=torch.float64, device=DEV)
    zs[2, 3] = 100.0
    with pytest.raises(wd.WDError, match=r"WD_E_MESH.*i=3, j=2"):
        wd.wd_build_mesh(zs, 0, 0, 1, 1, [0.0, 10.0, 20.0], 50.0)
    with pytest.raises(wd.WDError, match="WD_E_INVAL"):
        wd.wd_build_mesh(zs, 0, 0, 1, 1, [0.0, 10.0, 10.0], 500.0)


def test_build_mesh_reproduces_paper_config(wd):
    """Paper-scale (configs[3]) terrain and levels -> the synthetic input mesh
    (sampled rows; 1.4e8 nodes)."""
    p = synth.make("paper", device=DEV)
    Z = p.Z
    zs = Z[0].contiguous()
    jj, ii = divmod(int(torch.argmax(zs)), zs.shape[1])
    zeta = (Z[:, jj, ii] - zs[jj, ii]).cpu().numpy()
    zeta[0] = 0.0
    H = float(Z[-1].max())
    dx = float(p.X[0, 0, 1] - p.X[0, 0, 0])
    dy = float(p.Y[0, 1, 0] - p.Y[0, 0, 0])
    X, Y, Zg = wd.wd_build_mesh(zs, 0.0, 0.0, dx, dy, zeta, H)
    for j in (0, 1, 1500, 2999, 3000):
        assert torch.allclose(Zg[:, j], Z[:, j], rtol=0, atol=1e-10 * H)
        assert torch.allclose(X[:, j], p.X[:, j], rtol=0, atol=1e-9)
    del X, Y, Zg, p


def _coarse_field(seed, nxc=6, nyc=5, nzc=7):
    rng = np.random.default_rng(seed)
    uc = rng.standard_normal((3, nzc, nyc, nxc)) * np.array([5.0, 5.0, 0.5])[:, None, None, None]
    hc = np.concatenate([[2.0], 2.0 + np.cumsum(rng.uniform(10, 200, nzc - 1))])
    return uc, hc


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_interp_wind_parity(wd, name):
    p = synth.make(name)
    X, Y, Z, _ = p.numpy()
    uc, hc = _coarse_field(1)
    Lx, Ly = X.max(), Y.max()
    args = (-0.1 * Lx, -0.05 * Ly, 0.25 * Lx, 0.3 * Ly)   # covers the domain, some clamping
    got = wd.wd_interp_wind(torch.as_tensor(uc, device=DEV), *args, hc, p.X.to(DEV), p.Y.to(DEV),
                            p.Z.to(DEV)).cpu().numpy()
    want = oracle.interp_wind(uc, *args, hc, X, Y, Z)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_mass_consistency_diagnostics(wd, name):
    """D1 norms against the oracle's one-point weak divergence; D1(u0) = -f;
    the recovered wind's D1 is below u0's (reading C12)."""
    p = synth.make(name)
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=100))
    m = free_mask(X.shape)
    d_o = oracle.d1(X, Y, Z, u0)
    l2, mx = wd.wd_mass_consistency(ctx, g.u0)
    assert abs(l2 - np.linalg.norm(d_o[m])) <= 1e-12 * np.linalg.norm(d_o[m])
    assert abs(mx - np.abs(d_o[m]).max()) <= 1e-12 * np.abs(d_o[m]).max()
    f = wd.wd_rhs(ctx, g.u0).cpu().numpy()
    assert abs(l2 - np.linalg.norm(f[m])) <= 1e-12 * np.linalg.norm(f[m])
    lam, rep = wd.wd_solve(ctx, torch.as_tensor(f, device=DEV), rel_tol=1e-10)
    u = wd.wd_recover_wind(ctx, lam, g.u0)
    l2u, _ = wd.wd_mass_consistency(ctx, u)
    du = oracle.d1(X, Y, Z, u.cpu().numpy())
    assert abs(l2u - np.linalg.norm(du[m])) <= 1e-10 * np.linalg.norm(du[m])
    assert l2u < l2   # Tiny: 0.35 of D1(u0) (the one-point quadrature floor of C12)
    ctx.close()


def test_downscale_step_equals_its_parts_and_warm_restart(wd):
    p = synth.small(device=DEV)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
    lam = torch.zeros(ctx.node_shape, dtype=torch.float64, device=DEV)
    u, rep = wd.wd_downscale_step(ctx, p.u0, lam, warm=False, rel_tol=1e-9)
    f = wd.wd_rhs(ctx, p.u0)
    l2, r2 = wd.wd_solve(ctx, f, rel_tol=1e-9)
    u2 = wd.wd_recover_wind(ctx, l2, p.u0)
    torch.cuda.synchronize()
    assert rep["cycles"] == r2["cycles"] and torch.equal(lam, l2) and torch.equal(u, u2)
    # a second step with the same u0, warm-started from the solution: <= 1 cycle
    u3, rep3 = wd.wd_downscale_step(ctx, p.u0, lam, warm=True, rel_tol=1e-9)
    assert rep3["cycles"] <= 1
    assert torch.allclose(u3, u, rtol=0, atol=1e-8 * float(u.abs().max()))
    ctx.close()


def test_recover_host_pointer_pipeline(wd):
    """wd_recover_wind with host arrays runs chunk-pipelined (copy-in of one
    chunk of element rows overlapping the recovery and copy-out of the
    previous one); every mix of host / device arguments gives the device
    result bit for bit (ragged row count: uneven chunks)."""
    import itertools
    p = synth.hill(nx=61, ny=77, nz=7, dx=40.0, height=150.0, sigma=400.0, dz0=8.0, r=1.2,
                   a=(1, 1, 5), device=DEV)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=100))
    f = wd.wd_rhs(ctx, p.u0)
    lam, _ = wd.wd_solve(ctx, f, rel_tol=1e-9)
    ref = wd.wd_recover_wind(ctx, lam, p.u0)
    torch.cuda.synchronize()
    for hl, hu0, hu in itertools.product([False, True], repeat=3):
        if not (hl or hu0 or hu):
            continue
        l_ = lam.cpu().pin_memory() if hl else lam
        u0_ = p.u0.cpu().pin_memory() if hu0 else p.u0
        out = torch.empty(p.u0.shape, dtype=torch.float64, device="cpu" if hu else DEV)
        if hu:
            out = out.pin_memory()
        got = wd.wd_recover_wind(ctx, l_, u0_, out)
        torch.cuda.synchronize()
        assert torch.equal(got.cpu(), ref.cpu()), (hl, hu0, hu)
    ctx.close()


def test_assemble_from_host_arrays_pipelined(wd):
    """wd_assemble with host X, Y, Z copies the coordinates in row chunks and
    starts the assembly of each chunk's tile rows as they arrive: the operator
    on every level equals the device-input assembly bit for bit."""
    p = synth.hill(nx=150, ny=93, nz=9, dx=40.0, height=200.0, sigma=600.0, dz0=8.0, r=1.2,
                   a=(1, 1, 10))
    g = p.to(DEV)
    opt = wd.default_options(coarsest_max_free=100)
    cd = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    ch = wd.wd_assemble(p.X.pin_memory(), p.Y.pin_memory(), p.Z.pin_memory(), p.a, opt)
    assert cd.num_levels() == ch.num_levels()
    for l in range(cd.num_levels()):
        assert torch.equal(wd.wd_get_stencil(cd, l).cpu(), wd.wd_get_stencil(ch, l).cpu()), l
    cd.close()
    ch.close()


def test_example_downscale_demo_runs():
    """examples/downscale_demo.py (mesh -> interpolation -> hierarchy -> warm
    time steps -> diagnostics) at a small size."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "examples", "downscale_demo.py"),
                          "--nx", "64", "--ny", "48", "--nz", "8", "--steps", "3"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = [l.split() for l in out.stdout.splitlines() if l.strip() and l.split()[0].isdigit()]
    assert len(rows) == 3
    for r in rows:
        assert float(r[3]) <= 1e-8            # converged
        assert float(r[5]) < float(r[4])      # projected wind more mass-consistent than u0
    assert int(rows[1][1]) < int(rows[0][1])  # warm start needs fewer cycles


def test_downscale_step_host_arrays(wd):
    """wd_downscale_step on pinned host arrays (u0 staged once, lambda and u
    copied back) equals the device-array call bit for bit, cold and warm."""
    p = synth.small(device=DEV)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
    lam_d = torch.zeros(ctx.node_shape, dtype=torch.float64, device=DEV)
    u_d, r_d = wd.wd_downscale_step(ctx, p.u0, lam_d, warm=False, rel_tol=1e-9)
    lam_h = torch.zeros(ctx.node_shape, dtype=torch.float64).pin_memory()
    u_h = torch.empty(p.u0.shape, dtype=torch.float64).pin_memory()
    u0_h = p.u0.cpu().pin_memory()
    _, r_h = wd.wd_downscale_step(ctx, u0_h, lam_h, warm=False, rel_tol=1e-9, u=u_h)
    torch.cuda.synchronize()
    assert r_h["cycles"] == r_d["cycles"]
    assert torch.equal(lam_h, lam_d.cpu()) and torch.equal(u_h, u_d.cpu())
    u0b = (p.u0 * 1.01).contiguous()
    _, r2d = wd.wd_downscale_step(ctx, u0b, lam_d, warm=True, rel_tol=1e-9)
    _, r2h = wd.wd_downscale_step(ctx, u0b.cpu().pin_memory(), lam_h, warm=True, rel_tol=1e-9, u=u_h)
    torch.cuda.synchronize()
    assert r2h["cycles"] == r2d["cycles"] and torch.equal(lam_h, lam_d.cpu())
    ctx.close()


def test_c_api_demo_runs(tmp_path):
    """examples/c_api_demo.c (host arrays through the C ABI only): converges,
    the projection lowers the weak divergence, and the lowest-layer vertical
    wind is up on the windward and down on the lee side of the hill."""
    import subprocess
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_abi import _build_c_demo
    exe = str(tmp_path / "c_api_demo")
    r = _build_c_demo(exe)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    vals = {}
    for line in out.stdout.splitlines():
        toks = line.replace("|", " ").split()
        for a, b in zip(toks, toks[1:]):
            try:
                vals.setdefault(a, float(b))
            except ValueError:
                pass
    assert vals["residual"] <= 1e-8
    assert float(out.stdout.split("|D1 u| =")[1].split()[0]) < float(out.stdout.split("|D1 u0| =")[1].split()[0])
    assert vals["windward"] > 0 and vals["lee"] < 0
