"""Seeded synthetic inputs for the wind-downscaling hot path.

This module is shared by the oracle tests and the GPU path.  It holds NONE of
the method's arithmetic (no element integrals, no solver): it only builds the
inputs the paper's problem statement takes -- node coordinates X, Y, Z of a
terrain-following grid of hexahedra and the initial wind u0 at element centres
(Sec. 2, "Given vector field u0 on domain Omega ...", and the
element/node layout of P:116-118).

Recipes follow SURVEY.md Sec. 8(d) ("Concrete synthetic inputs") and the
reading R1 of the domain top, restated in DESIGN.md Sec. 3:

* x_i = i*dx, y_j = j*dy;
* zeta_k = dz0*(r**k - 1)/(r - 1), T = zeta_nz;
* terrain shifted so that min z_s = 0, H = max z_s + T;
* Z(i,j,k) = z_s + zeta_k*(H - z_s)/T   (flat top at H, every cell valid).

Array conventions (C-contiguous, float64):
* node arrays X, Y, Z: shape (n3, n2, n1), i fastest;
* element array u0: shape (3, nz, ny, nx) (components u, v, w).

Random draws use ``numpy.random.default_rng(seed)`` in the order stated in
each recipe; the (large) evaluations use torch so they can run on either the
host or a device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

F64 = torch.float64


@dataclass
class Problem:
    name: str
    nx: int
    ny: int
    nz: int
    X: torch.Tensor
    Y: torch.Tensor
    Z: torch.Tensor
    u0: torch.Tensor
    a: tuple
    meta: dict = field(default_factory=dict)

    @property
    def dims(self):
        return (self.nx + 1, self.ny + 1, self.nz + 1)

    @property
    def n_nodes(self):
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_free(self):
        return (self.nx - 1) * (self.ny - 1) * self.nz

    def to(self, device):
        return Problem(self.name, self.nx, self.ny, self.nz, self.X.to(device),
                       self.Y.to(device), self.Z.to(device), self.u0.to(device),
                       self.a, dict(self.meta))

    def numpy(self):
        """(X, Y, Z, u0) as contiguous float64 numpy arrays."""
        return tuple(np.ascontiguousarray(t.detach().cpu().numpy())
                     for t in (self.X, self.Y, self.Z, self.u0))


# ---------------------------------------------------------------------------
# grid construction
# ---------------------------------------------------------------------------

def stretched_levels(nz: int, dz0: float, r: float) -> np.ndarray:
    """zeta_k = dz0 (r^k - 1)/(r - 1), k = 0..nz (geometric stretching)."""
    k = np.arange(nz + 1, dtype=np.float64)
    if r == 1.0:
        return dz0 * k
    return dz0 * (r ** k - 1.0) / (r - 1.0)


def terrain_following(zs: torch.Tensor, zeta: np.ndarray, dx: float, dy: float,
                      shift_min: bool = True):
    """Node coordinates of the terrain-following grid (reading R1).

    zs: (n2, n1) terrain heights.  Returns X, Y, Z of shape (n3, n2, n1).
    """
    dev = zs.device
    n2, n1 = zs.shape
    n3 = len(zeta)
    if shift_min:
        zs = zs - zs.min()
    T = float(zeta[-1])
    H = float(zs.max()) + T
    zt = torch.as_tensor(zeta, dtype=F64, device=dev).view(n3, 1, 1)
    Z = zs.unsqueeze(0) + zt * ((H - zs) / T).unsqueeze(0)
    x = torch.arange(n1, dtype=F64, device=dev) * dx
    y = torch.arange(n2, dtype=F64, device=dev) * dy
    X = x.view(1, 1, n1).expand(n3, n2, n1).contiguous()
    Y = y.view(1, n2, 1).expand(n3, n2, n1).contiguous()
    return X, Y, Z.contiguous()


def element_centres(X, Y, Z):
    """Centre of each element = mean of its 8 node coordinates."""
    def c(A):
        return 0.125 * (A[:-1, :-1, :-1] + A[:-1, :-1, 1:] + A[:-1, 1:, :-1] + A[:-1, 1:, 1:]
                        + A[1:, :-1, :-1] + A[1:, :-1, 1:] + A[1:, 1:, :-1] + A[1:, 1:, 1:])
    return c(X), c(Y), c(Z)


def height_above_ground(Z):
    """z_agl at element centres: centre z minus the mean of the column's 4 bottom z_s."""
    zc = element_centres(Z, Z, Z)[2]
    zs = Z[0]
    zb = 0.25 * (zs[:-1, :-1] + zs[:-1, 1:] + zs[1:, :-1] + zs[1:, 1:])
    return zc - zb.unsqueeze(0)


# ---------------------------------------------------------------------------
# terrains
# ---------------------------------------------------------------------------

def gaussian_hills(n1, n2, dx, dy, heights, sigmas, cx, cy, device="cpu"):
    x = torch.arange(n1, dtype=F64, device=device) * dx
    y = torch.arange(n2, dtype=F64, device=device) * dy
    zs = torch.zeros(n2, n1, dtype=F64, device=device)
    for h, s, xc, yc in zip(heights, sigmas, cx, cy):
        gx = torch.exp(-((x - xc) ** 2) / (2 * s * s))
        gy = torch.exp(-((y - yc) ** 2) / (2 * s * s))
        zs += h * gy.view(n2, 1) * gx.view(1, n1)
    return zs


def sinusoid_field(n1, n2, dx, dy, kvec, phase, amp, device="cpu"):
    """sum_m amp_m sin(kx_m x + ky_m y + phase_m), evaluated separably."""
    x = torch.arange(n1, dtype=F64, device=device) * dx
    y = torch.arange(n2, dtype=F64, device=device) * dy
    out = torch.zeros(n2, n1, dtype=F64, device=device)
    for (kx, ky), ph, am in zip(kvec, phase, amp):
        ax = kx * x
        by = ky * y + ph
        # sin(a + b) = sin a cos b + cos a sin b
        out += am * (torch.cos(by).view(n2, 1) * torch.sin(ax).view(1, n1)
                     + torch.sin(by).view(n2, 1) * torch.cos(ax).view(1, n1))
    return out


def fractal_ridges(rng, n1, n2, dx, dy, rms, slope_deg=35.0, device="cpu"):
    """64 random-phase sinusoids, |k_m| = 2 pi m / L, amplitude ~ |k_m|^-2,
    scaled to the given rms over the nodes; slopes capped at slope_deg
    (centred differences), min shifted to 0.  Draw order: theta[64], phi[64]."""
    L = max((n1 - 1) * dx, (n2 - 1) * dy)
    m = np.arange(1, 65, dtype=np.float64)
    kmag = 2 * np.pi * m / L
    theta = rng.uniform(0.0, np.pi, 64)
    phi = rng.uniform(0.0, 2 * np.pi, 64)
    kvec = np.stack([kmag * np.cos(theta), kmag * np.sin(theta)], 1)
    amp = kmag ** -2.0
    zs = sinusoid_field(n1, n2, dx, dy, kvec, phi, amp, device)
    zs = zs - zs.mean()
    zs = zs * (rms / float(torch.sqrt((zs * zs).mean())))
    gx = (zs[:, 2:] - zs[:, :-2]) / (2 * dx)
    gy = (zs[2:, :] - zs[:-2, :]) / (2 * dy)
    smax = max(float(gx.abs().max()), float(gy.abs().max()))
    cap = math.tan(math.radians(slope_deg))
    if smax > cap:
        zs = zs * (cap / smax)
    return zs - zs.min()


def direction_field(rng, n1, n2, dx, dy, device="cpu"):
    """g(x,y) in [-1,1]: normalised sum of 8 random-phase sinusoids with
    wavelengths >= L/4.  Draw order: psi[8], nu[8], phase[8]."""
    L = max((n1 - 1) * dx, (n2 - 1) * dy)
    psi = rng.uniform(0.0, np.pi, 8)
    nu = rng.uniform(1.0, 4.0, 8)           # wavelength = L / nu >= L/4
    ph = rng.uniform(0.0, 2 * np.pi, 8)
    kmag = 2 * np.pi * nu / L
    kvec = np.stack([kmag * np.cos(psi), kmag * np.sin(psi)], 1)
    g = sinusoid_field(n1, n2, dx, dy, kvec, ph, np.ones(8), device)
    return g / float(g.abs().max())


# ---------------------------------------------------------------------------
# winds
# ---------------------------------------------------------------------------

def log_profile_speed(z_agl, u_star_over_kappa=None, ref_speed=None, z_ref=10.0, z0=0.1):
    if ref_speed is not None:
        return ref_speed * torch.log((z_agl + z0) / z0) / math.log((z_ref + z0) / z0)
    return u_star_over_kappa * torch.log((z_agl + z0) / z0)


def _cell_avg2(a):
    return 0.25 * (a[:-1, :-1] + a[:-1, 1:] + a[1:, :-1] + a[1:, 1:])


# ---------------------------------------------------------------------------
# the five BASELINE configs
# ---------------------------------------------------------------------------

def tiny(device="cpu", seed=0):
    nx = ny = 16
    nz = 8
    dx = dy = 30.0
    n1, n2 = nx + 1, ny + 1
    rng = np.random.default_rng(seed)
    zs = gaussian_hills(n1, n2, dx, dy, [150.0], [120.0], [240.0], [240.0], device)
    X, Y, Z = terrain_following(zs, stretched_levels(nz, 5.0, 1.15), dx, dy)
    noise = torch.as_tensor(rng.normal(0.0, 0.1, (3, nz, ny, nx)), dtype=F64, device=device)
    u0 = noise.clone()
    u0[0] += 5.0
    return Problem("tiny", nx, ny, nz, X, Y, Z, u0.contiguous(), (1.0, 1.0, 1.0),
                   dict(dx=dx, dy=dy, dz0=5.0, r=1.15, seed=seed))


def small(device="cpu", seed=1):
    nx = ny = 128
    nz = 10
    dx = dy = 50.0
    n1, n2 = nx + 1, ny + 1
    rng = np.random.default_rng(seed)
    h = rng.uniform(50, 400, 6)
    s = rng.uniform(200, 800, 6)
    cx = rng.uniform(0, 6400, 6)
    cy = rng.uniform(0, 6400, 6)
    zs = gaussian_hills(n1, n2, dx, dy, h, s, cx, cy, device)
    X, Y, Z = terrain_following(zs, stretched_levels(nz, 10.0, 1.2), dx, dy)
    zagl = height_above_ground(Z)
    S = log_profile_speed(zagl, u_star_over_kappa=0.5 / 0.4)
    th = math.radians(30.0)
    noise = torch.as_tensor(rng.normal(0.0, 0.2, (3, nz, ny, nx)), dtype=F64, device=device)
    u0 = noise.clone()
    u0[0] += S * math.cos(th)
    u0[1] += S * math.sin(th)
    return Problem("small", nx, ny, nz, X, Y, Z, u0.contiguous(), (1.0, 1.0, 10.0),
                   dict(dx=dx, dy=dy, dz0=10.0, r=1.2, seed=seed))


def _ridge_config(name, nx, ny, nz, dx, rms, ref_speed, seed, device):
    n1, n2 = nx + 1, ny + 1
    rng = np.random.default_rng(seed)
    zs = fractal_ridges(rng, n1, n2, dx, dx, rms, device=device)
    X, Y, Z = terrain_following(zs, stretched_levels(nz, 10.0, 1.25), dx, dx)
    zagl = height_above_ground(Z)
    S = log_profile_speed(zagl, ref_speed=ref_speed)
    g = direction_field(rng, n1, n2, dx, dx, device)
    th = (math.pi / 4) * _cell_avg2(g)
    u0 = torch.zeros(3, nz, ny, nx, dtype=F64, device=device)
    u0[0] = S * torch.cos(th).unsqueeze(0)
    u0[1] = S * torch.sin(th).unsqueeze(0)
    del S
    return Problem(name, nx, ny, nz, X, Y, Z, u0, (1.0, 1.0, 10.0),
                   dict(dx=dx, dy=dx, dz0=10.0, r=1.25, seed=seed, rms=rms))


def medium(device="cpu", seed=2):
    return _ridge_config("medium", 1000, 1000, 15, 30.0, 200.0, 8.0, seed, device)


def paper(device="cpu", seed=3):
    return _ridge_config("paper", 3000, 3000, 15, 33.0, 300.0, 10.0, seed, device)


def warm_increment(prob: Problem, seed: int, rms=0.5, corr_len=2000.0):
    """Smooth horizontal increment Delta_s (u, v only), identical at all k:
    white noise on the (i,j) element grid, Gaussian filter sigma = corr_len via
    FFT, scaled to the given rms per component.  Draw order: u-noise, v-noise."""
    rng = np.random.default_rng(seed)
    nx, ny = prob.nx, prob.ny
    dx = prob.meta["dx"]
    out = []
    kx = np.fft.rfftfreq(nx, d=dx) * 2 * np.pi
    ky = np.fft.fftfreq(ny, d=dx) * 2 * np.pi
    filt = np.exp(-0.5 * corr_len ** 2 * (ky[:, None] ** 2 + kx[None, :] ** 2))
    for _ in range(2):
        w = rng.standard_normal((ny, nx))
        sm = np.fft.irfft2(np.fft.rfft2(w) * filt, s=(ny, nx))
        sm *= rms / np.sqrt(np.mean(sm * sm))
        out.append(sm)
    d = torch.zeros(3, prob.nz, ny, nx, dtype=F64, device=prob.u0.device)
    d[0] = torch.as_tensor(out[0], dtype=F64, device=d.device).unsqueeze(0)
    d[1] = torch.as_tensor(out[1], dtype=F64, device=d.device).unsqueeze(0)
    return d


def warm_sequence(prob: Problem, steps=10, first_seed=4):
    """u0_s = u0_{s-1} + Delta_s, s = 1..steps (seeds 4..13)."""
    u = prob.u0
    for s in range(steps):
        u = u + warm_increment(prob, first_seed + s)
        yield u


CONFIGS = {"tiny": tiny, "small": small, "medium": medium, "paper": paper}


def make(name: str, device="cpu") -> Problem:
    return CONFIGS[name](device=device)


# ---------------------------------------------------------------------------
# correctness-only grids
# ---------------------------------------------------------------------------

def box(nx, ny, nz, dx=1.0, dy=1.0, dz=None, a=(1.0, 1.0, 1.0), u0=(0.0, 0.0, 0.0),
        device="cpu", name="box"):
    """Flat box grid; dz is a scalar or an array of nz layer thicknesses."""
    n1, n2, n3 = nx + 1, ny + 1, nz + 1
    if dz is None:
        dz = 1.0
    dzs = np.full(nz, float(dz)) if np.isscalar(dz) else np.asarray(dz, dtype=np.float64)
    zeta = np.concatenate([[0.0], np.cumsum(dzs)])
    x = torch.arange(n1, dtype=F64, device=device) * dx
    y = torch.arange(n2, dtype=F64, device=device) * dy
    z = torch.as_tensor(zeta, dtype=F64, device=device)
    X = x.view(1, 1, n1).expand(n3, n2, n1).contiguous()
    Y = y.view(1, n2, 1).expand(n3, n2, n1).contiguous()
    Z = z.view(n3, 1, 1).expand(n3, n2, n1).contiguous()
    U = torch.zeros(3, nz, ny, nx, dtype=F64, device=device)
    for c in range(3):
        U[c] = u0[c]
    return Problem(name, nx, ny, nz, X, Y, Z, U, tuple(a), dict(dx=dx, dy=dy, dz=dzs))


def hill(nx=64, ny=64, nz=16, dx=50.0, height=300.0, sigma=500.0, dz0=10.0, r=1.3,
         a=(1.0, 1.0, 1.0), u0=(5.0, 0.0, 0.0), device="cpu", name="hill"):
    """Single centred Gaussian hill (SPEC acceptance-2 style grid)."""
    n1, n2 = nx + 1, ny + 1
    cx = 0.5 * nx * dx
    cy = 0.5 * ny * dx
    zs = gaussian_hills(n1, n2, dx, dx, [height], [sigma], [cx], [cy], device)
    X, Y, Z = terrain_following(zs, stretched_levels(nz, dz0, r), dx, dx)
    U = torch.zeros(3, nz, ny, nx, dtype=F64, device=device)
    for c in range(3):
        U[c] = u0[c]
    return Problem(name, nx, ny, nz, X, Y, Z, U, tuple(a), dict(dx=dx, dy=dx, dz0=dz0, r=r))


def flat_variant(prob: Problem) -> Problem:
    """Same levels and u0 recipe location, terrain == 0 (flat box with stretching)."""
    # the highest-terrain column of reading R1 carries zeta_k exactly
    n1 = prob.dims[0]
    flat_idx = int(torch.argmax(prob.Z[0]))
    jm, im = divmod(flat_idx, n1)
    col = prob.Z[:, jm, im] - prob.Z[0, jm, im]
    Z = col.view(-1, 1, 1).expand_as(prob.Z).contiguous()
    return Problem(prob.name + "_flat", prob.nx, prob.ny, prob.nz, prob.X, prob.Y, Z,
                   prob.u0, prob.a, dict(prob.meta))


def crop(prob: Problem, i0, j0, mx, my, name=None) -> Problem:
    """Sub-domain of mx x my element columns starting at element (i0, j0), all layers."""
    sl = (slice(None), slice(j0, j0 + my + 1), slice(i0, i0 + mx + 1))
    su = (slice(None), slice(None), slice(j0, j0 + my), slice(i0, i0 + mx))
    X = prob.X[sl].contiguous()
    X = X - X[0, 0, 0]
    Y = prob.Y[sl].contiguous()
    Y = Y - Y[0, 0, 0]
    return Problem(name or f"{prob.name}_crop{mx}x{my}", mx, my, prob.nz, X, Y,
                   prob.Z[sl].contiguous(), prob.u0[su].contiguous(), prob.a, dict(prob.meta))


def random_lambda(prob: Problem, seed=0, device=None):
    """lambda ~ U[-1, 1] on free nodes, 0 on the Dirichlet set (lateral + top)."""
    rng = np.random.default_rng(seed)
    n1, n2, n3 = prob.dims
    lam = rng.uniform(-1.0, 1.0, (n3, n2, n1))
    lam[-1] = 0.0
    lam[:, 0, :] = 0.0
    lam[:, -1, :] = 0.0
    lam[:, :, 0] = 0.0
    lam[:, :, -1] = 0.0
    return torch.as_tensor(lam, dtype=F64, device=device or prob.X.device)
