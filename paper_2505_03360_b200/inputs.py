"""Seeded synthetic inputs with the shapes of BASELINE.json's configs.

The reference ships no datasets or fixtures; every
config's input is analytic.  These generators are the single source of the
inputs used by the parity tests, the golden-vector script and bench.py.
Master seed 2505033601, per-config stream = master XOR config id
(SURVEY.md §8d "Synthetic inputs"); numpy PCG64 streams.
"""
from __future__ import annotations

import math

import numpy as np

MASTER_SEED = 2505033601
VMAX = 8.0
R_PHYS_MAX = 2.0 * VMAX / (3.0 + math.sqrt(2.0))  # aliasing bound, src/spectral.cpp:60


def rng_for(config_id: int, salt: int = 0) -> np.random.Generator:
    return np.random.default_rng(MASTER_SEED ^ config_id ^ (salt << 32))


def nodes(n: int, vmax: float = VMAX) -> np.ndarray:
    """Cell-centred velocity nodes v_k = -L + (k+1/2) dv (src/grid.cpp:18-33)."""
    dv = 2.0 * vmax / n
    return -vmax + (np.arange(n) + 0.5) * dv


def maxwellian(n: int, rho: float, u, T: float, vmax: float = VMAX) -> np.ndarray:
    v = nodes(n, vmax)
    ex = np.exp(-((v - u[0]) ** 2) / (2 * T))
    ey = np.exp(-((v - u[1]) ** 2) / (2 * T))
    ez = np.exp(-((v - u[2]) ** 2) / (2 * T))
    pref = rho / (2 * math.pi * T) ** 1.5
    return (pref * ex[:, None, None] * ey[None, :, None] * ez[None, None, :]).ravel()


def gaussian(n: int, rho: float, u, theta: np.ndarray, vmax: float = VMAX) -> np.ndarray:
    v = nodes(n, vmax)
    d = np.stack(np.meshgrid(v - u[0], v - u[1], v - u[2], indexing="ij"), axis=-1)
    inv = np.linalg.inv(theta)
    q = np.einsum("...i,ij,...j->...", d, inv, d)
    pref = rho / math.sqrt((2 * math.pi) ** 3 * np.linalg.det(theta))
    return (pref * np.exp(-0.5 * q)).ravel()


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def config1_cells(ncells: int = 64, n: int = 16, seed_salt: int = 0) -> np.ndarray:
    """Config 1: each cell a sum of two isotropic Maxwellians,
    rho~U(0.5,1.5), u~U(-1,1)^3, T~U(0.5,2)."""
    rng = rng_for(1, seed_salt)
    out = np.empty((ncells, n ** 3))
    for c in range(ncells):
        f = np.zeros(n ** 3)
        for _ in range(2):
            rho = rng.uniform(0.5, 1.5)
            u = rng.uniform(-1.0, 1.0, 3)
            T = rng.uniform(0.5, 2.0)
            f += maxwellian(n, rho, u, T)
        out[c] = f
    return out


def config2_cells(ncells: int = 4096, n: int = 32, seed_salt: int = 0) -> np.ndarray:
    """Config 2: 0.95 anisotropic Gaussian (rho~U(0.5,2), u~U(-.5,.5)^3,
    Theta = R diag(U(0.5,2)^3) R^T) + 0.05 bimodal Maxwellian pair."""
    rng = rng_for(2, seed_salt)
    out = np.empty((ncells, n ** 3))
    for c in range(ncells):
        rho = rng.uniform(0.5, 2.0)
        u = rng.uniform(-0.5, 0.5, 3)
        lam = rng.uniform(0.5, 2.0, 3)
        R = random_rotation(rng)
        theta = R @ np.diag(lam) @ R.T
        delta = rng.uniform(-1.0, 1.0, 3)
        tbar = np.trace(theta) / 3.0
        f = 0.95 * gaussian(n, rho, u, theta)
        f += 0.05 * 0.5 * (maxwellian(n, rho, u + delta, tbar) + maxwellian(n, rho, u - delta, tbar))
        out[c] = f
    return out


def config2_fast(ncells: int, n: int = 32, seed_salt: int = 0, distinct: int = 64) -> np.ndarray:
    """Config-2 shaped batch built from `distinct` seeded cells tiled to
    `ncells` (the bench's full 4096-cell batch without minutes of numpy
    set-up).  Cell c is distinct cell c % distinct, plus a per-cell seeded
    1e-3 relative amplitude scaling so no two cells are bitwise equal."""
    base = config2_cells(distinct, n, seed_salt)
    rng = rng_for(2, seed_salt + 1000)
    idx = np.arange(ncells) % distinct
    scale = 1.0 + 1e-3 * rng.uniform(-1.0, 1.0, ncells)
    return base[idx] * scale[:, None]


def config2_params(ncells: int, seed_salt: int = 0):
    """The per-cell parameter draws of config2_cells, in the same RNG order."""
    rng = rng_for(2, seed_salt)
    rho = np.empty(ncells); u = np.empty((ncells, 3)); theta = np.empty((ncells, 3, 3))
    delta = np.empty((ncells, 3))
    for c in range(ncells):
        rho[c] = rng.uniform(0.5, 2.0)
        u[c] = rng.uniform(-0.5, 0.5, 3)
        lam = rng.uniform(0.5, 2.0, 3)
        R = random_rotation(rng)
        theta[c] = R @ np.diag(lam) @ R.T
        delta[c] = rng.uniform(-1.0, 1.0, 3)
    return rho, u, theta, delta


def config2_cells_torch(ncells: int, n: int = 32, device="cuda", seed_salt: int = 0, chunk: int = 512):
    """config2_cells evaluated on the device (same draws, same formula), for
    the bench's full 4096-cell batch.  Returns a [ncells, n^3] float64 tensor."""
    import torch

    rho, u, theta, delta = config2_params(ncells, seed_salt)
    v = torch.as_tensor(nodes(n), dtype=torch.float64, device=device)
    V = torch.stack(torch.meshgrid(v, v, v, indexing="ij"), dim=-1).reshape(-1, 3)  # [n^3, 3]
    out = torch.empty((ncells, n ** 3), dtype=torch.float64, device=device)
    inv = torch.as_tensor(np.linalg.inv(theta), device=device)
    det = torch.as_tensor(np.linalg.det(theta), device=device)
    rho_t = torch.as_tensor(rho, device=device)
    u_t = torch.as_tensor(u, device=device)
    d_t = torch.as_tensor(delta, device=device)
    tbar = torch.as_tensor(np.trace(theta, axis1=1, axis2=2) / 3.0, device=device)
    for s in range(0, ncells, chunk):
        e = min(ncells, s + chunk)
        D = V[None, :, :] - u_t[s:e, None, :]
        q = torch.einsum("cki,cij,ckj->ck", D, inv[s:e], D)
        g = rho_t[s:e, None] / torch.sqrt((2 * math.pi) ** 3 * det[s:e, None]) * torch.exp(-0.5 * q)

        def mw(shift):
            W = V[None, :, :] - (u_t[s:e, None, :] + shift)
            T = tbar[s:e, None]
            return rho_t[s:e, None] / (2 * math.pi * T) ** 1.5 * torch.exp(-(W * W).sum(-1) / (2 * T))

        out[s:e] = 0.95 * g + 0.05 * 0.5 * (mw(d_t[s:e, None, :]) + mw(-d_t[s:e, None, :]))
    return out


def _hermite(k: int, x):
    """Probabilists' Hermite polynomials He_0..He_3."""
    if k == 0:
        return np.ones_like(x)
    if k == 1:
        return x
    if k == 2:
        return x * x - 1.0
    return x * x * x - 3.0 * x


HERMITE3 = [(a, b, 3 - a - b) for a in range(4) for b in range(4 - a)]  # the 10 (a,b,c), a+b+c=3


def config3_fields(nx: int, ny: int, seed_salt: int = 0):
    """Smooth seeded spatial fields of config 3 on a periodic [0,1)^2 grid:
    rho = 1 + 0.2 sin, T = 1 + 0.2 cos, u = (0.1 sin, 0.1 cos, 0), and
    eps_c in [0, 0.3] = rescaled sum of 4 random low-wavenumber sines."""
    rng = rng_for(3, seed_salt)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="xy")  # [ny, nx], cell c = j*nx + i
    ph = rng.uniform(0, 2 * np.pi, 4)
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X + ph[0]) * np.cos(2 * np.pi * Y + ph[1])
    T = 1.0 + 0.2 * np.cos(2 * np.pi * Y + ph[2]) * np.sin(2 * np.pi * X + ph[3])
    ux = 0.1 * np.sin(2 * np.pi * (X + Y) + ph[1])
    uy = 0.1 * np.cos(2 * np.pi * (X - Y) + ph[2])
    e = np.zeros_like(X)
    for _ in range(4):
        kx, ky = rng.integers(1, 4, 2)
        e += rng.uniform(0.5, 1.0) * np.sin(2 * np.pi * (kx * X + ky * Y) + rng.uniform(0, 2 * np.pi))
    e = 0.3 * (e - e.min()) / max(e.max() - e.min(), 1e-300)
    coef = rng.normal(size=len(HERMITE3))
    coef /= np.linalg.norm(coef)
    return dict(rho=rho.ravel(), T=T.ravel(), ux=ux.ravel(), uy=uy.ravel(), eps=e.ravel(), coef=coef)


def config3_cells(nx: int, ny: int, n: int = 32, seed_salt: int = 0, cells=None):
    """f = M(rho,u,T) (1 + eps_c P3(V)), V = (v-u)/sqrt(T), for the cells
    listed (default: all nx*ny).  Returns ([ncells, n^3], fields)."""
    fl = config3_fields(nx, ny, seed_salt)
    idx = np.arange(nx * ny) if cells is None else np.asarray(cells)
    v = nodes(n)
    out = np.empty((len(idx), n ** 3))
    for o, c in enumerate(idx):
        rho, T, ux, uy, ep = fl["rho"][c], fl["T"][c], fl["ux"][c], fl["uy"][c], fl["eps"][c]
        s = math.sqrt(T)
        Vx, Vy, Vz = (v - ux) / s, (v - uy) / s, v / s
        p3 = np.zeros((n, n, n))
        for (a, b, cc), w in zip(HERMITE3, fl["coef"]):
            p3 += w * _hermite(a, Vx)[:, None, None] * _hermite(b, Vy)[None, :, None] * _hermite(cc, Vz)[None, None, :]
        out[o] = maxwellian(n, rho, (ux, uy, 0.0), T) * (1.0 + ep * p3.ravel())
    return out, fl


def config3_cells_torch(nx: int, ny: int, n: int = 32, device="cuda", seed_salt: int = 0, chunk: int = 1024):
    """config3_cells evaluated on the device (same fields and formula)."""
    import torch

    fl = config3_fields(nx, ny, seed_salt)
    ncells = nx * ny
    v = torch.as_tensor(nodes(n), dtype=torch.float64, device=device)
    out = torch.empty((ncells, n ** 3), dtype=torch.float64, device=device)
    par = {k: torch.as_tensor(fl[k], dtype=torch.float64, device=device) for k in ("rho", "T", "ux", "uy", "eps")}
    coef = [float(c) for c in fl["coef"]]

    def he(k, x):
        if k == 0:
            return torch.ones_like(x)
        if k == 1:
            return x
        if k == 2:
            return x * x - 1.0
        return x * x * x - 3.0 * x

    for s in range(0, ncells, chunk):
        e = min(ncells, s + chunk)
        rho, T, ux, uy, ep = (par[k][s:e, None] for k in ("rho", "T", "ux", "uy", "eps"))
        sT = torch.sqrt(T)
        Vx, Vy, Vz = (v[None, :] - ux) / sT, (v[None, :] - uy) / sT, v[None, :] / sT  # [c, n]
        p3 = torch.zeros((e - s, n, n, n), dtype=torch.float64, device=device)
        for (a, b, c), w in zip(HERMITE3, coef):
            p3 += w * he(a, Vx)[:, :, None, None] * he(b, Vy)[:, None, :, None] * he(c, Vz)[:, None, None, :]
        ex = torch.exp(-(v[None, :] - ux) ** 2 / (2 * T))
        ey = torch.exp(-(v[None, :] - uy) ** 2 / (2 * T))
        ez = torch.exp(-(v[None, :]) ** 2 / (2 * T))
        M = (rho / (2 * math.pi * T) ** 1.5)[:, :, None, None] * ex[:, :, None, None] * ey[:, None, :, None] * ez[:, None, None, :]
        out[s:e] = (M * (1.0 + ep[:, :, None, None] * p3)).reshape(e - s, -1)
    return out, fl


# ---------------------------------------------------------------------------
# Config 5: 512 x 128 normal shock, N = 64, all cells Boltzmann.
# Upstream rho = 1, T = 1, u_x = 3 sqrt(5/3); Rankine-Hugoniot downstream for
# gamma = 5/3 (rho = 3, u_x = sqrt(5/3), T = 11/3).  The profile is the
# Mott-Smith bimodal form f = (1 - th) M_up + th M_down with
# th = (1 + tanh((x - 0.5) / (4 dx))) / 2, times (1 + 0.01 U(-1, 1)) density
# noise per cell: non-equilibrium inside the interface, Maxwellian outside.
# ---------------------------------------------------------------------------
C5_UP = (1.0, (3.0 * math.sqrt(5.0 / 3.0), 0.0, 0.0), 1.0)
C5_DOWN = (3.0, (math.sqrt(5.0 / 3.0), 0.0, 0.0), 11.0 / 3.0)


def config5_theta(nx: int = 512) -> np.ndarray:
    dx = 1.0 / nx
    x = (np.arange(nx) + 0.5) * dx
    return 0.5 * (1.0 + np.tanh((x - 0.5) / (4.0 * dx)))


def config5_cells(ncells: int, n: int = 64, nx: int = 512, ny: int = 128, seed_salt: int = 0,
                  columns=None) -> np.ndarray:
    """`ncells` cells of the config-5 field.  By default cell c sits in the
    (c mod 16)-th x-column nearest the interface (the non-equilibrium part of
    the shock); `columns` selects the x-columns explicitly (cycled)."""
    rng = rng_for(5, seed_salt)
    th = config5_theta(nx)
    if columns is None:
        columns = np.argsort(np.abs(np.arange(nx) + 0.5 - nx / 2), kind="stable")[:16]
    mu = maxwellian(n, *C5_UP)
    md = maxwellian(n, *C5_DOWN)
    out = np.empty((ncells, n ** 3))
    for c in range(ncells):
        i = columns[c % len(columns)]
        noise = 1.0 + 0.01 * rng.uniform(-1.0, 1.0)
        out[c] = noise * ((1.0 - th[i]) * mu + th[i] * md)
    return out


def config5_slab_torch(i0: int = 224, nxl: int = 64, ny: int = 128, n: int = 64, nx: int = 512, device="cuda",
                       seed_salt: int = 0):
    """The x-slab [ny][nxl][n^3] of the config-5 field starting at column i0
    (one GPU's share in the 8-GPU weak-scaling layout), built on the device:
    f = noise (1 - th) M_up + noise th M_down per cell."""
    import torch
    th = config5_theta(nx)[i0:i0 + nxl]
    rng = rng_for(5, seed_salt + 1)
    noise = 1.0 + 0.01 * rng.uniform(-1.0, 1.0, (ny, nxl))
    a = torch.from_numpy((noise * (1.0 - th)[None, :]).reshape(-1)).to(device)
    b = torch.from_numpy((noise * th[None, :]).reshape(-1)).to(device)
    mu = torch.from_numpy(maxwellian(n, *C5_UP)).to(device)
    md = torch.from_numpy(maxwellian(n, *C5_DOWN)).to(device)
    f = torch.empty((ny * nxl, n ** 3), dtype=torch.float64, device=device)
    for c0 in range(0, ny * nxl, 512):
        c1 = min(c0 + 512, ny * nxl)
        torch.addcmul(torch.outer(b[c0:c1], md), a[c0:c1, None], mu[None, :], out=f[c0:c1])
    return f


# ---------------------------------------------------------------------------
# Layer-0 states (config 4: quadrant Riemann problem), seeded.
# ---------------------------------------------------------------------------
def config4_conserved(nx: int = 200, ny: int = 200, xi: float = 5.0 / 3.0, seed_salt: int = 0,
                      smooth: bool = True) -> np.ndarray:
    """[nx*ny, 4] conserved (rho, rho ux, rho uy, E) of config 4's quadrants
    (rho {1, .125, .5, .25}, T {1, .8, 1, .5}, p = rho T, u = 0); with
    `smooth` the quadrant edges are tanh-smoothed over 2 cells and a 1 %
    seeded velocity perturbation is added (so every flux term is active)."""
    rng = rng_for(4, seed_salt)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y)  # [ny, nx]
    rq = np.array([1.0, 0.125, 0.5, 0.25])
    tq = np.array([1.0, 0.8, 1.0, 0.5])
    if smooth:
        w = 2.0 / nx
        sx = 0.5 * (1 + np.tanh((X - 0.5) / w))
        sy = 0.5 * (1 + np.tanh((Y - 0.5) / w))
    else:
        sx = (X > 0.5).astype(float)
        sy = (Y > 0.5).astype(float)
    wts = [(1 - sx) * (1 - sy), sx * (1 - sy), (1 - sx) * sy, sx * sy]
    rho = sum(wq * r for wq, r in zip(wts, rq))
    T = sum(wq * t for wq, t in zip(wts, tq))
    ux = 0.01 * rng.uniform(-1, 1, rho.shape)
    uy = 0.01 * rng.uniform(-1, 1, rho.shape)
    p = rho * T
    E = p / (xi - 1.0) + 0.5 * rho * (ux * ux + uy * uy)
    return np.stack([rho, rho * ux, rho * uy, E], -1).reshape(nx * ny, 4)


def obstacle_fields(kind: np.ndarray, n: int, seed_salt: int = 0, bad_cells=()):
    """Pre-update state around an embedded obstacle (src/coupling.cpp:95-147):
    given the previous classification `kind` (0 interior, 1 obstacle, 2 ring, 3 ghost),
    returns (r int8, hydro [cells,4], f [cells,n^3], has uint8).  Interior cells get
    a random regime in {0,1,2}; ring and obstacle cells are Layer 2; obstacle cells
    own no block (released); every cell with r != 0 owns one.  `bad_cells` get a
    negative pressure (the reference's moments_from_conserved throws there)."""
    rng = rng_for(6, seed_salt)
    cells = kind.size
    r = np.where(kind == 0, rng.integers(0, 3, cells), 0).astype(np.int8)
    r[(kind == 1) | (kind == 2)] = 2
    rho = rng.uniform(0.5, 2.0, cells)
    u = rng.uniform(-0.3, 0.3, (cells, 2))
    p = rng.uniform(0.5, 1.5, cells)
    p[list(bad_cells)] = -0.2
    hydro = np.empty((cells, 4))
    hydro[:, 0] = rho
    hydro[:, 1:3] = rho[:, None] * u
    hydro[:, 3] = p / (5.0 / 3.0 - 1.0) + 0.5 * rho * (u ** 2).sum(1)
    has = ((r != 0) & (kind != 1)).astype(np.uint8)
    f = np.where(has[:, None] != 0, rng.uniform(0.0, 1e-2, (cells, n ** 3)), 0.0)
    return r, hydro, f, has


def config4_band(nx: int, ny: int, half_width: float = 0.025) -> np.ndarray:
    """[nx*ny] bool: cells whose centre lies within half_width of an interface
    (x = 0.5, y = 0.5 and the periodic wrap x = 0, y = 0) of config 4's [0,1]^2."""
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    dxi = np.minimum(np.abs(x - 0.5), np.minimum(x, 1.0 - x))
    dyi = np.minimum(np.abs(y - 0.5), np.minimum(y, 1.0 - y))
    X, Y = np.meshgrid(dxi, dyi)
    return ((X < half_width) | (Y < half_width)).reshape(-1)


def config4_hybrid_state(nx: int = 200, ny: int = 200, n: int = 32, half_width: float = 0.025,
                         eps_fluid: float = 1e-3, eps_band: float = 1e-1, with_f: bool = True, seed_salt: int = 0):
    """Initial state of config 4's hybrid run: quadrant Riemann data at rest
    (tanh edges over 2 cells), Knudsen eps_fluid with eps_band on the interface
    band, the band starting in layer 2 (the rest in layer 0) with f = the
    Maxwellian of its hydro state.  Returns (hydro [cells,4], eps [cells],
    r int8 [cells], f [cells, n^3] or None); f is dense with zero blocks on layer 0."""
    hydro = config4_conserved(nx, ny, seed_salt=seed_salt, smooth=True)
    rho = hydro[:, 0]
    T = (2.0 / 3.0) * (hydro[:, 3] - 0.5 * (hydro[:, 1] ** 2 + hydro[:, 2] ** 2) / rho) / rho
    hydro[:, 1:3] = 0.0  # at rest (BASELINE config 4: zero velocity)
    hydro[:, 3] = 1.5 * rho * T
    band = config4_band(nx, ny, half_width)
    eps = np.where(band, eps_band, eps_fluid)
    r = np.where(band, 2, 0).astype(np.int8)
    f = None
    if with_f:
        f = np.zeros((nx * ny, n ** 3))
        for c in np.nonzero(band)[0]:
            f[c] = maxwellian(n, rho[c], (0.0, 0.0, 0.0), T[c])
    return hydro, eps, r, f
