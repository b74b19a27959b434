"""GPU parity of the cross-layer stencil synthesis (SURVEY §8f "next" #1,
src/coupling.cpp:57-93) through the C-ABI against the C oracle, which
tests/test_oracle_vs_ref.py pins bitwise to the reference.  Bars: copied
blocks and obstacle / layer-0 conserved states bitwise; Maxwellian blocks
1e-13 (device exp); conserved states from kinetic moments 1e-13 relative
(moments_of's summation order differs)."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu

VMAX = inputs.VMAX


def _field(n=8, nx=20, ny=18, seed=5):
    import oracle.oracle as om
    from paper_2505_03360_b200 import kinetic
    orc = om.Oracle()
    args = dict(shape=2, center_i=9, center_j=9, radius=2, rho=1.3, pressure=0.9, ux=0.2, uy=-0.1)
    ospec = om.Obstacle()
    for k, v in args.items():
        setattr(ospec, k, v)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=seed)
    rng = np.random.default_rng(seed)
    for c in np.flatnonzero(has):
        f[c] = inputs.maxwellian(n, rng.uniform(0.5, 2), rng.uniform(-0.3, 0.3, 3), rng.uniform(0.6, 1.5))
    return orc, ospec, kinetic.ObstacleSpec(**args), kind, r, hydro, f


def _dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def test_hydro_synthesis_every_cell(hk):
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 8, 20, 18
    orc, ospec, spec, kind, r, hydro, f = _field(n, nx, ny)
    rd, kd, hd, fd = _dev(r, kind, hydro, f)
    vg = hk.make_velocity_grid(n, VMAX)
    got = kinetic.synthesize_hydro_state(nx, ny, vg, rd, kd, hd, fd, spec).cpu().numpy()
    cells = [(i, j) for j in range(ny) for i in range(nx)]
    st, ref = orc.synthesize(0, nx, ny, n, VMAX, ospec, r, kind, hydro, f, cells)
    assert st == 0
    src = np.array([min(max(j, 4), ny - 5) * nx + min(max(i, 4), nx - 5) for i, j in cells])
    exact = (kind[src] == 1) | (r[src] == 0)
    assert np.array_equal(got[exact], ref[exact])
    rel = np.abs(got[~exact] - ref[~exact]).max(axis=1) / np.abs(ref[~exact]).max(axis=1)
    assert (~exact).sum() > 50 and rel.max() < 1e-13


def test_distribution_synthesis_list(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 8, 20, 18
    orc, ospec, spec, kind, r, hydro, f = _field(n, nx, ny)
    rd, kd, hd, fd = _dev(r, kind, hydro, f)
    vg = hk.make_velocity_grid(n, VMAX)
    cells = np.random.default_rng(1).permutation(nx * ny)[:150]
    got = kinetic.synthesize_distribution(nx, ny, vg, rd, kd, hd, fd, torch.from_numpy(cells), spec).cpu().numpy()
    st, ref = orc.synthesize(1, nx, ny, n, VMAX, ospec, r, kind, hydro, f, [(c % nx, c // nx) for c in cells])
    assert st == 0
    gap = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert gap.max() < 1e-13
    src = np.array([min(max(c // nx, 4), ny - 5) * nx + min(max(c % nx, 4), nx - 5) for c in cells])
    copied = (kind[src] != 1) & (r[src] != 0)
    assert copied.sum() > 10 and np.array_equal(got[copied], ref[copied])


def test_distribution_halo_fill_in_place(hk):
    """Stencil mode: exactly the non-kinetic cells on a kinetic cell's +-2 cross
    receive the synthesized block; every other block is untouched."""
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 8, 20, 18
    orc, ospec, spec, kind, r, hydro, f = _field(n, nx, ny)
    r = r.copy()
    r[(np.arange(nx * ny) % nx) < 9] = 0  # left half layer 0: a layer interface
    f = np.where((r != 0)[:, None] & (kind != 1)[:, None], f, -7.0)
    rd, kd, hd, fd = _dev(r, kind, hydro, f)
    vg = hk.make_velocity_grid(n, VMAX)
    filled = kinetic.synthesize_distribution(nx, ny, vg, rd, kd, hd, fd, None, spec)
    got = fd.cpu().numpy()

    def kin(i, j):
        c = j * nx + i
        return 4 <= i < nx - 4 and 4 <= j < ny - 4 and kind[c] != 1 and r[c] != 0

    want = []
    for j in range(ny):
        for i in range(nx):
            if kin(i, j):
                continue
            near = any(0 <= i + d < nx and kin(i + d, j) for d in (-2, -1, 1, 2)) or \
                any(0 <= j + d < ny and kin(i, j + d) for d in (-2, -1, 1, 2))
            if near:
                want.append((i, j))
    assert filled == len(want) > 20
    st, ref = orc.synthesize(1, nx, ny, n, VMAX, ospec, r, kind, hydro, f, want)
    assert st == 0
    idx = np.array([j * nx + i for i, j in want])
    gap = np.linalg.norm(got[idx] - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert gap.max() < 1e-13
    untouched = np.setdiff1d(np.arange(nx * ny), idx)
    assert np.array_equal(got[untouched], f[untouched])


def test_synthesis_errors(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 8, 20, 18
    orc, ospec, spec, kind, r, hydro, f = _field(n, nx, ny)
    c0 = int(np.flatnonzero((r == 0) & (kind == 0))[0])
    hydro = hydro.copy(); hydro[c0, 3] = -1.0
    rd, kd, hd, fd = _dev(r, kind, hydro, f)
    vg = hk.make_velocity_grid(n, VMAX)
    with pytest.raises(hk.positivity_error):
        kinetic.synthesize_distribution(nx, ny, vg, rd, kd, hd, fd, torch.tensor([0, c0]), spec)
    c1 = int(np.flatnonzero((r != 0) & (kind == 0))[0])
    f = f.copy(); f[c1] = -f[c1]
    rd, kd, hd, fd = _dev(r, kind, hydro, f)
    with pytest.raises(hk.degenerate_state_error):
        kinetic.synthesize_hydro_state(nx, ny, vg, rd, kd, hd, fd, spec)
    with pytest.raises(hk.config_error):  # no interior inside the ghost frame
        kinetic.synthesize_hydro_state(8, 8, vg, rd[:64], kd[:64], hd[:64], fd[:64], spec)
