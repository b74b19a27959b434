"""GPU parity of the hybrid time step (hk_hybrid_step) against the oracle's
restatement (oracle/hk_oracle.c:hko_hybrid_step, itself pinned to the
single-layer steps by tests/test_hybrid_oracle.py): layer maps identical,
hydro states of layer-0 cells to 1e-12, kinetic distributions to 1e-10
relative L2 per cell, transition counts identical."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu


def _run_both(hk, oracle, nx, ny, n, a1, a2, band_layer, steps, params=None, state=None):
    import torch
    from paper_2505_03360_b200 import kinetic
    hydro, eps, r, f = state if state is not None else inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    if band_layer is not None:
        r = np.where(r != 0, band_layer, 0).astype(np.int8)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    ok = oracle.kernel(n, inputs.VMAX, a1, a2, inputs.R_PHYS_MAX)
    dx, dy = 1.0 / nx, 1.0 / ny
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
    p = params or kinetic.HybridParams()
    rd = torch.from_numpy(r).cuda()
    hd = torch.from_numpy(hydro).cuda()
    fd = torch.from_numpy(f).cuda()
    ed = torch.from_numpy(eps).cuda()
    ro, ho, fo = r, hydro, f
    for s in range(steps):
        r_before = ro
        cg = kinetic.hybrid_step(kern, nx, ny, dx, dy, dt, ed, rd, hd, fd, p)
        st, ro, ho, fo, co = oracle.hybrid_step(ok, nx, ny, dx, dy, dt, eps, ro, ho, fo, p)
        assert st == 0
        assert list(cg) == [int(c) for c in co], (s, cg, co)
        rg = rd.cpu().numpy()
        assert np.array_equal(rg, ro), s
        hg = hd.cpu().numpy()
        fl = ro == 0
        assert np.max(np.abs(hg[fl] - ho[fl]) / np.abs(ho[fl]).max(axis=1, keepdims=True)) < 1e-12, s
        fg = fd.cpu().numpy()
        for c in np.nonzero(ro != 0)[0]:
            e = np.linalg.norm(fg[c] - fo[c]) / np.linalg.norm(fo[c])
            assert e < 1e-10, (s, c, e)
        yield s, r_before, ro, cg


def test_hybrid_config4_shape_n16(hk, oracle):
    """Quadrant Riemann data, Boltzmann band, Algorithm 1 on: 2 steps with transitions."""
    seen = []
    for s, rb, ra, cg in _run_both(hk, oracle, 16, 12, 16, 4, 4, 2, 2):
        seen.append(cg)
    assert seen[0].layer2 > 0 and any(c.to_kinetic for c in seen)


def test_hybrid_esbgk_band_n32(hk, oracle):
    """N = 32 transport path, ES-BGK band (layer 1), Algorithm 1 on."""
    for _ in _run_both(hk, oracle, 10, 8, 32, 4, 4, 1, 1):
        pass


def test_hybrid_frozen_layers(hk, oracle):
    """update_regimes off: the given layer map is kept, all three layers present."""
    from paper_2505_03360_b200 import kinetic
    nx, ny, n = 12, 10, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    r = r.copy()
    r[(np.arange(nx * ny) % nx) < 3] = 1  # a layer-1 stripe next to the layer-2 band
    kin = (r != 0) & ~np.any(f != 0, axis=1)
    for c in np.nonzero(kin)[0]:
        rho = hydro[c, 0]
        T = hydro[c, 3] / (1.5 * rho)
        f[c] = inputs.maxwellian(n, rho, (0.0, 0.0, 0.0), T)
    for s, rb, ra, cg in _run_both(hk, oracle, nx, ny, n, 4, 4, None, 1,
                                   params=kinetic.HybridParams(update_regimes=False), state=(hydro, eps, r, f)):
        assert np.array_equal(rb, ra)


def test_hybrid_all_fluid_and_positivity(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    nx, ny, n = 8, 8, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1e-9)
    assert not np.any(r)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, 4, 4, inputs.R_PHYS_MAX)
    rd, hd, fd, ed = (torch.from_numpy(x).cuda() for x in (r, hydro, f, eps))
    cg = kinetic.hybrid_step(kern, nx, ny, 1 / nx, 1 / ny, 1e-3, ed, rd, hd, fd, kinetic.HybridParams())
    assert cg.layer0 == nx * ny and cg.layer1 + cg.layer2 == 0 and cg.halo_blocks == 0
    bad = hydro.copy()
    bad[37, 3] = -1.0  # negative pressure: moments_from_conserved throws positivity_error
    hd = torch.from_numpy(bad).cuda()
    with pytest.raises(hk.positivity_error):
        kinetic.hybrid_step(kern, nx, ny, 1 / nx, 1 / ny, 1e-3, ed, rd, hd, fd, kinetic.HybridParams())


def _hybrid_setup(hk, nx, ny, n):
    import torch
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, 4, 4, inputs.R_PHYS_MAX)
    dx, dy = 1.0 / nx, 1.0 / ny
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
    dev = [torch.from_numpy(x.copy()).cuda() for x in (r, hydro, f, eps)]
    return kern, dx, dy, dt, dev


def test_hybrid_slab_world1_equals_torus(hk):
    """x-slab hybrid step (8 ghost columns, local periodic torus) at world 1 == the torus step."""
    from paper_2505_03360_b200 import kinetic
    from paper_2505_03360_b200.partition import XSlab, hybrid_step_slab
    nx, ny, n = 20, 8, 16
    kern, dx, dy, dt, (r, h, f, e) = _hybrid_setup(hk, nx, ny, n)
    r2, h2, f2 = r.clone(), h.clone(), f.clone()
    part = XSlab(nx, ny, 1, 0)
    for _ in range(2):
        kinetic.hybrid_step(kern, nx, ny, dx, dy, dt, e, r, h, f)
        counts = hybrid_step_slab(part, kern, dx, dy, dt, e, r2, h2, f2)
        assert list(counts.long().tolist()) == [int((r == k).sum()) for k in range(3)]
        assert bool((r == r2).all())
        kin = r != 0
        assert float((h2 - h)[~kin].abs().max()) <= 1e-13 * float(h.abs().max())
        assert float((f2 - f)[kin].abs().max()) <= 1e-13 * float(f.abs().max())


def test_hybrid_slab_native_is_the_python_slab_step(hk):
    """hk_hybrid_step_slab (exchange / padding / counts in C++) at world 1 (the slab
    wraps onto itself) is bitwise partition.hybrid_step_slab's Python host logic."""
    import torch
    from paper_2505_03360_b200.partition import XSlab, hybrid_step_slab
    nx, ny, n = 20, 8, 16
    kern, dx, dy, dt, (r, h, f, e) = _hybrid_setup(hk, nx, ny, n)
    r2, h2, f2 = r.clone(), h.clone(), f.clone()
    part = XSlab(nx, ny, 1, 0)
    for _ in range(2):
        c1 = hybrid_step_slab(part, kern, dx, dy, dt, e, r, h, f)
        c2 = hybrid_step_slab(part, kern, dx, dy, dt, e, r2, h2, f2, native=True)
        assert torch.equal(c1, c2)
        assert torch.equal(r, r2) and torch.equal(h, h2) and torch.equal(f, f2)


def test_hybrid_slab_native_argument_checks(hk):
    """hk_hybrid_step_slab rejects a ghost width it cannot fill before touching the state."""
    import pytest
    from paper_2505_03360_b200 import kinetic
    nx, ny, n = 6, 4, 16
    kern, dx, dy, dt, (r, h, f, e) = _hybrid_setup(hk, nx, ny, n)
    before = [t.clone() for t in (r, h, f)]
    for ghost in (0, nx + 1):
        with pytest.raises(hk.contract_violation):
            kinetic.hybrid_step_slab_native(kern, nx, ny, dx, dy, dt, e, r, h, f, ghost=ghost)
    assert all(bool((a == b).all()) for a, b in zip(before, (r, h, f)))


def test_hybrid_two_slabs_equal_torus(hk):
    """Two x-slabs stepped in one process with exchanged 8-column halos reproduce the torus step."""
    import torch
    from paper_2505_03360_b200 import kinetic
    from paper_2505_03360_b200.partition import HYB_GHOST as W, XSlab, hybrid_step_slab
    nx, ny, n = 22, 6, 16
    kern, dx, dy, dt, (r, h, f, e) = _hybrid_setup(hk, nx, ny, n)
    parts = [XSlab(nx, ny, 2, k) for k in range(2)]
    loc = [[p.scatter(t.view(nx * ny, -1)) for t in (r, e, h, f)] for p in parts]
    for _ in range(2):
        halos = []
        for k, p in enumerate(parts):
            o = loc[1 - k]
            hk_ = []
            for fi in range(4):
                nb = o[fi].shape[-1]
                src = o[fi].view(ny, parts[1 - k].nxl, nb)
                hk_.append((src[:, -W:].contiguous(), src[:, :W].contiguous()))
            halos.append(hk_)
        for k, p in enumerate(parts):
            rl, el, hl, fl = loc[k]
            hybrid_step_slab(p, kern, dx, dy, dt, el.view(-1), rl.view(-1), hl, fl, halos=halos[k])
        kinetic.hybrid_step(kern, nx, ny, dx, dy, dt, e, r, h, f)
    glob = [torch.cat([loc[k][fi].view(ny, parts[k].nxl, -1) for k in range(2)], 1).reshape(nx * ny, -1)
            for fi in range(4)]
    assert bool((glob[0].view(-1) == r).all())
    kin = r != 0
    assert float((glob[2] - h)[~kin].abs().max()) <= 1e-13 * float(h.abs().max())
    assert float((glob[3] - f)[kin].abs().max()) <= 1e-13 * float(f.abs().max())


def test_hybrid_all_kinetic_algorithm1(hk, oracle):
    """Every cell kinetic at t = 0 (band layer 2, the rest layer 1): Algorithm 1 moves
    cells between layers 1 and 2 and down to 0; a 6 x 5 grid (stencils wrap twice)."""
    nx, ny, n = 6, 5, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    r = np.where(r != 0, 2, 1).astype(np.int8)
    for c in np.nonzero(r == 1)[0]:
        rho = hydro[c, 0]
        f[c] = inputs.maxwellian(n, rho, (0.0, 0.0, 0.0), hydro[c, 3] / (1.5 * rho))
    for s, rb, ra, cg in _run_both(hk, oracle, nx, ny, n, 4, 4, None, 2, state=(hydro, eps, r, f)):
        pass
