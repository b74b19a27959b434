"""GPU parity of the embedded-obstacle update (SURVEY §8f "next" #4):
classify_cells (src/grid.cpp:74-110) and apply_obstacle
(src/coupling.cpp:95-147) through the C-ABI against the C oracle, which
tests/test_oracle_vs_ref.py pins bitwise to the reference.  Bar: regimes,
kinds, hydro states and the moved spec bitwise; Maxwellian blocks to 1e-13
(device exp); blocks of covered cells untouched; the reference's exception
at the reference's cell."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu

VMAX = inputs.VMAX


def _pair(hk, om, shape, ci, cj, hi=0, hj=0, rad=0, mdi=0, mdj=0, pressure=0.9):
    from paper_2505_03360_b200 import kinetic
    args = dict(shape=shape, center_i=ci, center_j=cj, half_i=hi, half_j=hj, radius=rad, rho=1.3, pressure=pressure,
                ux=0.2, uy=-0.1, move_di=mdi, move_dj=mdj)
    o = om.Obstacle()
    for k, v in args.items():
        setattr(o, k, v)
    return kinetic.ObstacleSpec(**args), o


def test_classify_matches_oracle(hk):
    import oracle.oracle as om
    from paper_2505_03360_b200 import kinetic
    orc = om.Oracle()
    for nx, ny, sh in ((24, 20, (1, 10, 9, 2, 1)), (40, 36, (2, 20, 17, 0, 0, 6)), (30, 22, (0, 0, 0)),
                       (24, 24, (2, 14, 12, 0, 0, 4)), (24, 24, (1, 3, 12, 1, 1))):
        spec, ospec = _pair(hk, om, *sh)
        st, ko, bad = orc.classify_cells(nx, ny, ospec)
        if st == 0:
            k = kinetic.classify_cells(nx, ny, spec).cpu().numpy()
            assert np.array_equal(k, ko), sh
        else:
            with pytest.raises(hk.config_error, match="ghost frame"):
                kinetic.classify_cells(nx, ny, spec)
            assert bad >= 0


def _run(hk, orc, spec, ospec, nx, ny, n, steps, kind, r, hydro, f, has):
    import torch
    from paper_2505_03360_b200 import kinetic
    vg = hk.make_velocity_grid(n, VMAX)
    rd, kd = torch.from_numpy(r).cuda(), torch.from_numpy(kind).cuda()
    hd, fd = torch.from_numpy(hydro).cuda(), torch.from_numpy(f).cuda()
    ro, ko, ho, fo = r, kind, hydro, f
    for step in range(steps):
        st_o, ospec, ro, ko, ho, fo, co, vo = orc.apply_obstacle(nx, ny, n, VMAX, ospec, ro, ko, ho, fo)
        err = None
        try:
            res = kinetic.apply_obstacle(nx, ny, vg, spec, rd, kd, hd, fd)
        except hk.error as e:
            err = e
        assert (spec.center_i, spec.center_j) == (ospec.center_i, ospec.center_j)
        assert np.array_equal(rd.cpu().numpy(), ro), step
        assert np.array_equal(kd.cpu().numpy(), ko), step
        assert np.array_equal(hd.cpu().numpy(), ho), step
        fg = fd.cpu().numpy()
        gap, ref = np.linalg.norm(fg - fo, axis=1), np.linalg.norm(fo, axis=1)
        assert np.all(gap <= 1e-13 * ref), (step, np.flatnonzero(gap > 1e-13 * ref)[:5])
        if st_o:
            assert err is not None
            return st_o, err
        assert err is None, err
        assert (res.covered, res.vacated) == (co, vo), step
    return 0, None


def test_moving_disk_until_scenario_end(hk):
    import oracle.oracle as om
    orc = om.Oracle()
    n, nx, ny = 8, 24, 22
    spec, ospec = _pair(hk, om, 2, 9, 11, rad=2, mdi=1)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=12)
    st, err = _run(hk, orc, spec, ospec, nx, ny, n, 12, kind, r, hydro, f, has)
    assert st == 10 and isinstance(err, hk.scenario_end_error)


def test_diagonal_rectangle_n32(hk):
    import oracle.oracle as om
    orc = om.Oracle()
    n, nx, ny = 32, 26, 24
    spec, ospec = _pair(hk, om, 1, 9, 9, 2, 1, mdi=1, mdj=1)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=4)
    st, _ = _run(hk, orc, spec, ospec, nx, ny, n, 4, kind, r, hydro, f, has)
    assert st == 0


def test_static_overlap_is_config_error(hk):
    import oracle.oracle as om
    orc = om.Oracle()
    n, nx, ny = 8, 24, 22
    spec, ospec = _pair(hk, om, 1, 11, 10, 2, 1)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=1)
    assert _run(hk, orc, spec, ospec, nx, ny, n, 2, kind, r, hydro, f, has)[0] == 0
    spec.half_i = ospec.half_i = 6  # the ring now reaches the ghost frame
    st, err = _run(hk, orc, spec, ospec, nx, ny, n, 1, kind, r, hydro, f, has)
    assert st == 1 and isinstance(err, hk.config_error)


def test_ring_cell_positivity_error_midway(hk):
    """The reference throws at the first failing forced-ring cell; earlier cells
    are already updated, later ones untouched."""
    import oracle.oracle as om
    orc = om.Oracle()
    n, nx, ny = 8, 24, 22
    spec, ospec = _pair(hk, om, 1, 11, 10, 2, 1, mdi=1, mdj=1)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    nxt = ospec.copy(); nxt.center_i += 1; nxt.center_j += 1
    _, k2, _ = orc.classify_cells(nx, ny, nxt)
    bad = [int(np.flatnonzero((k2 == 2) & (kind == 0))[3])]
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=2, bad_cells=bad)
    r[bad] = 0; f[bad] = 0.0
    st, err = _run(hk, orc, spec, ospec, nx, ny, n, 2, kind, r, hydro, f, has)
    assert st == 8 and isinstance(err, hk.positivity_error)


def test_degenerate_fixed_state(hk):
    import oracle.oracle as om
    orc = om.Oracle()
    n, nx, ny = 8, 24, 22
    spec, ospec = _pair(hk, om, 1, 10, 10, 1, 1, mdi=1, pressure=-0.5)
    _, kind, _ = orc.classify_cells(nx, ny, ospec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=3)
    st, err = _run(hk, orc, spec, ospec, nx, ny, n, 1, kind, r, hydro, f, has)
    assert st == 3 and isinstance(err, hk.degenerate_state_error)


def test_no_obstacle_is_a_noop(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    spec = kinetic.ObstacleSpec(move_di=1)
    vg = hk.make_velocity_grid(8, VMAX)
    r = torch.zeros(100, dtype=torch.int8, device="cuda")
    k = kinetic.classify_cells(10, 10, spec)
    h = torch.ones((100, 4), dtype=torch.float64, device="cuda")
    f = torch.ones((100, 512), dtype=torch.float64, device="cuda")
    assert kinetic.apply_obstacle(10, 10, vg, spec, r, k, h, f) == (0, 0)
    assert spec.center_i == 0 and not r.any() and bool((f == 1).all())
