"""Pins the C restatement (oracle/hk_oracle.c) to the reference's own
sources compiled here (oracle/_ref: unmodified src/*.cpp + FFTW/Eigen API
shims).  CPU only; skipped where _ref was not built."""
import math

import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

VMAX = 8.0


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.fixture(scope="module")
def k16(oracle, reflib):
    ko = oracle.kernel(16, VMAX, 2, 4, inputs.R_PHYS_MAX, closed_form=False)
    kr = reflib.kernel(16, VMAX, 2, 4, inputs.R_PHYS_MAX)
    return ko, kr


def test_precompute_tables_bitwise(k16):
    ko, kr = k16
    a, ap, ld, sc = kr.tables()
    assert np.array_equal(a, ko.alpha) and np.array_equal(ap, ko.alpha_prime)
    assert np.array_equal(ld, ko.loss_diag)
    assert sc[0] == ko.r and sc[1] == ko.jacobian and sc[2] == ko.weight


def test_closed_form_weights_match_quadrature(oracle, k16):
    ko, _ = k16
    kc = oracle.kernel(16, VMAX, 2, 4, inputs.R_PHYS_MAX, closed_form=True)
    assert rel(kc.alpha, ko.alpha) < 1e-13 and rel(kc.alpha_prime, ko.alpha_prime) < 1e-13


def test_collision_bitwise_and_throw_verdict(oracle, reflib, k16):
    ko, kr = k16
    f = inputs.config1_cells(3, 16)
    qo, so, _ = oracle.collision_batch(ko, f)
    qr, sr = reflib.collision_batch(kr, f)
    assert np.array_equal(qo, qr)
    assert np.array_equal(so, sr)  # both report the reference's numerical_consistency_error


def test_precompute_errors(oracle, reflib):
    for lib in (oracle, reflib):
        assert lib.kernel(16, VMAX, 2, 2, inputs.R_PHYS_MAX * 1.01).status == 2  # aliasing
        assert lib.kernel(16, VMAX, 0, 2, 1.0).status == 1                      # config
        assert lib.kernel(16, VMAX, 2, 2, 0.0).status == 1


def _cells3(n=8, nc=3):
    f, _ = inputs.config3_cells(4, 4, n, cells=list(range(nc)))
    return f


def test_moments_family(oracle, reflib):
    n = 8
    for f in _cells3(n):
        so, mo = oracle.moments(n, VMAX, f)
        sr, mr = reflib.moments(n, VMAX, f)
        assert so == sr == 0 and np.allclose(mo, mr, rtol=1e-14, atol=1e-16)
        assert np.allclose(oracle.second_moment(n, VMAX, f), reflib.second_moment(n, VMAX, f), rtol=1e-14, atol=1e-16)
        _, ao, bo, co = oracle.realizability(n, VMAX, f)
        _, ar, br, cr = reflib.realizability(n, VMAX, f)
        assert np.allclose(ao, ar, atol=1e-14) and np.allclose(bo, br, atol=1e-14) and abs(co - cr) < 1e-14
        _, Mo = oracle.maxwellian(n, VMAX, mo)
        _, Mr = reflib.maxwellian(n, VMAX, mr)
        assert rel(Mo, Mr) < 1e-14
        mom = np.array(mo[1:4]) * mo[0]
        E = 0.5 * mo[0] * sum(x * x for x in mo[1:4]) + 1.5 * mo[0] * mo[4]
        _, go = oracle.match_moments(n, VMAX, Mo, mo[0], mom, E)
        _, gr = reflib.match_moments(n, VMAX, Mr, mr[0], mom, E)
        assert rel(go, gr) < 1e-13
        assert abs(oracle.l1_distance(n, VMAX, f)[1] - reflib.l1_distance(n, VMAX, f)[1]) < 1e-13


def test_degenerate_moments(oracle, reflib):
    z = np.zeros(8 ** 3)
    assert oracle.moments(8, VMAX, z)[0] == 3 and reflib.moments(8, VMAX, z)[0] == 3


def test_stage_solves(oracle, reflib):
    n = 8
    for f in _cells3(n):
        po, s1 = oracle.penalized_stage_solve(n, VMAX, f, 0.3 * 1e-3, 1e-2)
        pr, s2 = reflib.penalized_stage_solve(n, VMAX, f, 0.3 * 1e-3, 1e-2)
        assert s1 == s2 == 0 and rel(po, pr) < 1e-13
        eo, s1, fbo = oracle.esbgk_stage_solve(n, VMAX, f, 1e-3, 1e-2)
        er, s2, fbr = reflib.esbgk_stage_solve(n, VMAX, f, 1e-3, 1e-2)
        assert s1 == s2 == 0 and fbo == fbr and rel(eo, er) < 1e-13


def test_esbgk_llt_fallback(oracle, reflib):
    """beta = 5 with a weak relaxation makes Tc = -4 T I + 5 Theta indefinite for
    a strongly anisotropic cell: both sides fall back to the Maxwellian
    (src/moments.cpp:128-134)."""
    n = 8
    th = np.diag([0.2, 2.0, 2.0])
    f = inputs.gaussian(n, 1.0, (0, 0, 0), th)
    eo, _, fbo = oracle.esbgk_stage_solve(n, VMAX, f, 1e-6, 1e-2, beta=5.0)
    er, _, fbr = reflib.esbgk_stage_solve(n, VMAX, f, 1e-6, 1e-2, beta=5.0)
    assert fbo == fbr == 1 and rel(eo, er) < 1e-13


def test_indicators_and_regime_truth_table(oracle, reflib):
    rng = np.random.default_rng(7)
    for _ in range(50):
        prim = np.column_stack([rng.uniform(0.5, 2, 5), rng.uniform(-0.3, 0.3, 5), rng.uniform(-0.3, 0.3, 5),
                                rng.uniform(0.5, 2, 5)])
        _, lo, bo = oracle.indicators(prim, 0.01, 0.01, 1e-2)
        lr, br = reflib.indicators(prim, 0.01, 0.01, 1e-2)
        assert np.allclose(lo, lr, rtol=1e-14) and math.isclose(bo, br, rel_tol=1e-14)
    # Algorithm 1 (src/regime.cpp:25-52): every branch incl. contract violations
    lam_near, lam_far = [1.0, 1.0, 1.0], [1.0, 1.5, 1.0]
    for r in (0, 1, 2, 3):
        for lam in (None, lam_near, lam_far):
            for lb in (None, 0.0, 1.0):
                for l1 in (None, 0.0, 1.0):
                    a = oracle.regime_update(r, lam, lb, l1, 1e-3, 1e-2, 1e-3)
                    b = reflib.regime_update(r, lam, lb, l1, 1e-3, 1e-2, 1e-3)
                    assert a[0] == b[0] and (a[0] != 0 or a[1] == b[1]), (r, lam, lb, l1, a, b)


def test_transport_periodic(oracle, reflib):
    n, nx, ny = 8, 5, 4
    f, _ = inputs.config3_cells(nx, ny, n)
    to = oracle.transport_rhs_periodic(f, nx, ny, n, VMAX, 0.1, 0.1)
    tr = reflib.transport_rhs_periodic(f, nx, ny, n, VMAX, 0.1, 0.1)
    assert np.array_equal(to, tr)
    assert abs(to.sum()) < 1e-12 * np.abs(to).sum()  # globally conservative


def test_penalized_residual(oracle, reflib, k16):
    ko, kr = k16
    f = inputs.config1_cells(2, 16)
    for c in range(2):
        ro, so, _ = oracle.penalized_residual(ko, f[c])
        rr, sr = reflib.penalized_residual_batch(kr, f[c:c + 1])
        assert so == sr[0] and rel(ro, rr[0]) < 1e-13


def test_imex_steps(oracle, reflib):
    n, nx, ny = 8, 4, 3
    f, fl = inputs.config3_cells(nx, ny, n)
    eps = np.full(nx * ny, 1e-2)
    a, sa = oracle.esbgk_imex_step(f, nx, ny, n, VMAX, 0.1, 0.1, 1e-3, eps)
    b, sb = reflib.esbgk_imex_step(f, nx, ny, n, VMAX, 0.1, 0.1, 1e-3, eps)
    assert sa == sb == 0 and rel(a, b) < 1e-13
    ko = oracle.kernel(n, VMAX, 2, 2, 2.0, closed_form=False)
    kr = reflib.kernel(n, VMAX, 2, 2, 2.0)
    a, sa = oracle.penalized_imex_step(ko, f, nx, ny, 0.1, 0.1, 1e-3, eps)
    b, sb = reflib.penalized_imex_step(kr, f, nx, ny, 0.1, 0.1, 1e-3, eps)
    assert sa == sb and rel(a, b) < 1e-13


def test_euler_layer_bitwise(oracle, reflib):
    """Layer-0 Euler residual and TVD-RK2 step (src/euler.cpp:159-181): the C
    restatement equals the reference bitwise; positivity failures agree."""
    nx, ny = 24, 20
    u = inputs.config4_conserved(nx, ny)
    st_o, r_o, _ = oracle.euler_rhs_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny)
    st_r, r_r = reflib.euler_rhs_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny)
    assert st_o == st_r == 0 and np.array_equal(r_o, r_r)
    st_o, u_o = oracle.tvd_rk2_step_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny, 2e-3)
    st_r, u_r = reflib.tvd_rk2_step_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny, 2e-3)
    assert st_o == st_r == 0 and np.array_equal(u_o, u_r)
    bad = u.copy()
    bad[37, 3] = 0.0  # negative pressure
    assert oracle.euler_rhs_periodic(bad, nx, ny, 0.1, 0.1)[0] == reflib.euler_rhs_periodic(bad, nx, ny, 0.1, 0.1)[0] == 8


def test_transitions_bitwise(oracle, reflib):
    """moments_from_conserved / conserved_from_moments (src/coupling.cpp:7-22)."""
    u = inputs.config4_conserved(6, 5)
    for c in range(len(u)):
        so, mo = oracle.moments_from_conserved(u[c])
        sr, mr = reflib.moments_from_conserved(u[c])
        assert so == sr == 0 and np.array_equal(mo, mr)
        assert np.array_equal(oracle.conserved_from_moments(mo), reflib.conserved_from_moments(mr))
    assert oracle.moments_from_conserved([-1.0, 0, 0, 1.0])[0] == reflib.moments_from_conserved([-1.0, 0, 0, 1.0])[0] == 8


def _spec(oracle_mod, shape, ci, cj, hi=0, hj=0, rad=0, mdi=0, mdj=0):
    s = oracle_mod.Obstacle()
    s.shape, s.center_i, s.center_j, s.half_i, s.half_j, s.radius = shape, ci, cj, hi, hj, rad
    s.rho, s.pressure, s.ux, s.uy, s.move_di, s.move_dj = 1.3, 0.9, 0.2, -0.1, mdi, mdj
    return s


def test_obstacle_classify_bitwise(oracle, reflib):
    """classify_cells (src/grid.cpp:74-110): ghost frame, footprint, 2-cell ring,
    and the config_error when either touches the ghost frame."""
    import oracle.oracle as om
    for nx, ny, spec in ((24, 20, _spec(om, 1, 10, 9, 2, 1)), (24, 24, _spec(om, 2, 12, 12, rad=3)),
                         (30, 22, _spec(om, 0, 0, 0)), (24, 24, _spec(om, 2, 14, 12, rad=4)),
                         (24, 24, _spec(om, 1, 7, 12, 0, 0)), (24, 24, _spec(om, 1, 3, 12, 1, 1))):
        st_o, k_o, bad = oracle.classify_cells(nx, ny, spec)
        st_r, k_r = reflib.classify_cells(nx, ny, spec)
        assert st_o == st_r, (spec.center_i, spec.radius)
        if st_o == 0:
            assert np.array_equal(k_o, k_r)
        else:
            assert st_o == 1 and bad >= 0


def test_obstacle_apply_bitwise(oracle, reflib):
    """apply_obstacle (src/coupling.cpp:95-147) over a moving disk until it leaves
    the domain (scenario_end_error), a static rectangle, and a forced-ring cell
    whose state throws mid-loop: r, kind, hydro, the surviving blocks, the
    moved spec and the covered/vacated counts all bitwise."""
    import oracle.oracle as om
    n, nx, ny = 8, 24, 22
    cases = [(_spec(om, 2, 9, 11, rad=2, mdi=1, mdj=0), 12, ()), (_spec(om, 1, 11, 10, 2, 1), 1, ()),
             (_spec(om, 1, 11, 10, 2, 1, mdi=1, mdj=1), 2, None)]
    for spec, steps, bad in cases:
        _, kind, _ = oracle.classify_cells(nx, ny, spec)
        if bad is None:  # an interior r=0 cell of the next ring with a negative pressure
            nxt = spec.copy(); nxt.center_i += 1; nxt.center_j += 1
            _, k2, _ = oracle.classify_cells(nx, ny, nxt)
            bad = [int(np.flatnonzero((k2 == 2) & (kind == 0))[3])]
        r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=steps, bad_cells=bad)
        if bad:
            r[bad] = 0; has[bad] = 0; f[bad] = 0.0
        so = sr = spec
        ko = kr = kind
        ro, rr, ho, hr, fo, fr, hs = r, r, hydro, hydro, f, f, has
        for step in range(steps):
            st_o, so, ro, ko, ho, fo, co, vo = oracle.apply_obstacle(nx, ny, n, VMAX, so, ro, ko, ho, fo)
            st_r, sr, rr, kr, hr, fr, hs, cr, vr = reflib.apply_obstacle(nx, ny, n, VMAX, sr, rr, kr, hr, fr, hs)
            assert st_o == st_r, step
            assert (so.center_i, so.center_j) == (sr.center_i, sr.center_j)
            assert np.array_equal(ro, rr) and np.array_equal(ko, kr) and np.array_equal(ho, hr)
            live = hs != 0
            assert np.array_equal(fo[live], fr[live])
            if st_o:
                break
            assert (co, vo) == (cr, vr)
        else:
            assert not (spec.move_di or spec.move_dj), "moving obstacle should have hit the ghost frame"
        if spec.move_di and bad == ():
            assert st_o == 10
        if bad:
            assert st_o == 8  # positivity_error from moments_from_conserved


def test_obstacle_degenerate_fixed_state(oracle, reflib):
    """A moving obstacle whose fixed state has T <= 0: maxwellian throws
    degenerate_state_error at the first vacated cell, after its r and hydro
    were overwritten (src/coupling.cpp:130-136)."""
    import oracle.oracle as om
    n, nx, ny = 8, 24, 22
    spec = _spec(om, 1, 10, 10, 1, 1, mdi=1)
    spec.pressure = -0.5
    _, kind, _ = oracle.classify_cells(nx, ny, spec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=3)
    st_o, so, ro, ko, ho, fo, _, _ = oracle.apply_obstacle(nx, ny, n, VMAX, spec, r, kind, hydro, f)
    st_r, sr, rr, kr, hr, fr, hs, _, _ = reflib.apply_obstacle(nx, ny, n, VMAX, spec, r, kind, hydro, f, has)
    assert st_o == st_r == 3
    assert np.array_equal(ro, rr) and np.array_equal(ko, kr) and np.array_equal(ho, hr)
    live = (hs != 0) & (has != 0)  # the failing vacated cell had no block before (ensure() made one)
    assert np.array_equal(fo[live], fr[live])


def _synth_state(oracle, om, nx=20, ny=18, n=8, seed=5, bad=()):
    """A mixed field: ghost frame, an obstacle with its ring, random regimes."""
    spec = _spec(om, 2, 9, 9, rad=2)
    _, kind, _ = oracle.classify_cells(nx, ny, spec)
    r, hydro, f, has = inputs.obstacle_fields(kind, n, seed_salt=seed, bad_cells=bad)
    # kinetic blocks with a physical moment structure (moments_of must succeed)
    rng = np.random.default_rng(seed)
    for c in np.flatnonzero(has):
        f[c] = inputs.maxwellian(n, rng.uniform(0.5, 2), rng.uniform(-0.3, 0.3, 3), rng.uniform(0.6, 1.5))
    cells = [(i, j) for j in range(ny) for i in range(nx)]
    return spec, kind, r, hydro, f, has, cells


def test_stencil_synthesis_bitwise(oracle, reflib):
    """synthesize_hydro_state / synthesize_distribution (src/coupling.cpp:57-93)
    at every cell of a mixed field, ghost frame included."""
    import oracle.oracle as om
    nx, ny, n = 20, 18, 8
    spec, kind, r, hydro, f, has, cells = _synth_state(oracle, om, nx, ny, n)
    for which in (0, 1):
        st_o, out_o = oracle.synthesize(which, nx, ny, n, VMAX, spec, r, kind, hydro, f, cells)
        st_r, out_r = reflib.synthesize(which, nx, ny, n, VMAX, spec, r, kind, hydro, f, has, cells)
        assert st_o == st_r == 0
        assert np.array_equal(out_o, out_r), which


def test_stencil_synthesis_errors(oracle, reflib):
    """A layer-0 cell with negative pressure: positivity_error from the
    distribution synthesis; a kinetic block with rho <= 0: degenerate_state_error
    from the hydro synthesis."""
    import oracle.oracle as om
    nx, ny, n = 20, 18, 8
    spec, kind, r, hydro, f, has, cells = _synth_state(oracle, om, nx, ny, n)
    c0 = int(np.flatnonzero((r == 0) & (kind == 0))[0])
    hydro = hydro.copy(); hydro[c0, 3] = -1.0
    ij = [(c0 % nx, c0 // nx)]
    assert oracle.synthesize(1, nx, ny, n, VMAX, spec, r, kind, hydro, f, ij)[0] == 8
    assert reflib.synthesize(1, nx, ny, n, VMAX, spec, r, kind, hydro, f, has, ij)[0] == 8
    c1 = int(np.flatnonzero((r != 0) & (kind == 0))[0])
    f = f.copy(); f[c1] = -f[c1]
    ij = [(c1 % nx, c1 // nx)]
    assert oracle.synthesize(0, nx, ny, n, VMAX, spec, r, kind, hydro, f, ij)[0] == 3
    assert reflib.synthesize(0, nx, ny, n, VMAX, spec, r, kind, hydro, f, has, ij)[0] == 3
