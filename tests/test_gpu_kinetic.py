"""GPU parity of the per-cell kinetic operators, the classifier, the
transport sweep and the PR(2,2,2) steps against the oracle / golden
fixtures (the oracle is pinned to the reference's own code by
tests/test_oracle_vs_ref.py and tests/test_golden.py)."""
import os

import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu
VMAX = 8.0
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.fixture(scope="module")
def kin(hk):
    from paper_2505_03360_b200 import kinetic
    return kinetic


@pytest.fixture(scope="module")
def cells32():
    f, fl = inputs.config3_cells(8, 8, 32, cells=[0, 5, 17, 42])
    return f


@pytest.mark.parametrize("n", [16, 32])
def test_moments_realizability_l1(hk, kin, oracle, n, cells32):
    import torch
    f = cells32 if n == 32 else inputs.config3_cells(8, 8, 16, cells=[1, 2, 3])[0]
    vg = hk.make_velocity_grid(n, VMAX)
    out = kin.moments_of(torch.from_numpy(f).cuda(), vg, sigma=True, realizability=True, l1=True)
    mom = out["moments"].cpu().numpy()
    sig = out["sigma"].cpu().numpy()
    real = out["realizability"].cpu().numpy()
    l1 = out["l1"].cpu().numpy()
    for c in range(len(f)):
        st, m = oracle.moments(n, VMAX, f[c])
        assert np.allclose(mom[c], m, rtol=1e-12, atol=1e-15)
        s = oracle.second_moment(n, VMAX, f[c])
        assert np.allclose(sig[c], s[[0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]], rtol=1e-12, atol=1e-15)
        _, a, b, cc = oracle.realizability(n, VMAX, f[c])
        assert np.allclose(real[c], np.concatenate([a.ravel(), b, [cc]]), rtol=1e-11, atol=1e-13)
        assert abs(l1[c] - oracle.l1_distance(n, VMAX, f[c])[1]) < 1e-12


def test_degenerate_cell_raises(hk, kin):
    import torch
    vg = hk.make_velocity_grid(16, VMAX)
    f = torch.zeros((2, 16 ** 3), dtype=torch.float64, device="cuda")
    f[0] = torch.from_numpy(inputs.maxwellian(16, 1.0, (0, 0, 0), 1.0)).cuda()
    with pytest.raises(hk.degenerate_state_error):
        kin.moments_of(f, vg)
    out = kin.moments_of(f, vg, check=False)
    assert out["status"].cpu().tolist() == [0, 3]


def test_maxwellian(hk, kin, oracle):
    import torch
    vg = hk.make_velocity_grid(32, VMAX)
    mom = np.array([[1.2, 0.1, -0.2, 0.05, 0.9], [0.7, -0.3, 0.0, 0.2, 1.7]])
    got = kin.maxwellian(torch.from_numpy(mom).cuda(), vg).cpu().numpy()
    for c in range(2):
        assert rel(got[c], oracle.maxwellian(32, VMAX, tuple(mom[c]))[1]) < 1e-13


def test_esbgk_stage_golden(hk, kin):
    import torch
    g = np.load(os.path.join(GOLD, "esbgk_cfg3_n16.npz"))
    vg = hk.make_velocity_grid(int(g["n"]), float(g["vmax"]))
    p = kin.EsbgkParams(beta=float(g["beta"]), nu_coeff=float(g["nu_coeff"]))
    out, info = kin.esbgk_stage_solve(torch.from_numpy(g["f"]).cuda(), float(g["a"]), float(g["eps"]), p, vg)
    out = out.cpu().numpy()
    assert np.array_equal((info.cpu().numpy() >> 8) & 1, g["fallback"])
    for c in range(len(out)):
        assert rel(out[c], g["esbgk"][c]) < 1e-11


def test_esbgk_stage_n32_and_fallback(hk, kin, oracle, cells32):
    import torch
    vg = hk.make_velocity_grid(32, VMAX)
    eps = torch.tensor([1e-2, 1e-1, 1.0, 1e-3], dtype=torch.float64)
    out, info = kin.esbgk_stage_solve(torch.from_numpy(cells32).cuda(), 1e-3, eps, kin.EsbgkParams(), vg)
    out = out.cpu().numpy()
    for c in range(len(cells32)):
        ref, st, fb = oracle.esbgk_stage_solve(32, VMAX, cells32[c], 1e-3, float(eps[c]))
        assert rel(out[c], ref) < 1e-11
    # LLT fallback (src/moments.cpp:128-134)
    n = 16
    vg = hk.make_velocity_grid(n, VMAX)
    f = inputs.gaussian(n, 1.0, (0, 0, 0), np.diag([0.3, 2.0, 2.0]))
    ref, _, fb = oracle.esbgk_stage_solve(n, VMAX, f, 1e-6, 1e-2, beta=5.0)
    out, info = kin.esbgk_stage_solve(torch.from_numpy(f[None]).cuda(), 1e-6, 1e-2, kin.EsbgkParams(beta=5.0), vg)
    assert fb == 1 and int(info[0]) >> 8 == 1
    assert rel(out.cpu().numpy()[0], ref) < 1e-11


def test_penalized_stage(hk, kin, oracle, cells32):
    import torch
    vg = hk.make_velocity_grid(32, VMAX)
    a = (1 - 2 ** -0.5) * 1e-3
    out, _ = kin.penalized_stage_solve(torch.from_numpy(cells32).cuda(), a, 1e-2, kin.PenalizationRule(), vg)
    out = out.cpu().numpy()
    for c in range(len(cells32)):
        ref, st = oracle.penalized_stage_solve(32, VMAX, cells32[c], a, 1e-2)
        assert rel(out[c], ref) < 1e-11


def test_penalized_residual_golden(hk, kin):
    import torch
    g = np.load(os.path.join(GOLD, "collision_n16_cfg1.npz"))
    vg = hk.make_velocity_grid(int(g["n"]), float(g["vmax"]))
    k = hk.precompute_kernel(vg, int(g["n"]), int(g["a1"]), int(g["a2"]), float(g["r_phys"]))
    out = kin.penalized_residual(torch.from_numpy(g["f"]).cuda(), k, vg).cpu().numpy()
    for c in range(len(out)):
        assert rel(out[c], g["residual"][c]) < 1e-10


def test_transport_golden_and_oracle(hk, kin, oracle):
    import torch
    g = np.load(os.path.join(GOLD, "transport_n8.npz"))
    vg = hk.make_velocity_grid(int(g["n"]), float(g["vmax"]))
    out = kin.kinetic_transport_rhs_periodic(torch.from_numpy(g["f"]).cuda(), int(g["nx"]), int(g["ny"]), vg,
                                             float(g["dx"]), float(g["dy"])).cpu().numpy()
    assert rel(out, g["rhs"]) < 1e-13
    n, nx, ny = 16, 6, 5
    f, _ = inputs.config3_cells(nx, ny, n)
    vg = hk.make_velocity_grid(n, VMAX)
    got = kin.kinetic_transport_rhs_periodic(torch.from_numpy(f).cuda(), nx, ny, vg, 0.1, 0.2).cpu().numpy()
    assert rel(got, oracle.transport_rhs_periodic(f, nx, ny, n, VMAX, 0.1, 0.2)) < 1e-13
    # x-slab with halos == periodic result on the interior columns
    fx = f.reshape(ny, nx, -1)
    ext = np.concatenate([fx[:, -2:], fx, fx[:, :2]], axis=1).reshape(-1, n ** 3)
    got2 = kin.kinetic_transport_rhs_periodic(torch.from_numpy(np.ascontiguousarray(ext)).cuda(), nx, ny, vg, 0.1,
                                              0.2, x_halo=2).cpu().numpy()
    assert np.array_equal(got2, got)


def test_classify_matches_oracle(hk, kin, oracle):
    import torch
    n, nx, ny = 16, 8, 6
    f, fl = inputs.config3_cells(nx, ny, n)
    vg = hk.make_velocity_grid(n, VMAX)
    out = kin.moments_of(torch.from_numpy(f).cuda(), vg, l1=True)
    mom = out["moments"].cpu().numpy()
    eps = np.full(nx * ny, 1e-2)
    rng = np.random.default_rng(3)
    r_in = rng.integers(0, 3, nx * ny).astype(np.int8)
    th = kin.Thresholds(eta0=1e-3, eta1=1e-4, delta0=2e-2)
    r_out, ind, st = kin.classify(out["moments"], nx, ny, 1 / nx, 1 / ny, torch.from_numpy(eps), torch.from_numpy(r_in),
                                  th, l1=out["l1"])
    r_out, ind = r_out.cpu().numpy(), ind.cpu().numpy()
    prim = mom[:, [0, 1, 2, 4]]
    for c in range(nx * ny):
        i, j = c % nx, c // nx
        nb = lambda ii, jj: prim[(jj % ny) * nx + (ii % nx)]
        p5 = np.stack([prim[c], nb(i - 1, j), nb(i + 1, j), nb(i, j - 1), nb(i, j + 1)])
        _, lam, lb = oracle.indicators(p5, 1 / nx, 1 / ny, 1e-2)
        assert np.allclose(ind[c, :3], lam, rtol=1e-13) and np.isclose(ind[c, 3], lb, rtol=1e-12)
        st_o, r_o = oracle.regime_update(int(r_in[c]), lam, lb, float(out["l1"][c]), th.eta0, th.eta1, th.delta0)
        assert r_o == r_out[c], c
    assert len(set(r_out.tolist())) >= 2  # the thresholds exercise several branches


def test_esbgk_imex_step(hk, kin, oracle):
    import torch
    g = np.load(os.path.join(GOLD, "transport_n8.npz"))
    n, nx, ny = int(g["n"]), int(g["nx"]), int(g["ny"])
    vg = hk.make_velocity_grid(n, float(g["vmax"]))
    f = torch.from_numpy(g["f"].copy()).cuda()
    kin.esbgk_imex_step(f, nx, ny, vg, float(g["dx"]), float(g["dy"]), float(g["dt"]), torch.from_numpy(g["eps"]))
    assert rel(f.cpu().numpy(), g["esbgk_step"]) < 1e-11


def test_penalized_imex_step(hk, kin, oracle):
    import torch
    n, nx, ny = 16, 3, 3
    f, _ = inputs.config3_cells(nx, ny, n)
    eps = np.array([1e-2, 1e-1, 1.0] * 3)
    vg = hk.make_velocity_grid(n, VMAX)
    k = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX)
    ko = oracle.kernel(n, VMAX, 2, 4, inputs.R_PHYS_MAX, closed_form=False)
    ref, st = oracle.penalized_imex_step(ko, f, nx, ny, 0.1, 0.1, 1e-3, eps)
    ft = torch.from_numpy(f.copy()).cuda()
    kin.penalized_imex_step(ft, nx, ny, k, 0.1, 0.1, 1e-3, torch.from_numpy(eps))
    assert rel(ft.cpu().numpy(), ref) < 1e-10


def test_moment_operators_one_at_a_time(hk, kin, oracle, cells32):
    """anisotropic_gaussian / match_moments / remove_invariant_moments as
    stand-alone device operators (inc/moments.hpp:55-70) vs the oracle."""
    import torch
    n = 32
    vg = hk.make_velocity_grid(n, VMAX)
    f = cells32
    mom = np.array([oracle.moments(n, VMAX, f[c])[1] for c in range(len(f))])
    theta = np.array([oracle.stress_tensor(n, VMAX, f[c], mom[c]) for c in range(len(f))])
    # anisotropic Gaussian (beta = -1/2, the ES-BGK value), plus an LLT fallback cell
    th = theta.copy()
    th[2] = np.diag([10.0 * mom[2, 4], 1.0, 1.0])  # (1 - beta) T - beta theta_xx < 0: LLT fails
    g, fb = kin.anisotropic_gaussian(torch.from_numpy(mom).cuda(), torch.from_numpy(th).cuda(), -0.5, vg)
    g, fb = g.cpu().numpy(), fb.cpu().numpy()
    for c in range(len(f)):
        st, ref, rfb = oracle.anisotropic_gaussian(n, VMAX, tuple(mom[c]), th[c], -0.5)
        assert st == 0 and bool(rfb) == bool(fb[c]) and rel(g[c], ref) < 1e-12, c
    assert fb[2] and not fb[0]
    # match_moments of the Gaussians to the cells' own (rho, rho u, E)
    E = 0.5 * mom[:, 0] * (mom[:, 1:4] ** 2).sum(1) + 1.5 * mom[:, 0] * mom[:, 4]
    targets = np.concatenate([mom[:, :1], mom[:, :1] * mom[:, 1:4], E[:, None]], 1)
    gm = torch.from_numpy(g.copy()).cuda()
    kin.match_moments(gm, vg, torch.from_numpy(targets).cuda())
    gm = gm.cpu().numpy()
    for c in range(len(f)):
        st, ref = oracle.match_moments(n, VMAX, g[c], targets[c, 0], targets[c, 1:4], targets[c, 4])
        assert st == 0 and rel(gm[c], ref) < 1e-12, c
    # remove_invariant_moments of q = f - G~ with weight G~ and centre u
    q = f - gm
    qd = torch.from_numpy(q.copy()).cuda()
    kin.remove_invariant_moments(qd, torch.from_numpy(gm).cuda(), vg, torch.from_numpy(mom[:, 1:4].copy()).cuda())
    qd = qd.cpu().numpy()
    for c in range(len(f)):
        st, ref = oracle.remove_invariant_moments(n, VMAX, q[c], gm[c], mom[c, 1:4])
        assert st == 0
        assert np.abs(qd[c] - ref).max() <= 1e-12 * np.abs(q[c]).max(), c


def test_imex_steps_run_in_three_work_fields(hk, kin):
    """The regrouped PR(2,2,2) steps (n a power of two >= 8, ny >= 3) keep Y, f_acc and
    the residual only: a caller's work buffer of 3 fields gives the same step, bitwise,
    as the context-owned one (include/hykin_b200.h: hk_esbgk_imex_step)."""
    import torch
    n, nx, ny = 16, 4, 3
    vg = hk.make_velocity_grid(n, VMAX)
    f0, _ = inputs.config3_cells(nx, ny, n)
    eps = torch.full((nx * ny,), 1e-2, dtype=torch.float64, device="cuda")
    ctx = hk.default_context()
    P = kin.EsbgkParams()
    a = torch.from_numpy(f0.copy()).cuda()
    kin.esbgk_imex_step(a, nx, ny, vg, 0.1, 0.1, 1e-3, eps)
    b = torch.from_numpy(f0.copy()).cuda()
    work = torch.full((3, nx * ny, n ** 3), float("nan"), dtype=torch.float64, device="cuda")
    ctx.check(ctx._lib.hk_esbgk_imex_step(ctx.h, n, VMAX, b.data_ptr(), nx, ny, 0.1, 0.1, 1e-3, eps.data_ptr(),
                                          P.beta, P.nu_coeff, P.eps_weno, work.data_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    k = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX)
    c = torch.from_numpy(f0.copy()).cuda()
    kin.penalized_imex_step(c, nx, ny, k, 0.1, 0.1, 1e-3, eps)
    d = torch.from_numpy(f0.copy()).cuda()
    ctx.check(ctx._lib.hk_penalized_imex_step(ctx.h, k.h, d.data_ptr(), nx, ny, 0.1, 0.1, 1e-3, eps.data_ptr(),
                                              kin.PenalizationRule().coeff, 1e-6, 0, work.data_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(c, d)
