"""Layer-0 Euler solver and layer transitions on the device (hk_euler.cu)
against the CPU oracle, which is pinned bitwise to the reference
(tests/test_oracle_vs_ref.py::test_euler_layer_bitwise).  The kernels keep the
reference's statement order without FMA contraction: bitwise parity."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu


def test_euler_rhs_and_step_bitwise(hk, oracle):
    import torch
    from paper_2505_03360_b200 import kinetic
    nx, ny = 40, 36
    u = inputs.config4_conserved(nx, ny)
    ud = torch.from_numpy(u).cuda()
    rhs = kinetic.euler_rhs_periodic(ud, nx, ny, 1.0 / nx, 1.0 / ny).cpu().numpy()
    st, ref, _ = oracle.euler_rhs_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny)
    assert st == 0 and np.array_equal(rhs, ref)
    for _ in range(3):
        kinetic.tvd_rk2_step_periodic(ud, nx, ny, 1.0 / nx, 1.0 / ny, 1e-3)
        st, u = oracle.tvd_rk2_step_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny, 1e-3)
        assert st == 0
    assert np.array_equal(ud.cpu().numpy(), u)


def test_euler_conserves_totals(hk):
    """Periodic finite volumes: mass, momentum and energy totals are constant."""
    import torch
    from paper_2505_03360_b200 import kinetic
    nx = ny = 64
    ud = torch.from_numpy(inputs.config4_conserved(nx, ny)).cuda()
    tot0 = ud.sum(0).cpu().numpy()
    for _ in range(5):
        kinetic.tvd_rk2_step_periodic(ud, nx, ny, 1.0 / nx, 1.0 / ny, 5e-4)
    tot1 = ud.sum(0).cpu().numpy()
    assert np.allclose(tot1, tot0, rtol=0, atol=1e-12 * np.abs(tot0).max())


def test_euler_positivity_error(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    nx, ny = 8, 8
    u = inputs.config4_conserved(nx, ny)
    u[19, 3] = 0.0  # E = 0: negative pressure
    ud = torch.from_numpy(u).cuda()
    with pytest.raises(hk.positivity_error):
        kinetic.euler_rhs_periodic(ud, nx, ny, 0.1, 0.1)
    before = ud.clone()
    with pytest.raises(hk.positivity_error):
        kinetic.tvd_rk2_step_periodic(ud, nx, ny, 0.1, 0.1, 1e-3)
    assert torch.equal(ud, before)  # the reference throws before updating


def test_transitions_roundtrip_and_oracle(hk, oracle):
    """0 -> 1 (Maxwellian of the hydro state) then 1 -> 0 (hydro state of its
    moments): each step equals the oracle; the round trip returns the state up
    to the velocity-grid quadrature of the Maxwellian."""
    import torch
    from paper_2505_03360_b200 import kinetic
    n = 32
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    u = inputs.config4_conserved(4, 3)
    f = kinetic.conserved_to_maxwellian(torch.from_numpy(u).cuda(), vg).cpu().numpy()
    for c in range(len(u)):
        st, m = oracle.moments_from_conserved(u[c])
        assert st == 0
        _, fo = oracle.maxwellian(n, inputs.VMAX, tuple(m))
        assert np.linalg.norm(f[c] - fo) <= 1e-13 * np.linalg.norm(fo)
    back = kinetic.distribution_to_conserved(torch.from_numpy(f).cuda(), vg).cpu().numpy()
    for c in range(len(u)):
        _, mo = oracle.moments(n, inputs.VMAX, f[c])
        uo = oracle.conserved_from_moments(np.array(mo))
        np.testing.assert_allclose(back[c], uo, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(back[c], u[c], rtol=1e-6, atol=1e-8)


def test_gather_scatter_cells(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    src = torch.randn(10, 64, dtype=torch.float64, device="cuda")
    idx = torch.tensor([7, 2, 9, 2], device="cuda")
    g = kinetic.gather_cells(src, idx)
    assert torch.equal(g, src[idx])
    dst = torch.zeros_like(src)
    kinetic.scatter_cells(g[:3], idx[:3], dst)
    assert torch.equal(dst[idx[:3]], src[idx[:3]]) and not dst[0].any()


def test_euler_against_golden_fixture(hk):
    """The device Euler layer against the reference-generated fixture (no oracle)."""
    import os
    import torch
    from paper_2505_03360_b200 import kinetic
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "euler_cfg4.npz"))
    nx, ny = int(g["nx"]), int(g["ny"])
    ud = torch.from_numpy(g["u"]).cuda()
    rhs = kinetic.euler_rhs_periodic(ud, nx, ny, 1.0 / nx, 1.0 / ny).cpu().numpy()
    assert np.array_equal(rhs, g["rhs"])
    kinetic.tvd_rk2_step_periodic(ud, nx, ny, 1.0 / nx, 1.0 / ny, float(g["dt"]))
    assert np.array_equal(ud.cpu().numpy(), g["step"])
