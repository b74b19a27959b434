"""Edge cases of the device path: empty and ragged batches, a
single cell, degenerate and zero cells, invalid configurations, tiny grids.
Every case goes through the C-ABI and is checked against the CPU oracle or the
reference's error semantics (inc/errors.hpp)."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def k32(hk):
    vg = hk.make_velocity_grid(32, inputs.VMAX)
    return hk.precompute_kernel(vg, 32, 4, 4, inputs.R_PHYS_MAX)


@pytest.fixture(scope="module")
def ko32(oracle):
    return oracle.kernel(32, inputs.VMAX, 4, 4, inputs.R_PHYS_MAX, closed_form=True)


def test_empty_batch_is_a_noop(hk, k32):
    import torch
    f = torch.empty((0, 32 ** 3), dtype=torch.float64, device="cuda")
    q, st = hk.spectral_collision(f, k32, return_status=True)
    assert q.shape == (0, 32 ** 3) and len(st) == 0


def test_single_cell_and_ragged_batch(hk, k32, ko32, oracle):
    """1 cell and 19 cells (not a multiple of the team count) on the fast path."""
    import torch
    for ncell in (1, 19):
        fh = inputs.config2_cells(ncell, 32, seed_salt=7)
        q = hk.spectral_collision(torch.from_numpy(fh).cuda(), k32).cpu().numpy()
        q_ref, _, _ = oracle.collision_batch(ko32, fh)
        for c in range(ncell):
            assert rel_l2(q[c], q_ref[c]) < TOL, (ncell, c)


def test_zero_cell_gives_zero_and_no_nan(hk, k32):
    import torch
    f = torch.zeros((3, 32 ** 3), dtype=torch.float64, device="cuda")
    f[1] = torch.from_numpy(inputs.config2_cells(1, 32)[0]).cuda()
    q, st = hk.spectral_collision(f, k32, return_status=True)
    q = q.cpu().numpy()
    assert np.all(np.isfinite(q))
    assert not q[0].any() and not q[2].any()
    assert st["q_norm2"][0] == 0.0 and not (st["flags"][0] & 4)


def test_invalid_configurations_raise_reference_exceptions(hk):
    vg = hk.make_velocity_grid(32, inputs.VMAX)
    with pytest.raises(hk.aliasing_config_error):  # src/spectral.cpp:58-66
        hk.precompute_kernel(vg, 32, 4, 4, inputs.R_PHYS_MAX * 1.01)
    with pytest.raises(hk.config_error):
        hk.precompute_kernel(vg, 32, 0, 4, inputs.R_PHYS_MAX)
    with pytest.raises(hk.config_error):
        hk.precompute_kernel(vg, 16, 4, 4, inputs.R_PHYS_MAX)  # n != grid size
    vg48 = hk.make_velocity_grid(48, inputs.VMAX)
    assert hk.precompute_kernel(vg48, 48, 2, 2, inputs.R_PHYS_MAX).n == 48  # general n (hk_collgen.cu)
    vg192 = hk.make_velocity_grid(192, inputs.VMAX)
    with pytest.raises(hk.config_error):  # beyond the device path's size limit (HK_UNSUPPORTED)
        hk.precompute_kernel(vg192, 192, 4, 4, inputs.R_PHYS_MAX)
    with pytest.raises(hk.config_error):
        hk.make_velocity_grid(1, inputs.VMAX)


def test_degenerate_cells_in_stage_and_moments(hk, oracle):
    """rho <= 0 -> degenerate_state_error semantics per cell (status 3), the
    other cells unaffected; a <= 0 stage is the identity (src/boltzmann.cpp:37)."""
    import torch
    from paper_2505_03360_b200 import kinetic
    n = 16
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    fh = inputs.config1_cells(3, n)
    fh[1] = -np.abs(fh[1])  # negative density
    f = torch.from_numpy(fh).cuda()
    out = kinetic.moments_of(f, vg, check=False)
    st = out["status"].cpu().numpy()
    assert st.tolist() == [0, 3, 0]
    m0 = oracle.moments(n, inputs.VMAX, fh[0])[1]
    np.testing.assert_allclose(out["moments"].cpu().numpy()[0], m0, rtol=1e-12)
    ident, _ = kinetic.penalized_stage_solve(torch.from_numpy(inputs.config1_cells(2, n)).cuda(), 0.0, 1e-2,
                                             kinetic.PenalizationRule(), vg, check=False)
    np.testing.assert_array_equal(ident.cpu().numpy(), inputs.config1_cells(2, n))


def test_tiny_periodic_grids_transport(hk, oracle):
    """nx, ny in {1, 2, 3}: periodic wrap onto the cell itself / its neighbour
    (the y-marching kernel needs ny >= 3; smaller grids take the per-node kernel)."""
    import torch
    from paper_2505_03360_b200 import kinetic
    n = 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    rng = np.random.default_rng(5)
    for nx, ny in ((1, 1), (2, 3), (3, 2), (5, 4)):
        fh = rng.uniform(0.1, 1.0, (nx * ny, n ** 3))
        got = kinetic.kinetic_transport_rhs_periodic(torch.from_numpy(fh).cuda(), nx, ny, vg, 0.1, 0.2).cpu().numpy()
        ref = oracle.transport_rhs_periodic(fh, nx, ny, n, inputs.VMAX, 0.1, 0.2)
        # nx = ny = 1 is a uniform field: the exact right-hand side is 0
        scale = max(np.abs(ref).max(), np.abs(fh).max() / 0.1)
        assert np.abs(got - ref).max() <= 1e-13 * scale, (nx, ny)


@pytest.mark.parametrize("n", [4, 6])
def test_small_grids_take_the_generic_cell_kernels(hk, oracle, n):
    """n < 8 (and any n not a power of two) runs the thread-per-cell kernels:
    moments, the ES-BGK and penalized stages against the oracle."""
    import torch
    from paper_2505_03360_b200 import kinetic
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    fh = inputs.config3_cells(3, 2, n)[0]
    f = torch.from_numpy(fh).cuda()
    out = kinetic.moments_of(f, vg)
    for c in range(fh.shape[0]):
        np.testing.assert_allclose(out["moments"].cpu().numpy()[c], oracle.moments(n, inputs.VMAX, fh[c])[1],
                                   rtol=1e-12, atol=1e-14)  # u_z ~ 1e-18 is a rounding zero
    es, _ = kinetic.esbgk_stage_solve(f, 1e-2, 1e-2, kinetic.EsbgkParams(), vg)
    pen, _ = kinetic.penalized_stage_solve(f, 1e-2, 1e-2, kinetic.PenalizationRule(), vg)
    for c in range(fh.shape[0]):
        ref_es = oracle.esbgk_stage_solve(n, inputs.VMAX, fh[c], 1e-2, 1e-2)[0]
        ref_pen = oracle.penalized_stage_solve(n, inputs.VMAX, fh[c], 1e-2, 1e-2)[0]
        assert rel_l2(es.cpu().numpy()[c], ref_es) < 1e-12
        assert rel_l2(pen.cpu().numpy()[c], ref_pen) < 1e-12
