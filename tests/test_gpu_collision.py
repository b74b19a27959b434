"""GPU parity of the batched collision operator against the CPU oracle.

Bar (BASELINE.json north_star): Q within 1e-10 relative L2 of the reference
CPU path on the same seeded inputs.  The oracle is the C restatement pinned
bitwise to the reference's own sources (tests/test_oracle_vs_ref.py)."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def n16(oracle, hk):
    n, a1, a2 = 16, 4, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    ko = oracle.kernel(n, inputs.VMAX, a1, a2, inputs.R_PHYS_MAX, closed_form=False)
    f = inputs.config1_cells(6, n)
    q_ref, st_ref, res_ref = oracle.collision_batch(ko, f)
    return dict(vg=vg, kern=kern, ko=ko, f=f, q_ref=q_ref, st_ref=st_ref, res_ref=res_ref)


def test_n16_exact_matches_oracle(n16, hk):
    import torch
    f = torch.from_numpy(n16["f"]).cuda()
    q, st = hk.spectral_collision(f, n16["kern"], exact=True, return_status=True)
    q = q.cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], n16["q_ref"][c]) < TOL, c
    assert np.all(st["flags"] & 1)
    # residue ratio reproduces the reference's verdict (src/spectral.cpp:150)
    res = st["max_im"] / np.maximum(st["max_re"], 1e-300)
    np.testing.assert_allclose(res, n16["res_ref"], rtol=1e-6)
    assert np.array_equal((st["flags"] & 2) != 0, n16["st_ref"] == 4)


@pytest.mark.parametrize("ncells", [1, 2, 5, 7, 64, 211])
def test_n16_item_split_batches(hk, oracle, ncells):
    """The N = 16 kernel spreads the batch's cell halves evenly over one CTA per
    SM, so a cell's two halves run on one CTA or on two depending on the batch
    size (1 cell: 2 CTAs; 211 cells: 2.85 halves per CTA).  Every pattern must
    give the oracle's Q and status, a repeated call the same bits, and a cell
    the same bits alone as inside the batch."""
    import torch
    n, a1, a2 = 16, 4, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    ko = oracle.kernel(n, inputs.VMAX, a1, a2, inputs.R_PHYS_MAX, closed_form=True)
    f = inputs.config1_cells(ncells, n)
    sel = sorted({0, ncells // 3, ncells // 2, ncells - 1})
    q_ref, _, _ = oracle.collision_batch(ko, np.ascontiguousarray(f[sel]))
    fd = torch.from_numpy(f).cuda()
    q, st = hk.spectral_collision(fd, kern, return_status=True)
    q = q.cpu().numpy()
    for i, c in enumerate(sel):
        assert rel_l2(q[c], q_ref[i]) < TOL, (ncells, c)
    assert np.all(st["flags"] & 1)
    np.testing.assert_allclose(st["q_norm2"], (q ** 2).sum(axis=1), rtol=1e-12)
    q2 = hk.spectral_collision(fd, kern).cpu().numpy()
    assert np.array_equal(q, q2)
    # a cell's bits do not depend on the batch it is in (fixed halves, U0 + U1)
    for c in sel:
        q1 = hk.spectral_collision(fd[c:c + 1], kern).cpu().numpy()
        assert np.array_equal(q1[0], q[c]), (ncells, c)


def test_n16_default_path_reroutes_and_matches(n16, hk):
    import torch
    f = torch.from_numpy(n16["f"]).cuda()
    q, st = hk.spectral_collision(f, n16["kern"], return_status=True)
    q = q.cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], n16["q_ref"][c]) < TOL, c
    # at N=16 the Nyquist term matters: the default path is the
    # exact kernel (the fast path's guard would list every cell)
    assert np.all(st["flags"] & 1)


def test_n16_fast_noguard_is_not_exact(n16, hk):
    import torch
    f = torch.from_numpy(n16["f"]).cuda()
    q = hk.spectral_collision(f, n16["kern"], guard=False).cpu().numpy()
    errs = [rel_l2(q[c], n16["q_ref"][c]) for c in range(len(f))]
    assert max(errs) > 1e-9  # proves the guard is load-bearing at N=16
    assert max(errs) < 1e-3


def test_n16_strict_raises_lowest_cell(n16, hk):
    import torch
    f = torch.from_numpy(n16["f"]).cuda()
    with pytest.raises(hk.numerical_consistency_error) as ei:
        hk.spectral_collision(f, n16["kern"], strict=True)
    first = int(np.argmax(n16["st_ref"] == 4))
    assert ei.value.cell == first


def test_n16_reference_tables(n16, hk, oracle):
    """Kernel built from the reference's GK15 tables (bitwise the reference's)."""
    import torch
    ko = n16["ko"]
    kern = hk.precompute_kernel_from_tables(n16["vg"], 16, 4, 8, inputs.R_PHYS_MAX,
                                            ko.alpha, ko.alpha_prime, ko.loss_diag)
    f = torch.from_numpy(n16["f"]).cuda()
    q = hk.spectral_collision(f, kern, exact=True).cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], n16["q_ref"][c]) < 1e-12, c


@pytest.fixture(scope="module")
def n32(oracle, hk):
    n, a1, a2 = 32, 8, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    ko = oracle.kernel(n, inputs.VMAX, a1, a2, inputs.R_PHYS_MAX, closed_form=True)
    f = inputs.config2_cells(3, n)
    q_ref, st_ref, res_ref = oracle.collision_batch(ko, f)
    return dict(vg=vg, kern=kern, f=f, q_ref=q_ref, st_ref=st_ref, res_ref=res_ref)


def test_n32_fast_matches_oracle(n32, hk):
    import torch
    f = torch.from_numpy(n32["f"]).cuda()
    q, st = hk.spectral_collision(f, n32["kern"], return_status=True)
    q = q.cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], n32["q_ref"][c]) < TOL, c
    assert np.all(st["nyq_bound"] < 1e-11)
    assert not np.any(st["flags"] & 4)


def test_n32_exact_matches_oracle(n32, hk):
    import torch
    f = torch.from_numpy(n32["f"]).cuda()
    q, st = hk.spectral_collision(f, n32["kern"], exact=True, return_status=True)
    q = q.cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], n32["q_ref"][c]) < TOL, c
    res = st["max_im"] / np.maximum(st["max_re"], 1e-300)
    np.testing.assert_allclose(res, n32["res_ref"], rtol=1e-3, atol=1e-13)


def test_n32_host_path(n32, hk):
    q = hk.spectral_collision(np.ascontiguousarray(n32["f"]), n32["kern"])
    for c in range(len(q)):
        assert rel_l2(q[c], n32["q_ref"][c]) < TOL, c


@pytest.mark.parametrize("ncells", [1100, 4100])
def test_n32_streamed_host_path_matches_device_path(hk, ncells):
    """The e2e entry point (one persistent launch fed chunk by chunk from pinned
    host memory, results streamed back) gives the device path's Q bitwise,
    including the cells the Nyquist guard reroutes (1100 cells: 16 chunks;
    4100 cells: 128 chunks of 33, the last one ragged)."""
    import torch
    vg = hk.make_velocity_grid(32, inputs.VMAX)
    kern = hk.precompute_kernel(vg, 32, 8, 8, inputs.R_PHYS_MAX)
    f = inputs.config2_cells_torch(ncells, 32, device="cuda")
    q_dev, st_dev = hk.spectral_collision(f, kern, return_status=True)
    fh = f.cpu().pin_memory()
    qh = torch.empty_like(fh).pin_memory()
    q_host, st_host = hk.spectral_collision(fh.numpy(), kern, out=qh.numpy(), return_status=True)
    assert np.array_equal(q_host, q_dev.cpu().numpy())
    assert np.array_equal(st_host["flags"], st_dev["flags"])
    assert (st_host["flags"] & 4).sum() > 0  # some cells rerouted: the re-fetch path ran


def test_n32_nyquist_correction_equals_exact(hk):
    """Cells whose spectrum reaches the Nyquist planes (config-5 shock cells on
    the 32^3 grid: the truncated downstream Maxwellian) fail the guard; their
    fast result plus the exact Nyquist correction (hk_nyqfix.cu) must equal the
    exact kernel's Q to round-off."""
    import torch
    vg = hk.make_velocity_grid(32, inputs.VMAX)
    k = hk.precompute_kernel(vg, 32, 8, 8, inputs.R_PHYS_MAX)
    f = torch.from_numpy(inputs.config5_cells(48, 32, columns=list(range(240, 272)) + [400, 450, 500, 511])).cuda()
    qd, st = hk.spectral_collision(f, k, return_status=True)
    qe = hk.spectral_collision(f, k, exact=True)
    qd, qe = qd.cpu().numpy(), qe.cpu().numpy()
    fixed = (st["flags"] & 4) != 0
    assert fixed.sum() >= 4  # the correction path ran
    for c in range(len(qd)):
        gap = np.linalg.norm(qd[c] - qe[c])
        # round-off of either path: 1e-12 of ||Q||, or 1e-14 of the loss term for near-equilibrium cells
        floor = max(1e-12 * np.linalg.norm(qe[c]), 1e-14 * np.sqrt(st["loss_norm2"][c]))
        assert gap <= (floor if fixed[c] else max(TOL * np.linalg.norm(qe[c]), floor)), c
    # the corrected cells' verdicts describe the corrected Q
    np.testing.assert_allclose(st["q_norm2"][fixed], (qd[fixed] ** 2).sum(1), rtol=1e-12)


def test_n32_conservation_matches_reference_level(n32, hk):
    """Mass, momentum and energy of Q (the collision invariants) are preserved to
    the reference's own level: the invariant moments of the device Q match those
    of the reference's Q to 1e-10 of the moment scale (BASELINE north_star)."""
    import torch
    f = torch.from_numpy(n32["f"]).cuda()
    q = hk.spectral_collision(f, n32["kern"]).cpu().numpy()
    v = inputs.nodes(32)
    vx = np.broadcast_to(v[:, None, None], (32, 32, 32)).ravel()
    vy = np.broadcast_to(v[None, :, None], (32, 32, 32)).ravel()
    vz = np.broadcast_to(v[None, None, :], (32, 32, 32)).ravel()
    phis = [np.ones_like(vx), vx, vy, vz, vx * vx + vy * vy + vz * vz]
    for c in range(len(q)):
        scale = np.abs(n32["q_ref"][c]).sum() * 8.0 ** 2
        for phi in phis:
            ours, ref = float((q[c] * phi).sum()), float((n32["q_ref"][c] * phi).sum())
            assert abs(ours - ref) <= 1e-10 * scale, (c, ours, ref)


@pytest.mark.timeout(300)
def test_n32_pageable_host_buffers(hk):
    """Pageable (not page-locked) host buffers at a streamed-path size: the
    library must route them to the chunked path (a streamed D2H copy into
    pageable memory would block the host before the kernel that releases it is
    launched) and return the device path's Q bitwise."""
    import torch
    vg = hk.make_velocity_grid(32, inputs.VMAX)
    kern = hk.precompute_kernel(vg, 32, 8, 8, inputs.R_PHYS_MAX)
    f = inputs.config2_cells_torch(300, 32, device="cuda")
    q_dev = hk.spectral_collision(f, kern).cpu().numpy()
    fh = np.ascontiguousarray(f.cpu().numpy())
    q_host = hk.spectral_collision(fh, kern)
    assert np.array_equal(q_host, q_dev)


def test_out_argument_is_checked(hk):
    import torch
    vg = hk.make_velocity_grid(16, inputs.VMAX)
    kern = hk.precompute_kernel(vg, 16, 4, 8, inputs.R_PHYS_MAX)
    f = inputs.config1_cells(2, 16)
    with pytest.raises(hk.contract_violation):
        hk.spectral_collision(f, kern, out=np.empty((1, 16 ** 3)))
    with pytest.raises(hk.contract_violation):
        hk.spectral_collision(f, kern, out=np.empty(f.shape, dtype=np.float32))
    fd = torch.from_numpy(f).cuda()
    with pytest.raises(hk.contract_violation):
        hk.spectral_collision(fd, kern, out=torch.empty(16 ** 3, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("n,a1,a2", [(8, 2, 4), (12, 2, 3), (24, 3, 4)])
def test_general_n_matches_oracle(hk, oracle, n, a1, a2):
    """Any n (src/spectral.cpp:53-57 accepts every size; FFTW plans any length):
    the generic device path (direct DFTs, hk_collgen.cu), including n with odd
    prime factors, against the oracle built on the reference's GK15 tables."""
    import torch
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kern = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    ko = oracle.kernel(n, inputs.VMAX, a1, a2, inputs.R_PHYS_MAX, closed_form=False)
    f = inputs.config1_cells(3, n)
    q_ref, st_ref, res_ref = oracle.collision_batch(ko, f)
    q, st = hk.spectral_collision(torch.from_numpy(f).cuda(), kern, return_status=True)
    q = q.cpu().numpy()
    for c in range(len(f)):
        assert rel_l2(q[c], q_ref[c]) < TOL, (n, c)
    res = st["max_im"] / np.maximum(st["max_re"], 1e-300)
    np.testing.assert_allclose(res, res_ref, rtol=1e-4, atol=1e-13)
    qh = hk.spectral_collision(f, kern)  # host entry point, same path
    assert np.array_equal(qh, q)
