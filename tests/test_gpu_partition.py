"""Single-GPU check of the slab path: transport with separate halo buffers and
the slab PR(2,2,2) step (world 1: halos by local periodic wrap) reproduce the
periodic single-GPU step."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu


def test_slab_step_equals_periodic_step(hk):
    import torch
    from paper_2505_03360_b200 import kinetic
    from paper_2505_03360_b200.partition import XSlab, penalized_imex_step_slab

    n, nx, ny = 16, 6, 4
    f, _ = inputs.config3_cells(nx, ny, n)
    eps = torch.full((nx * ny,), 1e-2, dtype=torch.float64)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX)
    a = torch.from_numpy(f.copy()).cuda()
    kinetic.penalized_imex_step(a, nx, ny, k, 0.1, 0.1, 1e-3, eps)
    part = XSlab(nx, ny, 1, 0)
    b = part.scatter(torch.from_numpy(f.copy()).cuda())
    penalized_imex_step_slab(part, b, k, 0.1, 0.1, 1e-3, eps.cuda())
    torch.cuda.synchronize()
    assert torch.allclose(a, b, rtol=0, atol=1e-13 * float(a.abs().max()))


def test_native_slab_step_equals_periodic_step(hk):
    """hk_penalized_imex_step_slab (the C++ slab driver, halos on a comm stream)
    at world 1, without and with a one-rank NCCL communicator, equals the
    periodic single-GPU step and the Python slab driver."""
    import torch
    from paper_2505_03360_b200 import kinetic
    from paper_2505_03360_b200.partition import XSlab, imex_step_slab_native, penalized_imex_step_slab

    n, nx, ny = 16, 6, 4
    f, _ = inputs.config3_cells(nx, ny, n)
    eps = torch.full((nx * ny,), 1e-2, dtype=torch.float64)
    ctx = hk.Context(0, torch.cuda.current_stream())
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX, ctx=ctx)
    a = torch.from_numpy(f.copy()).cuda()
    kinetic.penalized_imex_step(a, nx, ny, k, 0.1, 0.1, 1e-3, eps)
    part = XSlab(nx, ny, 1, 0)
    b = part.scatter(torch.from_numpy(f.copy()).cuda())
    imex_step_slab_native(part, b, k, 0.1, 0.1, 1e-3, eps.cuda())
    c = part.scatter(torch.from_numpy(f.copy()).cuda())
    penalized_imex_step_slab(part, c, k, 0.1, 0.1, 1e-3, eps.cuda())
    torch.cuda.synchronize()
    tol = 1e-13 * float(a.abs().max())
    assert torch.allclose(a, b, rtol=0, atol=tol) and torch.allclose(c, b, rtol=0, atol=tol)
    try:
        uid = ctx.comm_unique_id()
    except hk.device_error:
        pytest.skip("libnccl.so.2 not loadable")
    ctx.comm_init(1, 0, uid)
    d = part.scatter(torch.from_numpy(f.copy()).cuda())
    imex_step_slab_native(part, d, k, 0.1, 0.1, 1e-3, eps.cuda())
    torch.cuda.synchronize()
    assert torch.equal(d, b)
