"""Memory-safety checks of every device operator without compute-sanitizer
(closed on this GPU pool): each operator runs on views carved out of one
buffer pre-filled with a signalling-NaN sentinel, with 1 MiB canary regions
between its inputs and outputs.  After the call every canary must still hold
the sentinel (no out-of-bounds write next to a buffer), every read-only input
must be unchanged, every output element must have been written (no sentinel
or NaN left: no read-before-write of an output), and a second run must give
the same bits (no race, no uninitialised read)."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu
SENT = np.array([0x7FF4DEADBEEF1234], dtype=np.uint64).view(np.float64)[0]  # signalling NaN payload
PAD = (1 << 20) // 8


class Arena:
    """Views into one sentinel-filled device buffer, separated by canaries."""

    def __init__(self, sizes):
        import torch
        total = PAD + sum(s + PAD for s in sizes)
        self.buf = torch.empty((total,), dtype=torch.float64, device="cuda")
        self.buf.view(torch.int64).fill_(int(np.array([SENT]).view(np.int64)[0]))  # the exact sentinel bits
        self.views, self.pads = [], [(0, PAD)]
        o = PAD
        for s in sizes:
            self.views.append(self.buf[o:o + s])
            self.pads.append((o + s, o + s + PAD))
            o += s + PAD

    def canaries_intact(self):
        import torch
        bits = self.buf.view(torch.int64)
        ref = int(np.array([SENT]).view(np.int64)[0])
        return all(bool((bits[a:b] == ref).all()) for a, b in self.pads)


def run_checked(fn, inputs_np, out_sizes):
    """fn(in_views, out_views) runs the operator; returns the outputs (numpy)."""
    results = []
    for rep in range(2):
        ar = Arena([x.size for x in inputs_np] + list(out_sizes))
        ins = ar.views[:len(inputs_np)]
        outs = ar.views[len(inputs_np):]
        import torch
        for v, x in zip(ins, inputs_np):
            v.copy_(torch.from_numpy(np.ascontiguousarray(x).ravel()))
        fn(ins, outs)
        torch.cuda.synchronize()
        assert ar.canaries_intact(), "a canary next to a buffer was overwritten"
        for v, x in zip(ins, inputs_np):
            assert np.array_equal(v.cpu().numpy(), np.ascontiguousarray(x).ravel()), "read-only input modified"
        o = [v.cpu().numpy() for v in outs]
        for a in o:
            assert not np.isnan(a).any(), "output element left unwritten (sentinel / NaN)"
        results.append(o)
    for a, b in zip(*results):
        assert np.array_equal(a.view(np.int64), b.view(np.int64)), "two runs differ"
    return results[0]


@pytest.mark.parametrize("n,a1,a2,exact", [(16, 4, 8, False), (32, 8, 8, False), (32, 4, 4, True),
                                           (64, 8, 8, False), (64, 2, 4, True)])
def test_collision(hk, n, a1, a2, exact):
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    if n == 16:
        f = inputs.config1_cells(5, n)
    elif n == 32:  # config-2 cells plus guard-listed (Nyquist-corrected) ones
        f = np.concatenate([inputs.config2_cells(3, n), inputs.config5_cells(3, n, columns=[300, 400, 511])])
    else:
        f = inputs.config5_cells(3, n, columns=[250, 256, 511])
    nc, nb = f.shape

    def op(i, o):
        hk.spectral_collision(i[0].view(nc, nb), k, out=o[0].view(nc, nb), exact=exact)

    run_checked(op, [f], [f.size])


def test_cell_operators(hk):
    from paper_2505_03360_b200 import kinetic
    import torch
    n = 32
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    f, _ = inputs.config3_cells(3, 2, n)
    nc, nb = f.shape
    k = hk.precompute_kernel(vg, n, 4, 8, inputs.R_PHYS_MAX)

    def op(i, o):
        fv = i[0].view(nc, nb)
        ctx = k.ctx
        L = ctx._lib
        mom, sig, real, l1 = o[0], o[1], o[2], o[3]
        st = torch.zeros(nc, dtype=torch.int32, device="cuda")
        ctx.check(L.hk_moments_batch(ctx.h, n, inputs.VMAX, fv.data_ptr(), nc, mom.data_ptr(), sig.data_ptr(),
                                     real.data_ptr(), l1.data_ptr(), st.data_ptr()))
        ctx.check(L.hk_esbgk_stage_batch(ctx.h, n, inputs.VMAX, fv.data_ptr(), o[4].data_ptr(), nc, 1e-3, None, 1e-2,
                                         -0.5, 0.5 * np.pi, st.data_ptr(), None))
        ctx.check(L.hk_penalized_stage_batch(ctx.h, n, inputs.VMAX, fv.data_ptr(), o[5].data_ptr(), nc, 1e-3, None,
                                             1e-2, 2 * np.pi, st.data_ptr(), None))
        ctx.check(L.hk_penalized_residual_batch(ctx.h, k.h, fv.data_ptr(), o[6].data_ptr(), nc, 2 * np.pi, 0,
                                                st.data_ptr(), None))
        ctx.check(L.hk_maxwellian_batch(ctx.h, n, inputs.VMAX, mom.data_ptr(), nc, o[7].data_ptr(), st.data_ptr()))

    run_checked(op, [f], [nc * 5, nc * 6, nc * 13, nc, f.size, f.size, f.size, f.size])


def test_transport_and_steps(hk):
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 16, 5, 4
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    f, _ = inputs.config3_cells(nx, ny, n)
    eps = np.full(nx * ny, 1e-2)
    k = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX)

    def op(i, o):
        import torch
        fv = i[0].view(nx * ny, -1)
        o[0].view(nx * ny, -1).copy_(kinetic.kinetic_transport_rhs_periodic(fv, nx, ny, vg, 0.1, 0.1))
        ctx = k.ctx
        ctx.check(ctx._lib.hk_transport_rhs(ctx.h, n, inputs.VMAX, fv.data_ptr(), o[1].data_ptr(), nx, ny, 0, 0.1,
                                            0.1, 1e-6))
        o[2].copy_(i[0])
        kinetic.esbgk_imex_step(o[2].view(nx * ny, -1), nx, ny, vg, 0.1, 0.1, 1e-3, i[1])
        o[3].copy_(i[0])
        kinetic.penalized_imex_step(o[3].view(nx * ny, -1), nx, ny, k, 0.1, 0.1, 1e-3, i[1])

    run_checked(op, [f, eps], [f.size] * 4)


def test_hybrid_step(hk):
    from paper_2505_03360_b200 import kinetic
    import torch
    nx, ny, n = 8, 6, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, 4, 4, inputs.R_PHYS_MAX)

    def op(i, o):
        o[0].copy_(i[0])
        o[1].copy_(i[1])
        rd = torch.from_numpy(r.copy()).cuda()
        kinetic.hybrid_step(k, nx, ny, 1 / nx, 1 / ny, 2e-3, i[2], rd, o[0].view(-1, 4), o[1].view(nx * ny, -1))
        o[2].copy_(rd.double())

    out = run_checked(op, [hydro, f, eps], [hydro.size, f.size, r.size])
    assert out[2].max() > 0
