"""x-slab partitioner host logic on CPU with the gloo backend (world 2 and 3):
halo exchange == periodic neighbour columns, gather/scatter, all-reduces."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nx, ny, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_03360_b200.partition import XSlab, HALO, regime_counts, conservation_sums
        g = torch.Generator().manual_seed(1234)
        glob = torch.randn((ny * nx, nb), generator=g, dtype=torch.float64)
        part = XSlab(nx, ny, world, rank)
        loc = part.scatter(glob)
        lh, rh = part.halo_buffers(nb, loc)
        part.exchange(loc, lh, rh)
        G = glob.view(ny, nx, nb)
        li = [(part.i0 - HALO + k) % nx for k in range(HALO)]
        ri = [(part.i0 + part.nxl + k) % nx for k in range(HALO)]
        ok = torch.equal(lh, G[:, li]) and torch.equal(rh, G[:, ri])
        ok = ok and torch.equal(part.gather(loc), glob)
        # async variant
        lh2, rh2 = part.halo_buffers(nb, loc)
        works = part.exchange(loc, lh2, rh2, async_op=True)
        for w in works:
            if hasattr(w, "wait"):
                w.wait()
        ok = ok and torch.equal(lh2, lh) and torch.equal(rh2, rh)
        # regime counts and conservation sums are global
        r = (torch.arange(part.cells) + part.i0) % 3
        counts = regime_counts(r)
        mom = torch.ones((part.cells, 5), dtype=torch.float64)
        sums = conservation_sums(mom)
        ok = ok and counts.sum().item() == nx * ny and abs(sums[0].item() - nx * ny) < 1e-9
        q.put((rank, ok, part.i0, part.nxl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx", [(2, 9), (3, 11)])
def test_halo_exchange_gloo(world, nx):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, 4, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res), res
    cols = sorted((i0, nxl) for _, _, i0, nxl in res)
    assert sum(n for _, n in cols) == nx and all(cols[k][0] + cols[k][1] == cols[k + 1][0] for k in range(world - 1))


def _wide_worker(rank, world, port, nx, ny, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_03360_b200.partition import XSlab, HYB_GHOST, hybrid_pad, hybrid_unpad
        W = HYB_GHOST
        g = torch.Generator().manual_seed(99)
        glob_f = torch.randn((ny * nx, 6), generator=g, dtype=torch.float64)
        glob_r = torch.randint(0, 3, (ny * nx, 1), generator=g).to(torch.int8)
        part = XSlab(nx, ny, world, rank)
        fields = [part.scatter(glob_r), part.scatter(glob_f)]
        halos = []
        for t in fields:
            lh, rh = part.halo_buffers(t.shape[-1], t, W)
            part.exchange(t, lh, rh, width=W)
            halos.append((lh, rh))
        pr, pf = hybrid_pad(part, W, fields, halos)
        cols = [(part.i0 - W + k) % nx for k in range(part.nxl + 2 * W)]
        ok = torch.equal(pr.view(ny, -1, 1), glob_r.view(ny, nx, 1)[:, cols])
        ok = ok and torch.equal(pf.view(ny, -1, 6), glob_f.view(ny, nx, 6)[:, cols])
        pf.mul_(2.0)
        out = torch.zeros_like(fields[1])
        hybrid_unpad(part, W, [pf], [out])
        ok = ok and torch.equal(out, 2.0 * fields[1])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx", [(2, 20), (3, 27)])
def test_hybrid_slab_padding_gloo(world, nx):
    """The slab hybrid step's padded local torus (8 exchanged columns per side,
    int8 layers and fp64 fields) is the global periodic window of the slab."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_wide_worker, args=(r, world, port, nx, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_slab_bounds():
    from paper_2505_03360_b200.partition import XSlab
    with pytest.raises(ValueError):
        XSlab(3, 4, 2, 0)
    p = XSlab(512, 128, 8, 7)
    assert p.nxl == 64 and p.i0 == 448 and p.left == 6 and p.right == 0


def test_weighted_bounds_balance():
    """Work-weighted slab boundaries: valid split, >= 8 columns each, and a lower
    maximum slab work than the even split on a banded work profile."""
    import numpy as np
    from paper_2505_03360_b200.partition import XSlab, weighted_bounds
    nx, world = 200, 8
    w = np.full(nx, 40.0)
    w[95:105] = 400.0
    w[:5] = w[-5:] = 400.0
    b = weighted_bounds(w, world)
    assert b[0] == 0 and b[-1] == nx and all(b[q + 1] - b[q] >= 8 for q in range(world))

    def worst(bounds):
        return max(w[np.arange(bounds[q] - 2, bounds[q + 1] + 2) % nx].sum() for q in range(world))

    even = [q * nx // world for q in range(world)] + [nx]
    assert worst(b) <= 0.85 * worst(even)
    parts = [XSlab(nx, 4, world, q, b) for q in range(world)]
    assert [p.i0 for p in parts] == list(b[:-1]) and sum(p.nxl for p in parts) == nx
    with pytest.raises(ValueError):
        XSlab(nx, 4, 2, 0, (0, 1, nx))


def test_native_slab_step_rejects_explicit_halos():
    """hybrid_step_slab(native=True) moves its halos over the context's own
    communicator: explicit halo tensors are a caller error (raised before any
    device work)."""
    import pytest
    import torch
    from paper_2505_03360_b200.partition import XSlab, hybrid_step_slab
    part = XSlab(8, 4, 1, 0)
    r = torch.zeros(32, dtype=torch.int8)
    e = torch.zeros(32, dtype=torch.float64)
    h = torch.zeros((32, 4), dtype=torch.float64)
    f = torch.zeros((32, 8), dtype=torch.float64)
    with pytest.raises(ValueError):
        hybrid_step_slab(part, None, 0.1, 0.1, 0.01, e, r, h, f, halos=[], native=True)
