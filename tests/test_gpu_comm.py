"""Native NCCL path of the C-ABI (hk_comm.cu) on one GPU: a one-rank
communicator wraps the x-slab halos onto itself (periodic), which exercises
the posting order of the grouped send/recv and the [ny][2][n^3] layout that
hk_transport_rhs_slab reads; all-reduce over one rank is the identity.
(Multi-rank halos are covered by the gloo tests of the Python partitioner,
tests/test_partition_gloo.py; this box has one GPU.)"""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm_ctx(hk):
    import torch
    ctx = hk.Context(0, torch.cuda.current_stream())
    ctx.comm_init(1, 0, hk.Context.comm_unique_id())
    return ctx


def test_halo_exchange_single_rank_is_periodic_wrap(comm_ctx):
    import torch
    n, nxl, ny = 8, 5, 3
    nb = n ** 3
    f = torch.randn(ny, nxl, nb, dtype=torch.float64, device="cuda")
    left = torch.full((ny, 2, nb), float("nan"), dtype=torch.float64, device="cuda")
    right = torch.full_like(left, float("nan"))
    comm_ctx.halo_exchange(f, n, nxl, ny, left, right)
    torch.cuda.synchronize()
    assert torch.equal(left, f[:, nxl - 2:])   # left ghosts = own last two columns
    assert torch.equal(right, f[:, :2])        # right ghosts = own first two columns


def test_halo_feeds_slab_transport(comm_ctx, hk):
    """Slab transport with natively exchanged halos == periodic transport."""
    import torch
    from paper_2505_03360_b200 import kinetic
    n, nx, ny = 8, 6, 4
    vg = hk.make_velocity_grid(n, 8.0)
    f = torch.rand(ny * nx, n ** 3, dtype=torch.float64, device="cuda") + 0.1
    left = torch.empty(ny, 2, n ** 3, dtype=torch.float64, device="cuda")
    right = torch.empty_like(left)
    comm_ctx.halo_exchange(f, n, nx, ny, left, right)
    out = torch.empty_like(f)
    lib = comm_ctx._lib
    import ctypes as C
    comm_ctx.check(lib.hk_transport_rhs_slab(comm_ctx.h, n, C.c_double(8.0), C.c_void_p(f.data_ptr()),
                                             C.c_void_p(left.data_ptr()), C.c_void_p(right.data_ptr()),
                                             C.c_void_p(out.data_ptr()), nx, ny, C.c_double(1.0 / nx),
                                             C.c_double(1.0 / ny), C.c_double(1e-6)))
    ref = kinetic.kinetic_transport_rhs_periodic(f, nx, ny, vg, 1.0 / nx, 1.0 / ny)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_allreduce_single_rank(comm_ctx):
    import torch
    x = torch.tensor([1.0, -2.0, 3.5], dtype=torch.float64, device="cuda")
    y = comm_ctx.allreduce_(x.clone(), "sum")
    z = comm_ctx.allreduce_(x.clone(), "max")
    torch.cuda.synchronize()
    assert torch.equal(y, x) and torch.equal(z, x)
