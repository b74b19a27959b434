"""x-slab domain partitioner with NCCL halo exchange.

The periodic nx x ny spatial grid is split into contiguous x-slabs, one per
rank (one process per GPU).  Collision, moments and relaxation stages are
per-cell and need no communication; the CWENO3 transport sweep needs a
2-column f halo from each x-neighbour before every PR(2,2,2) stage, and
the driver needs scalar all-reduces (regime counts, conservation sums,
CFL max).  Halos travel as grouped point-to-point send/recv on the
process group's backend: NCCL over NVLink/NVSwitch on GPUs, gloo on CPU
(the tests).  The exchange is issued asynchronously and overlapped with
the stage's collision work, which does not read halos.

Local layout: interior cells [ny][nxl][n^3] (cell (i, j) at j*nxl + i,
matching the reference's c = j*nx + i within the slab); halos are separate
[ny][2][n^3] buffers (left = global columns i0-2, i0-1; right = i0+nxl,
i0+nxl+1, periodic).  The reference is single-process; this
replaces its shared-memory row-stripe WorkerPool partition
(inc/threading.hpp:25-56) with a distributed one.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

HALO = 2  # CWENO3 stencil radius (src/transport.cpp:12-21)


@dataclass
class XSlab:
    nx: int
    ny: int
    world: int
    rank: int
    bounds: tuple = None  # optional column boundaries (world + 1 values, 0 .. nx); default: even split

    def __post_init__(self):
        if self.nx < self.world * HALO:
            raise ValueError(f"nx={self.nx} too small for {self.world} slabs with a {HALO}-column halo")
        if self.bounds is not None:
            b = list(self.bounds)
            if len(b) != self.world + 1 or b[0] != 0 or b[-1] != self.nx or any(b[q + 1] - b[q] < HALO for q in
                                                                              range(self.world)):
                raise ValueError(f"bounds {b} must split 0..{self.nx} into {self.world} slabs of >= {HALO} columns")
            self.i0, self.nxl = b[self.rank], b[self.rank + 1] - b[self.rank]
        else:
            base, rem = divmod(self.nx, self.world)
            self.nxl = base + (1 if self.rank < rem else 0)
            self.i0 = self.rank * base + min(self.rank, rem)
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world

    @property
    def cells(self) -> int:
        return self.nxl * self.ny

    def columns(self):
        return range(self.i0, self.i0 + self.nxl)

    def global_cells(self) -> torch.Tensor:
        """Global cell index (j*nx + i) of every local cell, in local order."""
        j = torch.arange(self.ny).repeat_interleave(self.nxl)
        i = torch.arange(self.i0, self.i0 + self.nxl).repeat(self.ny)
        return j * self.nx + i

    def scatter(self, global_field: torch.Tensor) -> torch.Tensor:
        """Local interior [ny*nxl, nb] from a global [ny*nx, nb] field."""
        g = global_field.view(self.ny, self.nx, -1)
        # always a new tensor (at world 1 the slice is the whole field: never alias it)
        return g[:, self.i0:self.i0 + self.nxl].reshape(self.cells, -1).clone(memory_format=torch.contiguous_format)

    def gather(self, local: torch.Tensor, group=None) -> torch.Tensor:
        """Global field assembled on every rank (tests / snapshots)."""
        nb = local.shape[-1]
        if self.world == 1:
            return local.clone()
        parts = [None] * self.world
        dist.all_gather_object(parts, (self.i0, self.nxl, local.cpu()), group=group)
        out = torch.empty((self.ny, self.nx, nb), dtype=local.dtype)
        for i0, nxl, t in parts:
            out[:, i0:i0 + nxl] = t.view(self.ny, nxl, nb)
        return out.view(self.ny * self.nx, nb).to(local.device)

    def halo_buffers(self, nb: int, like: torch.Tensor, width: int = HALO):
        shape = (self.ny, width, nb)
        return torch.empty(shape, dtype=like.dtype, device=like.device), torch.empty(shape, dtype=like.dtype,
                                                                                   device=like.device)

    def exchange(self, local: torch.Tensor, left: torch.Tensor, right: torch.Tensor, group=None, async_op=False,
                 width: int = HALO):
        """Fills left/right halos from the neighbours' edge columns.

        Ops are issued in the order [send right edge -> right, recv left halo <- left,
        send left edge -> left, recv right halo <- right], so that with world = 2
        (left == right) the two messages between the pair match in order.
        Returns a list of works (async_op) or None after completion."""
        if width > self.nxl:
            raise ValueError(f"halo width {width} exceeds the slab width {self.nxl}")
        nb = local.shape[-1]
        f = local.view(self.ny, self.nxl, nb)
        send_r = f[:, self.nxl - width:].contiguous()  # my last interior columns -> right's left halo
        send_l = f[:, :width].contiguous()             # my first interior columns -> left's right halo
        if self.world == 1:
            left.copy_(send_r)
            right.copy_(send_l)
            return [] if async_op else None
        ops = [dist.P2POp(dist.isend, send_r, self.right, group),
               dist.P2POp(dist.irecv, left, self.left, group),
               dist.P2POp(dist.isend, send_l, self.left, group),
               dist.P2POp(dist.irecv, right, self.right, group)]
        works = dist.batch_isend_irecv(ops)
        keep = (send_r, send_l)  # keep send buffers alive until completion
        if async_op:
            return works + [keep]
        for w in works:
            w.wait()
        return None


def wait_all(works):
    for w in works:
        if hasattr(w, "wait"):
            w.wait()


def allreduce_sum(values: torch.Tensor, group=None) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values


def allreduce_max(values: torch.Tensor, group=None) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.MAX, group=group)
    return values


def regime_counts(r: torch.Tensor, group=None) -> torch.Tensor:
    """Global number of cells in layers 0/1/2 (the paper's Table 1 statistic)."""
    c = torch.stack([(r == k).sum() for k in range(3)]).to(torch.float64)
    return allreduce_sum(c, group)


def conservation_sums(moments: torch.Tensor, group=None) -> torch.Tensor:
    """Global (mass, momentum x/y/z, energy) from per-cell moments [cells,5]
    (per unit cell volume; E = 1/2 rho |u|^2 + 3/2 rho T, inc/moments.hpp:19)."""
    rho, u, T = moments[:, 0], moments[:, 1:4], moments[:, 4]
    s = torch.stack([rho.sum(), (rho[:, None] * u).sum(0)[0], (rho[:, None] * u).sum(0)[1],
                     (rho[:, None] * u).sum(0)[2], (0.5 * rho * (u * u).sum(1) + 1.5 * rho * T).sum()])
    return allreduce_sum(s, group)


def penalized_imex_step_slab(part: XSlab, f: torch.Tensor, kernel, dx: float, dy: float, dt: float,
                             eps_cell: torch.Tensor, pen_coeff: float = 6.283185307179586, eps_weno: float = 1e-6,
                             group=None, work=None, peer=None):
    """penalized_imex_step (src/boltzmann.cpp:47-110) on one x-slab, in place.

    Same operation sequence as the single-GPU hk_penalized_imex_step; the
    stage field's halos are exchanged before each transport, overlapped with
    the residual (collision) evaluation of that stage.

    peer: a PeerHalo mapped on work[0] (the stage field Y): the transport then
    reads the neighbours' ghost columns of Y straight from their memory
    (hk_transport_rhs_peer over NVLink / CUDA IPC) instead of exchanging
    halos; Y is published (refresh) after each stage solve and released
    (done) before the next one overwrites it."""
    from . import _abi  # noqa: F401
    from . import make_velocity_grid

    ctx = kernel.ctx
    L = ctx._lib
    n = kernel.n
    nb = n ** 3
    cells = part.cells
    count = cells * nb
    if work is None:
        work = torch.empty((6, cells, nb), dtype=torch.float64, device=f.device)
    y, q1, k1, tr, res, fa = work
    if peer is not None and peer.slab.data_ptr() != y.data_ptr():
        raise ValueError("peer must be a PeerHalo mapped on work[0] (the stage field)")
    vg = make_velocity_grid(n, kernel.vmax)
    e = eps_cell.to(device=f.device, dtype=torch.float64).contiguous()
    lh, rh = part.halo_buffers(nb, f) if peer is None else (None, None)
    a00 = 1.0 - 2.0 ** -0.5
    a11 = 1.0 - 1.0 / (2.0 * 2.0 ** -0.5)

    def stage(fin, a, out):
        ctx.check(L.hk_penalized_stage_batch(ctx.h, n, kernel.vmax, fin.data_ptr(), out.data_ptr(), cells, a,
                                             e.data_ptr(), 0.0, pen_coeff, None, None))

    def residual(yv, out):
        ctx.check(L.hk_penalized_residual_batch(ctx.h, kernel.h, yv.data_ptr(), out.data_ptr(), cells, pen_coeff, 0,
                                                None, None))

    def transport(yv, out):
        ctx.check(L.hk_transport_rhs_slab(ctx.h, n, kernel.vmax, yv.data_ptr(), lh.data_ptr(), rh.data_ptr(),
                                          out.data_ptr(), part.nxl, part.ny, dx, dy, eps_weno))

    def comb(op, out, fv=None, yv=None, qv=None, kv=None, tv=None, rv=None):
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        ctx.check(L.hk_imex_combine(ctx.h, op, count, nb, dt, e.data_ptr(), out.data_ptr(), p(fv), p(yv), p(qv),
                                    p(kv), p(tv), p(rv)))

    def halo_transport(yv, out):
        if peer is not None:
            peer.refresh()             # every rank's Y is written
            residual(yv, res)
            peer.transport(out, vg, dx, dy, eps_weno)
            peer.done()                # the neighbours have read my ghost columns
        else:
            works = part.exchange(yv, lh, rh, group, async_op=True)
            residual(yv, res)          # overlaps the halo exchange
            wait_all(works)
            transport(yv, out)

    stage(f, a00 * dt, y)
    comb(0, k1, fv=f, yv=y)
    halo_transport(y, tr)
    comb(1, q1, tv=tr, rv=res)
    comb(2, fa, fv=f, qv=q1, kv=k1)
    stage(fa, a11 * dt, y)
    halo_transport(y, tr)
    comb(3, f, yv=y, qv=q1, kv=k1, tv=tr, rv=res)
    return f


def imex_step_slab_native(part: XSlab, f: torch.Tensor, kernel, dx: float, dy: float, dt: float,
                          eps_cell: torch.Tensor, pen_coeff: float = 6.283185307179586, eps_weno: float = 1e-6,
                          exact: bool = False, work=None):
    """penalized_imex_step (src/boltzmann.cpp:47-110) on one x-slab, in place, driven
    in C++ (hk_penalized_imex_step_slab): the halos travel over the context's own NCCL
    communicator (Context.comm_init; without one the slab wraps onto itself) on a
    separate stream, overlapped with each stage's collision."""
    from . import _abi

    ctx = kernel.ctx
    if not (f.is_cuda and f.dtype == torch.float64 and f.is_contiguous()):
        raise ValueError("f must be a contiguous float64 CUDA tensor")
    e = eps_cell.to(device=f.device, dtype=torch.float64).contiguous()
    ctx.check(ctx._lib.hk_penalized_imex_step_slab(ctx.h, kernel.h, f.data_ptr(), part.nxl, part.ny, dx, dy, dt,
                                                   e.data_ptr(), pen_coeff, eps_weno,
                                                   _abi.HK_COLL_EXACT if exact else 0,
                                                   None if work is None else work.data_ptr()))
    return f


def native_comm_init(ctx, group=None):
    """Gives the context its own NCCL communicator over the ranks of `group`
    (rank 0's unique id travels over torch.distributed)."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    uid = [ctx.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    ctx.comm_init(world, rank, uid[0])


# Ghost width of the slab hybrid step: the exact dependency radius of one
# hybrid step along x is 7 cells (regime update 1, halo Maxwellians +2, two
# transport sweeps +2 each; the layer-0 TVD-RK2 needs 4), so a slab padded with
# 8 exchanged columns per side and stepped as a local periodic torus gets
# every interior cell exactly as the global torus would.
HYB_GHOST = 8


def weighted_bounds(col_work, world: int, min_width: int = HYB_GHOST, ghost: int = 2):
    """Column boundaries of `world` x-slabs that balance the per-slab work: col_work[i]
    = work of column i (e.g. 2 x layer-2 cells + layer-1 cells / 10), a slab's work being
    its columns' plus that of `ghost` extra columns per side (the ghost cells whose
    residual the slab evaluates).  Exact min-max split by dynamic programming over the
    boundaries (slab 0 starts at column 0); every slab keeps >= min_width columns."""
    import numpy as np

    w = np.asarray(col_work, dtype=np.float64)
    nx = len(w)
    if nx < world * min_width:
        raise ValueError("grid too narrow for the requested slabs")
    ext = np.concatenate([w[nx - ghost:], w, w[:ghost]]) if ghost else w
    P = np.concatenate([[0.0], np.cumsum(ext)])
    work = lambda a, e: P[e + 2 * ghost] - P[a]  # noqa: E731  columns a-ghost .. e+ghost-1 (periodic)
    INF = float("inf")
    best = np.full((world + 1, nx + 1), INF)
    arg = np.zeros((world + 1, nx + 1), dtype=np.int64)
    best[0, 0] = 0.0
    for q in range(1, world + 1):
        for e in range(q * min_width, nx - (world - q) * min_width + 1):
            a = np.arange((q - 1) * min_width, e - min_width + 1)
            cand = np.maximum(best[q - 1, a], work(a, e))
            k = int(np.argmin(cand))
            best[q, e], arg[q, e] = cand[k], a[k]
    bounds = [nx]
    for q in range(world, 0, -1):
        bounds.append(int(arg[q, bounds[-1]]))
    return tuple(reversed(bounds))


def hybrid_pad(part: XSlab, width: int, fields, halos):
    """[ny][nxl + 2 width] padded copies of the local fields (each [cells, k]),
    halos = [(left [ny][width][k], right [ny][width][k]), ...]."""
    out = []
    for t, (lh, rh) in zip(fields, halos):
        k = t.shape[-1]
        pad = torch.empty((part.ny, part.nxl + 2 * width, k), dtype=t.dtype, device=t.device)
        pad[:, :width] = lh
        pad[:, width:width + part.nxl] = t.view(part.ny, part.nxl, k)
        pad[:, width + part.nxl:] = rh
        out.append(pad.view(part.ny * (part.nxl + 2 * width), k))
    return out


def hybrid_unpad(part: XSlab, width: int, padded, fields):
    for pad, t in zip(padded, fields):
        k = t.shape[-1]
        t.view(part.ny, part.nxl, k).copy_(pad.view(part.ny, part.nxl + 2 * width, k)[:, width:width + part.nxl])


def hybrid_step_slab(part: XSlab, kernel, dx: float, dy: float, dt: float, eps_cell: torch.Tensor, r: torch.Tensor,
                     hydro: torch.Tensor, f: torch.Tensor, params=None, group=None, width: int = HYB_GHOST,
                     halos=None, balance: bool = False, residual_hook=None, native: bool = False):
    """hk_hybrid_step on one x-slab, in place (r [cells] int8, hydro [cells,4], f [cells,n^3],
    eps [cells]; local cell order j*nxl + i).  One exchange of `width` columns of
    (r, eps, hydro, f) per side, then the step on the padded local torus; the
    interior is exactly the global step's.  Returns the global layer counts
    [n0, n1, n2] (all-reduced).  `halos` (tests) supplies the exchanged columns
    directly: [(left, right)] for r, eps, hydro, f as [ny][width][k].

    balance (SURVEY §8f "next" #3): the layer-2 residuals of the step (the
    collision evaluations, its dominant cost when Boltzmann cells cluster at
    an interface) are spread evenly over the ranks: balanced_apply ships the
    surplus stage values of over-loaded ranks to under-loaded ones, evaluates
    dense batches and returns the results; per-cell operators are
    deterministic, so the step is bitwise the unbalanced one.
    residual_hook: an explicit hk_hybrid_params.residual_fn (see kinetic.hybrid_step).
    native: the exchange, padding, step and counts in C++ (hk_hybrid_step_slab) over the
    kernel context's NCCL communicator (hk_ctx_comm_init; a single rank wraps onto
    itself), bitwise this function's result."""
    import dataclasses

    from .kinetic import HybridParams, hybrid_step, hybrid_step_slab_native, penalized_residual_rows

    # ghost results are discarded: their residuals only where an interior cell depends on them
    params = dataclasses.replace(params or HybridParams(), ghost_x=width)
    fields = [r.view(-1, 1), eps_cell.to(device=f.device, dtype=torch.float64).view(-1, 1), hydro, f]
    if balance and residual_hook is None:
        def residual_hook(y, res, status):
            balanced_residual(kernel, y, res, status, params.pen_coeff, params.exact, group)
    if native:
        if halos is not None:
            raise ValueError("native: the halos travel over the context's communicator")
        counts = hybrid_step_slab_native(kernel, part.nxl, part.ny, dx, dy, dt, fields[1].view(-1), r, hydro, f,
                                         params, ghost=width, residual_hook=residual_hook)
        return torch.tensor(counts, dtype=torch.float64, device=f.device)
    if halos is None:
        halos = []
        for t in fields:
            lh, rh = part.halo_buffers(t.shape[-1], t, width)
            part.exchange(t, lh, rh, group, width=width)
            halos.append((lh, rh))
    pr, pe, ph, pf = hybrid_pad(part, width, fields, halos)
    hybrid_step(kernel, part.nxl + 2 * width, part.ny, dx, dy, dt, pe.view(-1), pr.view(-1), ph, pf, params,
                residual_hook=residual_hook)
    hybrid_unpad(part, width, [pr, ph, pf], [fields[0], hydro, f])
    return regime_counts(r, group)


class PeerHalo:
    """x-slab transport over NVLink / NVSwitch peer memory: the neighbours'
    slabs are mapped into this process once (CUDA IPC), and the transport
    kernel reads their two ghost columns directly (hk_transport_rhs_peer): no
    exchange step and no halo buffers.  `refresh()` orders the neighbours'
    writes before the read (stream sync + barrier); call it before every
    transport of a field the neighbours just wrote, and again before they
    overwrite it (`done()`).  One rank maps its own slab (periodic wrap)."""

    def __init__(self, part: XSlab, slab: torch.Tensor, ctx, group=None):
        import ctypes as C
        from . import _abi
        self.part, self.slab, self.ctx, self.group = part, slab, ctx, group
        lib = ctx._lib
        handle = C.create_string_buffer(_abi.HK_IPC_HANDLE_BYTES)
        off = C.c_int64(0)
        ctx.check(lib.hk_ipc_handle(ctx.h, C.c_void_p(slab.data_ptr()), handle, C.byref(off)))
        mine = (handle.raw, off.value, part.nxl)
        if part.world == 1:
            infos = [mine]
        else:
            infos = [None] * part.world
            dist.all_gather_object(infos, mine, group=group)
        self._opened = []

        def ptr_of(rank):
            if rank == part.rank:
                return slab.data_ptr(), part.nxl
            h, o, nxl = infos[rank]
            base = C.c_void_p()
            ctx.check(lib.hk_ipc_open(ctx.h, C.c_char_p(h), C.byref(base)))
            self._opened.append(base)
            return base.value + o, nxl

        self.left_ptr, self.left_nx = ptr_of(part.left)
        if part.right == part.left:
            self.right_ptr, self.right_nx = self.left_ptr, self.left_nx
        else:
            self.right_ptr, self.right_nx = ptr_of(part.right)

    def refresh(self):
        torch.cuda.current_stream().synchronize()
        if self.part.world > 1:
            dist.barrier(group=self.group)

    done = refresh

    def transport(self, out: torch.Tensor, vgrid, dx: float, dy: float, eps_weno: float = 1e-6):
        import ctypes as C
        p = self.part
        self.ctx.check(self.ctx._lib.hk_transport_rhs_peer(
            self.ctx.h, vgrid.nv, C.c_double(vgrid.vmax), C.c_void_p(self.slab.data_ptr()),
            C.c_void_p(self.left_ptr), self.left_nx, C.c_void_p(self.right_ptr), self.right_nx,
            C.c_void_p(out.data_ptr()), p.nxl, p.ny, C.c_double(dx), C.c_double(dy), C.c_double(eps_weno)))
        return out

    def close(self):
        for b in self._opened:
            self.ctx._lib.hk_ipc_close(self.ctx.h, b)
        self._opened = []


# ---------------------------------------------------------------------------
# Dynamic load balancing of Boltzmann (layer-2) cells across ranks (SURVEY §8f
# "next" #3): x-slabs are imbalanced when layer-2 cells cluster at an
# interface.  Every rank lists its layer-2 cells; a deterministic plan (from
# the all-gathered counts) moves the excess of over-loaded ranks to
# under-loaded ones with one all-to-all of f blocks, each rank evaluates the
# operator on a dense batch, and a second all-to-all returns the results to
# the owners.  Per-cell operators are independent and deterministic, so the
# result is bitwise the owner's local evaluation.
# ---------------------------------------------------------------------------
def balance_plan(counts):
    """counts[r] = layer-2 cells on rank r -> send[r][s] = cells r ships to s.
    Targets differ by at most one; ranks keep their own cells first; surplus
    goes to deficits in rank order (identical on every rank)."""
    world = len(counts)
    total = sum(counts)
    target = [total // world + (1 if r < total % world else 0) for r in range(world)]
    send = [[0] * world for _ in range(world)]
    surplus = [max(0, counts[r] - target[r]) for r in range(world)]
    deficit = [max(0, target[r] - counts[r]) for r in range(world)]
    s = 0
    for r in range(world):
        while surplus[r] > 0:
            while deficit[s] == 0:
                s += 1
            m = min(surplus[r], deficit[s])
            send[r][s] += m
            surplus[r] -= m
            deficit[s] -= m
    return send


def balanced_apply(local: torch.Tensor, cells: torch.Tensor, fn, group=None):
    """out[cells] = fn(local[cells]) with the work of all ranks' `cells` spread
    evenly: `local` [n_local, nb] (this rank's slab), `cells` int64 indices
    into it, `fn` a per-cell batch operator ([m, nb] -> [m, nb], e.g.
    spectral_collision).  Returns (out rows for `cells`, plan)."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    if world == 1:
        return fn(local[cells]), [[len(cells)]]
    rank = dist.get_rank(group)
    counts = [None] * world
    dist.all_gather_object(counts, int(len(cells)), group=group)
    send = balance_plan(counts)
    keep = counts[rank] - sum(send[rank])
    # rows shipped: the tail of my list, in destination-rank order
    out_split = [send[rank][s] for s in range(world)]
    in_split = [send[s][rank] for s in range(world)]
    nb = local.shape[1]
    if local.is_cuda and len(cells):
        from .kinetic import gather_cells
        batch = gather_cells(local, cells)
    else:
        batch = local[cells]
    host_stage = local.is_cuda and dist.get_backend(group) == "gloo"  # gloo moves host tensors only (tests)

    def a2a(out, inp, osplit, isplit):
        if host_stage:
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), osplit, isplit, group=group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, osplit, isplit, group=group)

    ship = batch[keep:].contiguous()
    recv = torch.empty((sum(in_split), nb), dtype=local.dtype, device=local.device)
    a2a(recv, ship, in_split, out_split)
    work = torch.cat([batch[:keep], recv]) if recv.numel() else batch[:keep]
    res = fn(work)
    back = torch.empty((sum(out_split), nb), dtype=local.dtype, device=local.device)
    a2a(back, res[keep:].contiguous(), out_split, in_split)
    return torch.cat([res[:keep], back]), send


def balanced_residual(kernel, y: torch.Tensor, res: torch.Tensor, status: torch.Tensor, pen_coeff: float = 6.283185307179586,
                      exact: bool = False, group=None):
    """res = penalized_residual(y) for this rank's layer-2 batch y [m, n^3], the
    work of all ranks' batches spread evenly (balance_plan): the first `keep`
    rows are evaluated here straight into res, the surplus rows go out in one
    all-to-all, the received rows are evaluated as one dense batch and their
    results come back in a second all-to-all (into res[keep:]).  Statuses of
    shipped rows are evaluated by the receiving rank, which raises on failure.
    Returns the plan.  Collective: every rank calls it, also with m = 0."""
    from .kinetic import penalized_residual_rows

    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    m = y.shape[0]
    if world == 1:
        penalized_residual_rows(kernel, y, pen_coeff, exact, out=res, status=status)
        return [[m]]
    rank = dist.get_rank(group)
    counts = [None] * world
    dist.all_gather_object(counts, int(m), group=group)
    send = balance_plan(counts)
    keep = counts[rank] - sum(send[rank])
    out_split = [send[rank][s] for s in range(world)]
    in_split = [send[s][rank] for s in range(world)]
    nb = kernel.modes()
    host_stage = y.is_cuda and dist.get_backend(group) == "gloo"

    def a2a(out, inp, osplit, isplit):
        if not sum(osplit) and not sum(isplit):
            return
        if host_stage:
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), osplit, isplit, group=group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, osplit, isplit, group=group)

    dev = kernel_device(kernel, y)
    recv = torch.empty((sum(in_split), nb), dtype=torch.float64, device=dev)
    a2a(recv, y[keep:], in_split, out_split)
    if keep:
        penalized_residual_rows(kernel, y[:keep], pen_coeff, exact, out=res[:keep], status=status[:keep])
    back, back_st = penalized_residual_rows(kernel, recv, pen_coeff, exact)
    a2a(res[keep:], back, out_split, in_split)
    st_back = torch.empty(m - keep, dtype=torch.float64, device=dev)  # the evaluating ranks' statuses
    a2a(st_back.view(-1, 1), back_st.to(torch.float64).view(-1, 1), out_split, in_split)
    if m > keep:
        status[keep:].copy_(st_back.to(torch.int32))
    return send


def kernel_device(kernel, like: torch.Tensor):
    return like.device if like.numel() else torch.device("cuda", kernel.ctx.device)
