"""Dynamic load balancing of layer-2 cells (partition.balanced_apply) on CPU
with gloo: the plan is balanced and the result is bitwise the owners' local
evaluation (the operator here is the CPU oracle's collision, world 2 and 3)."""
import os
import socket

import numpy as np
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


def test_balance_plan_properties():
    from paper_2505_03360_b200.partition import balance_plan
    for counts in ([10, 0, 0], [3, 3, 3], [0, 7, 1, 0], [100, 1, 50, 2, 0], [0, 0]):
        send = balance_plan(counts)
        w = len(counts)
        final = [counts[r] - sum(send[r]) + sum(send[s][r] for s in range(w)) for r in range(w)]
        assert sum(final) == sum(counts) and max(final) - min(final) <= 1
        assert all(send[r][r] == 0 for r in range(w))
        # only over-loaded ranks send, only under-loaded ranks receive
        for r in range(w):
            assert not (sum(send[r]) and sum(send[s][r] for s in range(w)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2505_03360_b200 import inputs
        from paper_2505_03360_b200.partition import balanced_apply
        o = Oracle()
        k = o.kernel(8, inputs.VMAX, 2, 2, inputs.R_PHYS_MAX, closed_form=True)

        def fn(batch):
            q, _, _ = o.collision_batch(k, batch.numpy(), nthreads=1)
            return torch.from_numpy(q)

        nloc = 6
        local = torch.from_numpy(inputs.config1_cells(nloc, 8, seed_salt=rank))
        # clustered layer-2 cells: rank 0 holds most of them
        cells = torch.arange(nloc) if rank == 0 else torch.tensor([1]) if rank == 1 else torch.tensor([], dtype=torch.int64)
        out, plan = balanced_apply(local, cells, fn)
        ref = fn(local[cells]) if len(cells) else torch.empty((0, 512), dtype=torch.float64)
        ok = torch.equal(out, ref)
        q.put((rank, ok, plan))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_balanced_apply_equals_local(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    plan = res[0][2]
    assert sum(plan[0]) > 0  # rank 0 shipped cells away
