"""Worker of tests/test_gpu_peer_imex.py: one rank of an x-slab decomposition
running the penalized PR(2,2,2) step (src/boltzmann.cpp:47-110) with the
transport reading the neighbours' stage field through CUDA IPC (PeerHalo).
Its slab must equal, bitwise, the same rank's columns of the world-1 slab step
of the global field, and the single-GPU device step to 1e-13.  Exit 0 on
success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic, partition

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")  # host-side plumbing only (IPC handles, barriers)
torch.cuda.set_device(0)
n, ny = 16, 4
nx = 3 * world + 1  # uneven slabs (the last ranks get one column fewer)
dx, dy, dt = 1.0 / nx, 1.0 / ny, 1e-3
f0, _ = inputs.config3_cells(nx, ny, n)
eps = torch.tensor([1e-2, 1e-1, 1.0, 3e-2] * nx, dtype=torch.float64)[: nx * ny].cuda()
ctx = hk.Context(0, torch.cuda.current_stream())
vg = hk.make_velocity_grid(n, inputs.VMAX)
kern = hk.precompute_kernel(vg, n, 2, 4, inputs.R_PHYS_MAX, ctx=ctx)
glob = torch.from_numpy(f0.copy()).cuda()


def slab_steps(part, f, eps_l, steps=2):
    work = torch.empty((6, part.cells, n ** 3), dtype=torch.float64, device="cuda")
    peer = partition.PeerHalo(part, work[0], ctx)
    for _ in range(steps):
        partition.penalized_imex_step_slab(part, f, kern, dx, dy, dt, eps_l, work=work, peer=peer)
    torch.cuda.synchronize()
    peer.close()
    return f


part = partition.XSlab(nx, ny, world, rank)
eps_l = part.scatter(eps.view(-1, 1)).view(-1)
mine = slab_steps(part, part.scatter(glob).clone(), eps_l)
one = partition.XSlab(nx, ny, 1, 0)
ref = part.scatter(slab_steps(one, glob.clone(), eps))
dev = glob.clone()
for _ in range(2):
    kinetic.penalized_imex_step(dev, nx, ny, kern, dx, dy, dt, eps)
dev = part.scatter(dev)
torch.cuda.synchronize()
bitwise = bool(torch.equal(mine, ref))
err = float((mine - dev).abs().max() / dev.abs().max())
dist.destroy_process_group()
print(f"rank {rank}/{world}: slab columns {part.i0}..{part.i0 + part.nxl - 1}, bitwise vs world-1 {bitwise}, "
      f"vs single-GPU step {err:.2e}", flush=True)
sys.exit(0 if bitwise and err < 1e-13 else 1)
