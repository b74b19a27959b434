"""Worker of tests/test_gpu_peer_transport.py: one rank of an x-slab
decomposition; the transport reads its neighbours' ghost columns from their
slabs through CUDA IPC (PeerHalo) and must equal the single-domain periodic
transport of the global field.  Exit 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import kinetic, partition

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")  # host-side plumbing only (handles, barriers)
torch.cuda.set_device(0)
n, nx, ny = 8, 10, 6
vg = hk.make_velocity_grid(n, 8.0)
rng = np.random.default_rng(11)
glob = torch.from_numpy(rng.uniform(0.1, 1.0, (nx * ny, n ** 3))).cuda()
part = partition.XSlab(nx, ny, world, rank)
slab = part.scatter(glob)
ctx = hk.Context(0, torch.cuda.current_stream())
peer = partition.PeerHalo(part, slab, ctx)
peer.refresh()
out = torch.empty_like(slab)
peer.transport(out, vg, 1.0 / nx, 1.0 / ny)
peer.done()
ref = part.scatter(kinetic.kinetic_transport_rhs_periodic(glob, nx, ny, vg, 1.0 / nx, 1.0 / ny))
torch.cuda.synchronize()
err = float((out - ref).abs().max() / ref.abs().max())
peer.close()
dist.destroy_process_group()
print(f"rank {rank}: max rel err {err:.3e}", flush=True)
sys.exit(0 if err < 1e-14 else 1)
