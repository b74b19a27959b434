"""Worker of tests/test_gpu_balance.py: one x-slab rank of config 4's hybrid
step (N = 16, layer-2 band on two of the slabs); the layer-2 residuals are
spread over the ranks by partition.balanced_apply through hk_hybrid_step's
residual hook.  The balanced step must equal the unbalanced one bitwise and
must have moved cells.  Exit 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic
from paper_2505_03360_b200.partition import HYB_GHOST as W, XSlab, balanced_residual, hybrid_step_slab

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")  # the balanced exchange is staged through host memory on gloo
torch.cuda.set_device(0)
nx, ny, n = 11 * world, 6, 16
hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
right = (torch.arange(nx * ny) % nx >= nx // 2).numpy()  # layer 2 only in the left half: imbalanced slabs
r[right] = 0
f[right] = 0.0
ctx = hk.Context(0, torch.cuda.current_stream())
vg = hk.make_velocity_grid(n, inputs.VMAX)
kern = hk.precompute_kernel(vg, n, 4, 4, inputs.R_PHYS_MAX, ctx=ctx)
dx, dy = 1.0 / nx, 1.0 / ny
dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
glob = [torch.from_numpy(x.copy()).cuda() for x in (r, eps, hydro, f)]
part = XSlab(nx, ny, world, rank)


def halos_of(fields_global):
    out = []
    for t in fields_global:
        g = t.view(ny, nx, -1)
        cols_l = [(part.i0 - W + c) % nx for c in range(W)]
        cols_r = [(part.i0 + part.nxl + c) % nx for c in range(W)]
        out.append((g[:, cols_l].contiguous(), g[:, cols_r].contiguous()))
    return out


def run(balance):
    loc = [part.scatter(t.view(nx * ny, -1)) for t in glob]
    plans = []

    def hook(y, res, status):
        plans.append(balanced_residual(kern, y, res, status))

    rl, el, hl, fl = loc
    counts = hybrid_step_slab(part, kern, dx, dy, dt, el.view(-1), rl.view(-1), hl, fl, halos=halos_of(glob),
                              residual_hook=hook if balance else None)
    torch.cuda.synchronize()
    return loc, counts, plans


a, ca, _ = run(False)
b, cb, plans = run(True)
same = all(torch.equal(x, y) for x, y in zip(a, b)) and torch.equal(ca, cb)
moved = sum(sum(row[s] for s in range(world) if s != q) for plan in plans for q, row in enumerate(plan))
dist.destroy_process_group()
print(f"rank {rank}/{world}: bitwise {same}, residual calls {len(plans)}, cells moved {moved}", flush=True)
sys.exit(0 if same and len(plans) == 2 and (world == 1 or moved > 0) else 1)
