"""Small driver for ncu captures of the collision kernels (config-2 shapes)."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=1024)
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--a1", type=int, default=8)
ap.add_argument("--a2", type=int, default=8)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--exact", action="store_true")
args = ap.parse_args()

vg = hk.make_velocity_grid(args.n, 8.0)
kern = hk.precompute_kernel(vg, args.n, args.a1, args.a2, inputs.R_PHYS_MAX)
if args.n == 32:
    f = inputs.config2_cells_torch(args.cells, 32, device="cuda")
elif args.n == 64:
    f = torch.from_numpy(inputs.config5_cells(args.cells, 64)).cuda()
else:
    f = torch.from_numpy(inputs.config1_cells(args.cells, args.n)).cuda()
q = torch.empty_like(f)
for _ in range(args.iters):
    hk.spectral_collision(f, kern, out=q, exact=args.exact)
torch.cuda.synchronize()
print("ok", float(q.abs().max()))
