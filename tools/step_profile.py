import sys, os, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic
nx = ny = 256
vg = hk.make_velocity_grid(32, inputs.VMAX)
f, _ = inputs.config3_cells_torch(nx, ny, 32)
eps = torch.full((nx * ny,), 1e-2, dtype=torch.float64, device="cuda")
for _ in range(2):
    kinetic.esbgk_imex_step(f, nx, ny, vg, 1.0 / nx, 1.0 / ny, 1e-3, eps)
torch.cuda.synchronize()
print("ok")
