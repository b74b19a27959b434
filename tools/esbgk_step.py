"""Config-3 ES-BGK timing probe (256 x 256 cells, 32^3): `stage` times the
batched stage solve, `step` the PR(2,2,2) step with its per-part times
(hk_ctx_set_timing tags 10..13).  Used by tools/refresh_round.sh for the
ncu captures of the stage and transport kernels."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic
nx = ny = 256; n = 32
vg = hk.make_velocity_grid(n, inputs.VMAX)
f, fl = inputs.config3_cells_torch(nx, ny, n)
cells = nx * ny
eps = torch.full((cells,), 1e-2, dtype=torch.float64, device="cuda")
what = sys.argv[1] if len(sys.argv) > 1 else "step"
def step(): kinetic.esbgk_imex_step(f, nx, ny, vg, 1.0 / nx, 1.0 / ny, 1e-3, eps)
def stage(): kinetic.esbgk_stage_solve(f, 1e-3, eps, kinetic.EsbgkParams(), vg, check=False)
fn = step if what == "step" else stage
for _ in range(3): fn()
torch.cuda.synchronize()
import ctypes as C
ctx = hk.default_context(0); lib = ctx._lib
lib.hk_ctx_set_timing(ctx.h, 1)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): fn()
e1.record(); torch.cuda.synchronize()
print(what, "ms", e0.elapsed_time(e1) / 5, flush=True)
for tag in (10, 11, 12, 13, 0, 1, 2):
    ms = C.c_double(); nl = C.c_int64()
    lib.hk_ctx_timing_report(ctx.h, tag, C.byref(ms), C.byref(nl))
    if nl.value: print("tag", tag, "ms/launch", ms.value / nl.value, "launches", nl.value)
