"""Config-4 hybrid step: device time of the collision kernels, the Nyquist guard
and the exact Nyquist correction per step (hk_ctx_set_timing tags 0 / 1 / 2)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic

nx = ny = 200
n = 32
vg = hk.make_velocity_grid(n, inputs.VMAX)
k = hk.precompute_kernel(vg, n, 4, 8, inputs.R_PHYS_MAX)
hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n)
rd, hd, fd, ed = (torch.from_numpy(x.copy()).cuda() for x in (r, hydro, f, eps))
dx = 1.0 / nx
dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
for _ in range(3):
    kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, rd, hd, fd)
torch.cuda.synchronize()
ctx = k.ctx
lib = ctx._lib
lib.hk_ctx_set_timing(ctx.h, 1)
steps = 4
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, rd, hd, fd)
e1.record()
torch.cuda.synchronize()
out = {"step_ms": e0.elapsed_time(e1) / steps}
for tag, name in ((0, "collision"), (1, "guard"), (2, "nyquist_correction")):
    ms, nl = C.c_double(), C.c_int64()
    lib.hk_ctx_timing_report(ctx.h, tag, C.byref(ms), C.byref(nl))
    out[name + "_ms_per_step"] = ms.value / steps
lib.hk_ctx_set_timing(ctx.h, 0)
print(out)
