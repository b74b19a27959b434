import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic
nx = ny = 200
ud = torch.from_numpy(inputs.config4_conserved(nx, ny)).cuda()
dx = 1.0 / nx
x = (np.arange(nx) + 0.5) * dx
near = lambda z: (np.abs(z - 0.5) < 0.025) | (z < 0.025) | (z > 1 - 0.025)
X, Y = np.meshgrid(x, x)
band = np.flatnonzero((near(X) | near(Y)).ravel())
vg = hk.make_velocity_grid(32, inputs.VMAX)
k = hk.precompute_kernel(vg, 32, 4, 8, inputs.R_PHYS_MAX)
f = kinetic.conserved_to_maxwellian(ud, vg)
f += 0.05 * torch.roll(f, 1, 0)
g = kinetic.gather_cells(f, torch.from_numpy(band).cuda())
ctx = hk.default_context()
for guard in (True, False):
    for _ in range(2): hk.spectral_collision(g, k, guard=guard)
    torch.cuda.synchronize()
    ctx._lib.hk_ctx_set_timing(ctx.h, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): q, st = hk.spectral_collision(g, k, guard=guard, return_status=True)
    e1.record(); torch.cuda.synchronize()
    res = {}
    for tag in (0, 1, 2):
        t, n = C.c_double(0), C.c_int64(0)
        ctx._lib.hk_ctx_timing_report(ctx.h, tag, C.byref(t), C.byref(n)); res[tag] = t.value / max(n.value, 1)
    ctx._lib.hk_ctx_set_timing(ctx.h, 0)
    print("guard", guard, "ms", e0.elapsed_time(e1) / 3, "main", res[0], "guard", res[1], "fix", res[2], "listed", int(((st["flags"] & 4) != 0).sum()), "of", len(band))
idx = torch.from_numpy(band).cuda()
for name, fn in (("gather", lambda: kinetic.gather_cells(f, idx)), ("scatter", lambda: kinetic.scatter_cells(g, idx, f))):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, "ms", e0.elapsed_time(e1) / 3, "GB/s", 2 * g.numel() * 8 / (e0.elapsed_time(e1) / 3 * 1e-3) / 1e9)
