"""Config-5 Q on three x-slabs of the 512 x 128 shock (i0 = 0, 224, 448): time and
number of guard-listed cells per slab (the per-rank work spread of the weak-scaling run)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs
n = 64
vg = hk.make_velocity_grid(n, inputs.VMAX)
k = hk.precompute_kernel(vg, n, 8, 8, inputs.R_PHYS_MAX)
slabs = [int(a) for a in sys.argv[1:]] or [0, 224, 448]
out = {}
for i0 in slabs:
    f = inputs.config5_slab_torch(i0, 64, 128, n)
    q = torch.empty_like(f)
    hk.spectral_collision(f, k, out=q)
    torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); _, st = hk.spectral_collision(f, k, out=q, return_status=True); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out[i0] = {"ms": min(ts), "listed": int(((st["flags"] & 4) != 0).sum())}
    del f, q
    torch.cuda.empty_cache()
print(json.dumps(out))
