"""Distribution of the per-cell Nyquist bound (config-2 batch) and how many
cells each guard threshold would reroute."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs
vg = hk.make_velocity_grid(32, inputs.VMAX)
k = hk.precompute_kernel(vg, 32, 8, 8, inputs.R_PHYS_MAX)
f = inputs.config2_cells_torch(4096, 32)
q, st = hk.spectral_collision(f, k, return_status=True)
b = st["nyq_bound"]
print("percentiles", {p: float(np.percentile(b, p)) for p in (50, 90, 99, 99.9)}, "max", float(b.max()))
for tau in (1e-12, 1e-11, 2e-11, 5e-11):
    print(tau, int((b > tau).sum()))
# actual error of the fast path on the worst cells vs the exact kernel
worst = np.argsort(-b)[:8]
fw = f[torch.from_numpy(worst).cuda()]
qf = hk.spectral_collision(fw, k, guard=False).cpu().numpy()
qe = hk.spectral_collision(fw, k, exact=True).cpu().numpy()
for i, c in enumerate(worst):
    print(int(c), float(b[c]), float(np.linalg.norm(qf[i] - qe[i]) / np.linalg.norm(qe[i])))
