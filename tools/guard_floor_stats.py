"""Per-cell scales behind the Nyquist guard at N = 64 (config 5): ||Q||, the loss
term's scale ||jac f L||, the rigorous bound and the actual fast-vs-exact gap."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
vg = hk.make_velocity_grid(n, inputs.VMAX)
k = hk.precompute_kernel(vg, n, 8, 8, inputs.R_PHYS_MAX)
cols = [0, 1, 100, 200, 240, 250, 255, 256, 260, 270, 300, 400, 510, 511]
f = torch.from_numpy(inputs.config5_cells(len(cols), n, columns=cols)).cuda()
qn, st = hk.spectral_collision(f, k, guard=False, return_status=True)
qe = hk.spectral_collision(f, k, exact=True)
qn, qe = qn.cpu().numpy(), qe.cpu().numpy()
for c, col in enumerate(cols):
    qnorm = float(np.linalg.norm(qe[c]))
    lnorm = float(np.sqrt(st["loss_norm2"][c]))
    gap = float(np.linalg.norm(qn[c] - qe[c]))
    print(json.dumps({"col": col, "q": qnorm, "loss": lnorm, "q_over_loss": qnorm / lnorm,
                      "bound_abs": float(st["nyq_bound"][c]) * float(np.sqrt(st["q_norm2"][c])),
                      "gap": gap, "gap_over_q": gap / qnorm, "gap_over_loss": gap / lnorm}))
