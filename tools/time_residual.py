"""Times the penalized residual's epilogue (moment matching + invariant removal,
residual_finish) on config-3 / config-4-like cells: the residual batch minus
the collision batch of the same cells; one JSON line."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=2048)
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--tag", default="")
a = ap.parse_args()
vg = hk.make_velocity_grid(a.n, inputs.VMAX)
k = hk.precompute_kernel(vg, a.n, 4, 8, inputs.R_PHYS_MAX)
side = int(a.cells ** 0.5)
f, _ = inputs.config3_cells_torch(side, a.cells // side, a.n)
out = torch.empty_like(f)
st = torch.empty(f.shape[0], dtype=torch.int32, device="cuda")
ctx = k.ctx


def run(res):
    if res:
        kinetic.penalized_residual_rows(k, f, out=out, status=st)
    else:
        hk.spectral_collision(f, k, out=out)


def t(res, it=5):
    run(res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        run(res)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


tr, tc = t(True), t(False)
gb = 6 * f.numel() * 8 / 1e9
print(json.dumps({"tag": a.tag, "cells": f.shape[0], "n": a.n, "residual_ms": tr, "collision_ms": tc,
                  "finish_ms": tr - tc, "finish_GBps_at_6_passes": gb / ((tr - tc) * 1e-3)}))
