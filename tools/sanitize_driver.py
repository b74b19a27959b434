"""Tiny invocations of every device operator for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): `python tools/sanitize_driver.py OP`.
Run by tools/sanitize.sh; summaries land in profiles/r02_sanitizer.txt."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic, partition

op = sys.argv[1]
V = inputs.VMAX
R = inputs.R_PHYS_MAX


def coll(n, a1, a2, f, **kw):
    vg = hk.make_velocity_grid(n, V)
    k = hk.precompute_kernel(vg, n, a1, a2, R)
    q = hk.spectral_collision(torch.from_numpy(f).cuda(), k, **kw)
    torch.cuda.synchronize()
    return q


if op == "coll16":  # N = 16 exact (cell halves over persistent CTAs)
    coll(16, 4, 8, inputs.config1_cells(2, 16))
elif op == "coll32":  # N = 32 fast 12-warp team kernel + guard + Nyquist correction (listed cells present)
    f = np.concatenate([inputs.config2_cells(3, 32), inputs.config5_cells(3, 32, columns=[300, 400, 511])])
    coll(32, 8, 8, f)
elif op == "coll32x":  # N = 32 exact cluster kernel
    coll(32, 8, 8, inputs.config2_cells(2, 32), exact=True)
elif op == "coll64":  # N = 64 fast team kernel (TMA weights) + guard + correction
    coll(64, 8, 8, inputs.config5_cells(2, 64, columns=[256, 511]))
elif op == "coll64x":  # N = 64 exact
    coll(64, 2, 4, inputs.config5_cells(1, 64, columns=[256]), exact=True)
elif op == "host32":  # streamed host entry point (pinned) at its smallest size
    vg = hk.make_velocity_grid(32, V)
    k = hk.precompute_kernel(vg, 32, 4, 4, R)
    f = inputs.config2_cells_torch(256, 32, device="cuda").cpu().pin_memory()
    q = torch.empty_like(f).pin_memory()
    hk.spectral_collision(f.numpy(), k, out=q.numpy())
elif op == "cells":  # moments, stage solves, residual finish, moment operators
    n = 32
    vg = hk.make_velocity_grid(n, V)
    f, _ = inputs.config3_cells(4, 2, n)
    fd = torch.from_numpy(f).cuda()
    out = kinetic.moments_of(fd, vg, sigma=True, realizability=True, l1=True)
    kinetic.esbgk_stage_solve(fd, 1e-3, 1e-2, kinetic.EsbgkParams(), vg)
    kinetic.penalized_stage_solve(fd, 1e-3, 1e-2, kinetic.PenalizationRule(), vg)
    k = hk.precompute_kernel(vg, n, 4, 4, R)
    kinetic.penalized_residual(fd, k, vg)
    mom = out["moments"]
    th = torch.eye(3, dtype=torch.float64, device="cuda").expand(8, 3, 3).contiguous()
    g, _ = kinetic.anisotropic_gaussian(mom, th, -0.5, vg)
    E = 0.5 * mom[:, 0] * (mom[:, 1:4] ** 2).sum(1) + 1.5 * mom[:, 0] * mom[:, 4]
    kinetic.match_moments(g, vg, torch.cat([mom[:, :1], mom[:, :1] * mom[:, 1:4], E[:, None]], 1))
    kinetic.remove_invariant_moments(fd - g, g, vg, mom[:, 1:4])
    torch.cuda.synchronize()
elif op == "steps":  # transport, classifier, both PR(2,2,2) steps
    n, nx, ny = 16, 5, 4
    vg = hk.make_velocity_grid(n, V)
    f, _ = inputs.config3_cells(nx, ny, n)
    fd = torch.from_numpy(f).cuda()
    eps = torch.full((nx * ny,), 1e-2, dtype=torch.float64, device="cuda")
    kinetic.kinetic_transport_rhs_periodic(fd, nx, ny, vg, 0.1, 0.1)
    out = kinetic.moments_of(fd, vg, l1=True)
    kinetic.classify(out["moments"], nx, ny, 0.1, 0.1, eps, torch.ones(nx * ny, dtype=torch.int8), l1=out["l1"])
    kinetic.esbgk_imex_step(fd.clone(), nx, ny, vg, 0.1, 0.1, 1e-3, eps)
    k = hk.precompute_kernel(vg, n, 2, 4, R)
    kinetic.penalized_imex_step(fd.clone(), nx, ny, k, 0.1, 0.1, 1e-3, eps)
    part = partition.XSlab(nx, ny, 1, 0)
    partition.penalized_imex_step_slab(part, fd.clone(), k, 0.1, 0.1, 1e-3, eps)
    torch.cuda.synchronize()
elif op == "hybrid":  # Algorithm 1 + transitions + Euler + both kinetic layers
    nx, ny, n = 8, 6, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    vg = hk.make_velocity_grid(n, V)
    k = hk.precompute_kernel(vg, n, 4, 4, R)
    rd, hd, fd, ed = (torch.from_numpy(x.copy()).cuda() for x in (r, hydro, f, eps))
    for _ in range(2):
        kinetic.hybrid_step(k, nx, ny, 1 / nx, 1 / ny, 2e-3, ed, rd, hd, fd)
    torch.cuda.synchronize()
else:
    raise SystemExit(f"unknown op {op}")
print(f"sanitize {op}: ok", flush=True)
