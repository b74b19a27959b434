"""Measures the non-headline BASELINE configs on one B200 (JSON lines).

config 1: 64 homogeneous cells, 16^3, M = 4x8 (hard spheres; the reference has
          no 3-D Maxwell-molecule kernel), Q + forward Euler f + 0.01 Q.
config 3: 256 x 256 cells, 32^3: moments + realizability + L1 (classifier
          inputs), Algorithm-1 classification, ES-BGK stage (a = dt = 1e-3,
          eps = 1e-2, beta = -1/2, nu = pi/2 rho).  HBM-bound: achieved GB/s on
          algorithmic bytes (f read once per kernel, stage output written once).
Times are CUDA events on the launching stream, warm, median of `--iters`.
"""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs, kinetic

HBM = 6537.0  # GB/s, MEASURED_PEAKS.json


def timed(fn, iters):
    ts = []
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def config1(iters):
    n, a1, a2, cells = 16, 4, 8, 64
    ctx = hk.default_context()
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    f = torch.from_numpy(inputs.config1_cells(cells, n)).cuda()
    q = torch.empty_like(f)
    f1 = torch.empty_like(f)

    def step():
        hk.spectral_collision(f, k, out=q)
        ctx._lib.hk_axpby(ctx.h, f.numel(), f1.data_ptr(), f.data_ptr(), 0.01, q.data_ptr(), 0.0, None)

    def steps():  # back-to-back steps (as bench.py times its K steps): the launches of step s + 1
        for _ in range(20):  # are queued while step s runs, so host gaps do not enter the device time
            step()

    ms = timed(steps, iters) / 20
    md = (a1 - 1) * a2 + 1
    W = (2 * md + 2) * 5 * n ** 3 * math.log2(n ** 3) + (12 * md + 10) * n ** 3
    peak = ctx.fp64_peak_tflops()
    ach = W * cells / (ms * 1e-3) / 1e12
    return {"config": "config1: 64 cells, 16^3, M=4x8, hard spheres, Q + forward Euler dt=0.01",
            "path": "exact kernel (a cell's items in two fixed halves over one persistent CTA per SM, 16^3 spectrum in shared memory, Q = jac Re(U0 + U1))",
            "ms_per_step": ms, "cell_updates_per_s": cells / (ms * 1e-3),
            "roofline": {"bound": "fp64", "achieved_tflops": ach, "peak_tflops": peak, "frac": ach / peak,
                         "note": "64 cells = 128 halves of 13 items on 148 SMs; 8 warps per SM, barrier-phased shared-memory passes"}}


def config3(iters, nx=256, ny=256):
    n = 32
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    f, fl = inputs.config3_cells_torch(nx, ny, n)
    cells = nx * ny
    eps = torch.full((cells,), 1e-2, dtype=torch.float64, device="cuda")
    r_in = torch.ones(cells, dtype=torch.int8, device="cuda")
    th = kinetic.Thresholds(eta0=1e-3, eta1=1e-2, delta0=1e-3)
    res = {}

    def mom():
        res["m"] = kinetic.moments_of(f, vg, realizability=True, l1=True, check=False)

    def cls():
        res["c"] = kinetic.classify(res["m"]["moments"], nx, ny, 1.0 / nx, 1.0 / ny, eps, r_in, th, l1=res["m"]["l1"])

    def es():
        res["e"] = kinetic.esbgk_stage_solve(f, 1e-3, eps, kinetic.EsbgkParams(), vg, check=False)

    def tr():
        res["t"] = kinetic.kinetic_transport_rhs_periodic(f, nx, ny, vg, 1.0 / nx, 1.0 / ny)

    t_m = timed(mom, iters)
    t_c = timed(cls, iters)
    t_e = timed(es, iters)
    del res["e"]
    t_t = timed(tr, iters)
    del res["t"]
    torch.cuda.empty_cache()

    def step():  # one ES-BGK PR(2,2,2) step of the whole field (src/esbgk.cpp:47-99), in place
        kinetic.esbgk_imex_step(f, nx, ny, vg, 1.0 / nx, 1.0 / ny, 1e-3, eps)

    t_s = timed(step, max(1, iters // 2))
    # per-part times of the step (hk_ctx_set_timing tags 10..13, CUDA events on the context stream)
    import ctypes as _C
    ctx = hk.default_context()
    ctx._lib.hk_ctx_set_timing(ctx.h, 1)
    step()
    torch.cuda.synchronize()
    parts = {}
    for tag, name in ((10, "stage1"), (11, "transport_Y1_to_facc_G"), (12, "stage2"), (13, "transport_Y2_final")):
        ms_, nl = _C.c_double(), _C.c_int64()
        ctx._lib.hk_ctx_timing_report(ctx.h, tag, _C.byref(ms_), _C.byref(nl))
        parts[name] = ms_.value / max(1, nl.value)
    ctx._lib.hk_ctx_set_timing(ctx.h, 0)
    b_read = cells * n ** 3 * 8
    layers = [int((res["c"][0] == k).sum()) for k in range(3)]
    out = {"config": "config3: 256x256 cells, 32^3, classify + ES-BGK stage (a=dt=1e-3, eps=1e-2, Pr=2/3)",
           "ms": {"moments_realizability_l1": t_m, "classify": t_c, "esbgk_stage": t_e, "transport_rhs": t_t,
                  "esbgk_imex_step": t_s},
           "esbgk_step_parts_ms": parts,
           "ms_per_step": t_m + t_c + t_e, "cell_steps_per_s": cells / ((t_m + t_c + t_e) * 1e-3),
           "layers_after_classify": layers,
           "roofline": {"bound": "hbm", "peak_gbs": HBM,
                        "moments_gbs": b_read / (t_m * 1e-3) / 1e9, "moments_frac": b_read / (t_m * 1e-3) / 1e9 / HBM,
                        "esbgk_gbs": 2 * b_read / (t_e * 1e-3) / 1e9, "esbgk_frac": 2 * b_read / (t_e * 1e-3) / 1e9 / HBM,
                        "transport_gbs": 2 * b_read / (t_t * 1e-3) / 1e9,
                        "transport_frac": 2 * b_read / (t_t * 1e-3) / 1e9 / HBM,
                        "note": "algorithmic bytes: f read once (moments), f read + stage written (ES-BGK); the "
                                "kernels re-read f (realizability/L1 pass, Gaussian coupling pass) from L2/HBM"}}
    return out


def config4(iters):  # pieces; config4_hybrid runs the full step
    """Config 4 pieces on one GPU: the layer-0 Euler TVD-RK2 step on the
    200 x 200 quadrant field, and Q (N = 32, M = 4 x 8) for the ~19 % band
    cells (eps = 0.1 within 0.025 of x = 0.5, y = 0.5 and the periodic wrap
    lines) gathered into a dense batch, the Boltzmann part of a hybrid step."""
    nx = ny = 200
    ud = torch.from_numpy(inputs.config4_conserved(nx, ny)).cuda()
    dx = 1.0 / nx

    def eul():
        kinetic.tvd_rk2_step_periodic(ud, nx, ny, dx, dx, 0.1 * dx)

    t_e = timed(eul, iters)
    x = (np.arange(nx) + 0.5) * dx
    near = lambda z: (np.abs(z - 0.5) < 0.025) | (z < 0.025) | (z > 1 - 0.025)
    X, Y = np.meshgrid(x, x)
    band = np.flatnonzero((near(X) | near(Y)).ravel())
    n, a1, a2 = 32, 4, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    f = kinetic.conserved_to_maxwellian(ud, vg)  # layer 0 -> 1 for every cell
    f += 0.05 * torch.roll(f, 1, 0)  # non-equilibrium band content
    idx = torch.from_numpy(band).cuda()
    g = kinetic.gather_cells(f, idx)
    q = torch.empty_like(g)

    t_g = timed(lambda: kinetic.gather_cells(f, idx), iters)
    t_c = timed(lambda: hk.spectral_collision(g, k, out=q), iters)
    t_s = timed(lambda: kinetic.scatter_cells(q, idx, f), iters)
    t_q = t_g + t_c + t_s
    md = (a1 - 1) * a2 + 1
    W = (2 * md + 2) * 5 * n ** 3 * math.log2(n ** 3) + (12 * md + 10) * n ** 3
    ach = W * len(band) / (t_q * 1e-3) / 1e12
    return {"config": "config4: 200x200 quadrant Riemann problem; Euler layer on all cells, Boltzmann Q (N=32, M=4x8) "
                      "on the eps band", "band_cells": int(len(band)),
            "ms": {"euler_tvd_rk2_step": t_e, "band_gather": t_g, "band_collision": t_c, "band_scatter": t_s,
                   "band_collision_gather_scatter": t_q},
            "euler_cell_steps_per_s": nx * ny / (t_e * 1e-3), "band_cell_updates_per_s": len(band) / (t_q * 1e-3),
            "roofline": {"bound": "fp64", "collision_achieved_tflops": ach,
                         "collision_frac": ach / hk.default_context().fp64_peak_tflops()}}


def config4_hybrid(steps=20, full_sample=True):
    """Config 4 end to end: `steps` hybrid steps (hk_hybrid_step: Algorithm 1,
    transitions, Euler TVD-RK2 on layer 0, PR(2,2,2) ES-BGK / penalized
    Boltzmann on layers 1 / 2 with the cross-layer transport halo) of the
    200 x 200 quadrant Riemann problem, N = 32, M = 4 x 8, CFL 0.5, band in
    layer 2 at t = 0.  With `full_sample`, one all-Boltzmann step of the same
    field (every cell layer 2, regimes frozen) gives the paper's
    hybrid / full-kinetic ratio (SPEC.md estimate_full_kinetic_time)."""
    nx = ny = 200
    n, a1, a2 = 32, 4, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    hydro, eps, r, _ = inputs.config4_hybrid_state(nx, ny, n, with_f=False)
    hd = torch.from_numpy(hydro).cuda()
    ed = torch.from_numpy(eps).cuda()
    rd = torch.from_numpy(r).cuda()
    f = kinetic.conserved_to_maxwellian(hd, vg)
    dx = 1.0 / nx
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)  # CFL 0.5 on the fastest node
    p = kinetic.HybridParams()
    # warm-up: the whole run once on copies (the layer-2 batch grows over the steps; its
    # workspaces reach their final size here, not inside the timed run)
    rw, hw, fw = rd.clone(), hd.clone(), f.clone()
    for _ in range(steps):
        kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, rw, hw, fw, p)
    del rw, hw, fw
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hist = []
    e0.record()
    for _ in range(steps):
        hist.append(kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, rd, hd, f, p))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    q_evals = sum(2 * c.layer2 for c in hist)
    out = {"config": "config4: 200x200 quadrant Riemann problem, hybrid steps (Algorithm 1), N=32, M=4x8, CFL 0.5",
           "steps": steps, "ms_total": ms, "ms_per_step": ms / steps,
           "cell_steps_per_s": nx * ny * steps / (ms * 1e-3),
           "boltzmann_cell_updates_per_s": q_evals / (ms * 1e-3),
           "layers_first_step": list(hist[0][:3]), "layers_last_step": list(hist[-1][:3]),
           "transitions_0to1": sum(c.to_kinetic for c in hist), "transitions_1to0": sum(c.to_fluid for c in hist),
           "mean_kinetic_fraction": sum((c.layer1 + c.layer2) / (nx * ny) for c in hist) / steps}
    if full_sample:
        r2 = torch.full_like(rd, 2)
        pf = kinetic.HybridParams(update_regimes=False)
        kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, r2, hd.clone(), f, pf)  # workspaces for 40000 kinetic cells
        torch.cuda.synchronize()
        e0.record()
        kinetic.hybrid_step(k, nx, ny, dx, dx, dt, ed, r2, hd, f, pf)
        e1.record()
        torch.cuda.synchronize()
        full = e0.elapsed_time(e1)
        out["all_boltzmann_ms_per_step"] = full
        out["hybrid_speedup_vs_all_boltzmann"] = full / (ms / steps)
    return out


def config4_slabs(world=8, steps=3, weighted=False):
    """Config 4's hybrid step decomposed into `world` x-slabs (partition.hybrid_step_slab:
    8 exchanged ghost columns per side, residuals only where the interior depends on
    them), the slabs stepped one after another on this GPU with the halos copied
    between them (the exchange an NCCL run would do).  Reports each slab's step time:
    max over slabs ~ the per-GPU step time of a world-GPU run (exchange excluded),
    and the redundant work of the decomposition against the single-GPU step."""
    from paper_2505_03360_b200.partition import HYB_GHOST as W, XSlab, hybrid_step_slab, weighted_bounds
    nx = ny = 200
    n, a1, a2 = 32, 4, 8
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    hydro, eps, r, _ = inputs.config4_hybrid_state(nx, ny, n, with_f=False)
    hd, ed, rd = (torch.from_numpy(x).cuda() for x in (hydro, eps, r))
    f = kinetic.conserved_to_maxwellian(hd, vg)
    dx = 1.0 / nx
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
    bounds = None
    if weighted:  # balance 2 x layer-2 + layer-1 / 10 cells per column (the t = 0 layer map)
        rr = r.reshape(ny, nx)
        bounds = weighted_bounds(2.0 * (rr == 2).sum(0) + 0.1 * (rr == 1).sum(0) + 0.01 * ny, world)
    parts = [XSlab(nx, ny, world, q, bounds) for q in range(world)]
    loc = [[p_.scatter(t.view(nx * ny, -1)) for t in (rd, ed, hd, f)] for p_ in parts]
    del f
    torch.cuda.empty_cache()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in parts]
    per = [[] for _ in parts]
    warm = 2  # warm-up steps: the layer-2 batches grow over the first steps (workspace growth)
    for step in range(steps + warm):
        halos = []
        for q, p_ in enumerate(parts):
            lt, rt = loc[(q - 1) % world], loc[(q + 1) % world]
            lp, rp = parts[(q - 1) % world], parts[(q + 1) % world]
            halos.append([(lt[fi].view(ny, lp.nxl, -1)[:, -W:].contiguous(),
                           rt[fi].view(ny, rp.nxl, -1)[:, :W].contiguous()) for fi in range(4)])
        for q, p_ in enumerate(parts):
            rl, el, hl, fl = loc[q]
            ev[q][0].record()
            hybrid_step_slab(p_, k, dx, dx, dt, el.view(-1), rl.view(-1), hl, fl, halos=halos[q])
            ev[q][1].record()
        torch.cuda.synchronize()
        if step >= warm:
            for q in range(world):
                per[q].append(ev[q][0].elapsed_time(ev[q][1]))
    ms = [sum(v) / len(v) for v in per]
    return {"config": f"config4 on {world} x-slabs (hybrid_step_slab, 8 ghost columns, "
                      f"{'work-weighted' if weighted else 'even'} boundaries), slabs stepped in turn on 1 GPU",
            "slab_columns": [p_.nxl for p_ in parts], "ms_per_slab_step": ms, "max_slab_ms": max(ms),
            "sum_slab_ms": sum(ms),
            "note": "max_slab_ms ~ per-GPU step time of a world-GPU run without the halo exchange; "
                    "sum_slab_ms / single-GPU step = redundant-work factor of the decomposition"}


def config4_slabs_balanced(world=8, steps=3):
    """config4_slabs with the layer-2 residuals load-balanced across the slabs
    (partition.balanced_residual through hk_hybrid_step's residual hook), emulated
    on one GPU: each slab's plain step is timed (T_q), the same steps with a hook
    evaluating the residuals locally give the residual time R_q (CUDA events
    around the evaluation), the balanced per-rank residual batch
    (ceil(total / world) cells per call) is timed on real stage values (R_bal),
    and each slab's balanced step time is T_q - R_q + R_bal + the two
    all-to-alls of the shipped cells at 700 GB/s."""
    import math as _m
    from paper_2505_03360_b200.partition import HYB_GHOST as W, XSlab, hybrid_step_slab
    nx = ny = 200
    n, a1, a2 = 32, 4, 8
    nb = n ** 3
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    hydro, eps, r, _ = inputs.config4_hybrid_state(nx, ny, n, with_f=False)
    hd, ed, rd = (torch.from_numpy(x).cuda() for x in (hydro, eps, r))
    f = kinetic.conserved_to_maxwellian(hd, vg)
    dx = 1.0 / nx
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
    parts = [XSlab(nx, ny, world, q) for q in range(world)]
    loc = [[p_.scatter(t.view(nx * ny, -1)) for t in (rd, ed, hd, f)] for p_ in parts]
    del f
    torch.cuda.empty_cache()
    mode = {"collect": False}
    store = [[None, None] for _ in parts]
    rec = []  # per timed step: [(m, residual ms) per call] per slab

    def make_hook(q, calls):
        def hook(y, res, status):
            kcall = len(calls)
            if mode["collect"]:
                store[q][kcall] = y.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kinetic.penalized_residual_rows(k, y, out=res, status=status)  # in place: no allocation
            e1.record()
            calls.append((y.shape[0], e0, e1))
        return hook

    def step(timed, hooked=True):
        halos = []
        for q, p_ in enumerate(parts):
            lt, rt = loc[(q - 1) % world], loc[(q + 1) % world]
            lp, rp = parts[(q - 1) % world], parts[(q + 1) % world]
            halos.append([(lt[fi].view(ny, lp.nxl, -1)[:, -W:].contiguous(),
                           rt[fi].view(ny, rp.nxl, -1)[:, :W].contiguous()) for fi in range(4)])
        out = []
        for q, p_ in enumerate(parts):
            rl, el, hl, fl = loc[q]
            calls = []
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            hybrid_step_slab(p_, k, dx, dx, dt, el.view(-1), rl.view(-1), hl, fl, halos=halos[q],
                             residual_hook=make_hook(q, calls) if hooked else None)
            s1.record()
            out.append((s0, s1, calls))
        torch.cuda.synchronize()
        if timed and hooked:
            rec.append([(s0.elapsed_time(s1), [(m, e0.elapsed_time(e1)) for m, e0, e1 in calls]) for s0, s1, calls in out])
        if timed and not hooked:
            plain.append([s0.elapsed_time(s1) for s0, s1, _ in out])

    plain = []
    for _ in range(2):
        step(False)
    mode["collect"] = True
    step(False)
    mode["collect"] = False
    for _ in range(steps):  # alternate: plain steps time T_q, hooked steps time the residuals R_q
        step(True, hooked=False)
        step(True, hooked=True)
    T = [sum(plain[t][q] for t in range(steps)) / steps for q in range(world)]
    Rq = [sum(sum(ms for _, ms in rec[t][q][1]) for t in range(steps)) / steps for q in range(world)]
    ms_bal, a2a = [], []
    for kc in range(2):
        tot = sum(rec[0][q][1][kc][0] for q in range(world))
        avg = _m.ceil(tot / world)
        pool = torch.cat([store[q][kc] for q in range(world) if store[q][kc] is not None and store[q][kc].shape[0]])
        rows = pool[:avg].contiguous() if avg else pool[:0]
        kinetic.penalized_residual_rows(k, rows)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            kinetic.penalized_residual_rows(k, rows)
        e1.record()
        torch.cuda.synchronize()
        ms_bal.append(e0.elapsed_time(e1) / 3)
        shipped = max(abs(rec[0][q][1][kc][0] - avg) for q in range(world))
        a2a.append(2 * shipped * nb * 8 / 700e9 * 1e3)
    est = [T[q] - Rq[q] + sum(ms_bal) + sum(a2a) for q in range(world)]
    return {"config": f"config4 on {world} x-slabs, layer-2 residuals load-balanced (balanced_apply via the "
                      f"hk_hybrid_step residual hook), emulated on 1 GPU",
            "slab_columns": [p_.nxl for p_ in parts], "unbalanced_ms_per_slab_step": T,
            "hooked_ms_per_slab_step": [sum(rec[t][q][0] for t in range(steps)) / steps for q in range(world)],
            "residual_ms_per_slab_step": Rq, "layer2_rows_per_call": [[rec[0][q][1][kc][0] for q in range(world)]
                                                                        for kc in range(2)],
            "balanced_residual_ms_per_call": ms_bal, "alltoall_ms_per_call_at_700GBps": a2a,
            "ms_per_slab_step": est, "max_slab_ms": max(est), "sum_slab_ms": sum(est),
            "note": "ms_per_slab_step = T_q - R_q + balanced residual time + all-to-all estimate; "
                    "max_slab_ms ~ per-GPU step time of an 8-GPU run without the halo exchange"}


def config5(iters, steps=True):
    """Config 5, one GPU's x-slab (64 x 128 cells, N = 64, M = 8 x 8): Q over
    the slab (fast path + guard) and, with `steps`, one PR(2,2,2) IMEX step of
    the slab (periodic in x within the slab: the 1-GPU share of the weak-
    scaling layout; 2 Q evaluations per cell-step)."""
    n, a1, a2, nxl, ny = 64, 8, 8, 64, 128
    ctx = hk.default_context()
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    k = hk.precompute_kernel(vg, n, a1, a2, inputs.R_PHYS_MAX)
    f = inputs.config5_slab_torch(224, nxl, ny, n)
    cells = nxl * ny
    q = torch.empty_like(f)
    res = {}

    def coll():
        res["st"] = hk.spectral_collision(f, k, out=q, return_status=True)[1]

    ms_q = timed(coll, iters)
    md = (a1 - 1) * a2 + 1
    W = (2 * md + 2) * 5 * n ** 3 * math.log2(n ** 3) + (12 * md + 10) * n ** 3
    peak = ctx.fp64_peak_tflops()
    ach = W * cells / (ms_q * 1e-3) / 1e12
    out = {"config": "config5 slab: 64 x 128 cells (1 of 8 x-slabs of 512 x 128), N=64, M=8x8, hard spheres",
           "collision": {"ms": ms_q, "cell_updates_per_s": cells / (ms_q * 1e-3),
                         "rerouted": int(((res["st"]["flags"] & 4) != 0).sum()),
                         "roofline": {"bound": "fp64", "achieved_tflops": ach, "peak_tflops": peak, "frac": ach / peak,
                                      "algorithmic_flop_per_update": W}}}
    if steps:
        del q
        torch.cuda.empty_cache()
        dx = 1.0 / 512
        eps = torch.full((cells,), 1e-2, dtype=torch.float64, device="cuda")

        def step():
            kinetic.penalized_imex_step(f, nxl, ny, k, dx, 1.0 / ny, 0.1 * dx, eps)

        ms_s = timed(step, max(1, iters // 2))
        out["imex_step"] = {"ms": ms_s, "cell_updates_per_s": 2 * cells / (ms_s * 1e-3),
                            "note": "PR(2,2,2): 2 Q + 2 transports + stage solves per cell-step; dt = 0.1 dx, eps = 1e-2"}
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--configs", default="1,3")
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--no-steps", action="store_true")
    ap.add_argument("--hyb-steps", type=int, default=20)
    ap.add_argument("--no-full", action="store_true")
    args = ap.parse_args()
    for c in args.configs.split(","):
        if c == "1":
            r = config1(args.iters)
        elif c == "4":
            r = config4(args.iters)
        elif c == "4s":
            r = config4_slabs()
        elif c == "4w":
            r = config4_slabs(weighted=True)
        elif c == "4b":
            r = config4_slabs_balanced()
        elif c == "4h":
            r = config4_hybrid(args.hyb_steps, full_sample=not args.no_full)
        elif c == "5":
            r = config5(args.iters, steps=not args.no_steps)
        else:
            r = config3(args.iters, args.nx, args.nx)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()  # the next config starts from a clean device
        hk.default_context().trim()
