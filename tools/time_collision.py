"""Times hk_collision_batch (and its kernels) on config-2 shapes; one JSON line."""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03360_b200 as hk
from paper_2505_03360_b200 import inputs

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=4096)
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--a1", type=int, default=8)
ap.add_argument("--a2", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--noguard", action="store_true")
ap.add_argument("--tag", default="")
ap.add_argument("--slab", type=int, default=-1, help="N=64: x-slab of the config-5 field from this column (cells/128 columns)")
args = ap.parse_args()
ctx = hk.Context(0, torch.cuda.current_stream())
vg = hk.make_velocity_grid(args.n, 8.0)
kern = hk.precompute_kernel(vg, args.n, args.a1, args.a2, inputs.R_PHYS_MAX, ctx=ctx)
if args.n == 32:
    f = inputs.config2_cells_torch(args.cells, 32, device="cuda")
elif args.n == 64 and args.slab >= 0:
    f = inputs.config5_slab_torch(i0=args.slab, nxl=max(1, args.cells // 128), ny=128, n=64)
elif args.n == 64:
    base = torch.from_numpy(inputs.config5_cells(min(args.cells, 16), 64)).cuda()
    f = base.repeat((args.cells + len(base) - 1) // len(base), 1)[: args.cells].contiguous()
else:
    f = torch.from_numpy(inputs.config1_cells(args.cells, args.n)).cuda()
q = torch.empty_like(f)
kw = dict(exact=args.exact, guard=not args.noguard)
for _ in range(2):
    hk.spectral_collision(f, kern, out=q, **kw)
torch.cuda.synchronize()
ctx._lib.hk_ctx_set_timing(ctx.h, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.iters):
    hk.spectral_collision(f, kern, out=q, **kw)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.iters
res = {}
for tag in (0, 1, 2):
    t, n = C.c_double(0), C.c_int64(0)
    ctx._lib.hk_ctx_timing_report(ctx.h, tag, C.byref(t), C.byref(n))
    res[tag] = t.value / max(n.value, 1)
_, st = hk.spectral_collision(f, kern, out=q, return_status=True, **kw)
print(json.dumps({"tag": args.tag, "cells": args.cells, "ms_step": ms, "cells_per_s": args.cells / ms * 1e3,
                  "main_ms": res[0], "guard_ms": res[1], "reroute_ms": res[2],
                  "rerouted": int(((st["flags"] & 4) != 0).sum()), "qsum": float(q.abs().sum())}))
