"""Per-cell kinetic operators and the PR(2,2,2) steps on the device.

Python mirror of the reference's moments / ES-BGK / Boltzmann-layer /
indicator / transport interfaces (inc/moments.hpp, inc/esbgk.hpp,
inc/boltzmann.hpp, inc/indicators.hpp, inc/regime.hpp, inc/transport.hpp),
batched over a cell-major slab ``[cells, n^3]`` of float64 CUDA tensors and
executed by libhykin_b200.so.  Per-cell failures that the reference would
throw are returned as status arrays (``status`` = HK_* code per cell) and,
with ``check=True``, raised as the reference's exception class for the
lowest failing cell.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import NamedTuple
from dataclasses import dataclass

import torch

from . import _abi
from . import default_context, degenerate_state_error, contract_violation, VelocityGrid, SpectralKernel

_STATUS_EXC = {_abi.HK_DEGENERATE: degenerate_state_error, _abi.HK_CONTRACT: contract_violation}


def _ptr(t):
    return None if t is None else t.data_ptr()


def _check_cells(status, what):
    bad = torch.nonzero(status & 0xFF).flatten()
    if bad.numel():
        c = int(bad[0])
        code = int(status[c]) & 0xFF
        raise _STATUS_EXC.get(code, RuntimeError)(f"{what}: cell {c} failed with status {code}")


def _cells(f, n):
    if not (f.is_cuda and f.dtype == torch.float64):
        raise contract_violation("expected a float64 CUDA tensor")
    f = f.contiguous()
    nb = n ** 3
    if f.numel() % nb:
        raise contract_violation("not a whole number of velocity blocks")
    return f, f.numel() // nb


@dataclass
class EsbgkParams:  # inc/esbgk.hpp:17-23
    beta: float = -0.5
    nu_coeff: float = 0.5 * math.pi
    eps_weno: float = 1e-6


@dataclass
class PenalizationRule:  # inc/boltzmann.hpp:14-17
    coeff: float = 2.0 * math.pi


@dataclass
class Thresholds:  # inc/indicators.hpp:49-55
    eta0: float = 1e-3
    eta1: float = 1e-2
    delta0: float = 1e-3


def moments_of(f, vgrid: VelocityGrid, *, sigma=False, realizability=False, l1=False, check=True, ctx=None):
    """moments_of + second_moment + realizability_matrix + l1_distance_to_maxwellian,
    batched.  Returns dict with 'moments' [cells,5] = (rho, ux, uy, uz, T) and the
    requested extras ('sigma' [cells,6], 'realizability' [cells,13], 'l1' [cells])."""
    ctx = ctx or default_context(f.device.index or 0)
    f, nc = _cells(f, vgrid.nv)
    dev = f.device
    out = {"moments": torch.empty((nc, 5), dtype=torch.float64, device=dev),
           "status": torch.empty(nc, dtype=torch.int32, device=dev)}
    if sigma:
        out["sigma"] = torch.empty((nc, 6), dtype=torch.float64, device=dev)
    if realizability:
        out["realizability"] = torch.empty((nc, 13), dtype=torch.float64, device=dev)
    if l1:
        out["l1"] = torch.empty(nc, dtype=torch.float64, device=dev)
    ctx.check(ctx._lib.hk_moments_batch(ctx.h, vgrid.nv, vgrid.vmax, f.data_ptr(), nc, out["moments"].data_ptr(),
                                        _ptr(out.get("sigma")), _ptr(out.get("realizability")), _ptr(out.get("l1")),
                                        out["status"].data_ptr()))
    if check:
        _check_cells(out["status"], "moments_of")
    return out


def maxwellian(moments, vgrid: VelocityGrid, ctx=None):
    """maxwellian (src/moments.cpp:88-112) for moments [cells,5]."""
    ctx = ctx or default_context(moments.device.index or 0)
    moments = moments.contiguous()
    nc = moments.shape[0]
    out = torch.empty((nc, vgrid.nv ** 3), dtype=torch.float64, device=moments.device)
    st = torch.empty(nc, dtype=torch.int32, device=moments.device)
    ctx.check(ctx._lib.hk_maxwellian_batch(ctx.h, vgrid.nv, vgrid.vmax, moments.data_ptr(), nc, out.data_ptr(),
                                           st.data_ptr()))
    _check_cells(st, "maxwellian")
    return out


def anisotropic_gaussian(moments, theta, beta: float, vgrid: VelocityGrid, ctx=None):
    """anisotropic_gaussian (src/moments.cpp:120-157) for moments [cells,5] and stress
    tensors theta [cells,3,3]; returns (G [cells,n^3], fell_back bool [cells])."""
    ctx = ctx or default_context(moments.device.index or 0)
    moments = moments.contiguous()
    nc = moments.shape[0]
    th = theta.to(device=moments.device, dtype=torch.float64).reshape(nc, 9).contiguous()
    out = torch.empty((nc, vgrid.nv ** 3), dtype=torch.float64, device=moments.device)
    fb = torch.empty(nc, dtype=torch.int32, device=moments.device)
    ctx.check(ctx._lib.hk_anisotropic_gaussian_batch(ctx.h, vgrid.nv, vgrid.vmax, moments.data_ptr(), th.data_ptr(),
                                                     beta, nc, out.data_ptr(), fb.data_ptr()))
    return out, fb != 0


def match_moments(f, vgrid: VelocityGrid, targets, *, check=True, ctx=None):
    """match_moments (src/moments.cpp:225-246) in place; targets [cells,5] =
    (rho, momentum x, y, z, energy)."""
    ctx = ctx or default_context(f.device.index or 0)
    assert f.is_contiguous()
    _, nc = _cells(f, vgrid.nv)
    t = targets.to(device=f.device, dtype=torch.float64).reshape(nc, 5).contiguous()
    st = torch.empty(nc, dtype=torch.int32, device=f.device)
    ctx.check(ctx._lib.hk_match_moments_batch(ctx.h, vgrid.nv, vgrid.vmax, f.data_ptr(), t.data_ptr(), nc,
                                              st.data_ptr()))
    if check:
        _check_cells(st, "match_moments")
    return f


def remove_invariant_moments(q, weight, vgrid: VelocityGrid, uc, *, check=True, ctx=None):
    """remove_invariant_moments (src/moments.cpp:248-267) in place on q [cells,n^3]
    with weight [cells,n^3] and centres uc [cells,3]."""
    ctx = ctx or default_context(q.device.index or 0)
    assert q.is_contiguous()
    _, nc = _cells(q, vgrid.nv)
    w = weight.to(device=q.device, dtype=torch.float64).contiguous()
    if w.numel() != q.numel():
        raise contract_violation("remove_invariant_moments: weight must match q")
    u = uc.to(device=q.device, dtype=torch.float64).reshape(nc, 3).contiguous()
    st = torch.empty(nc, dtype=torch.int32, device=q.device)
    ctx.check(ctx._lib.hk_remove_invariant_moments_batch(ctx.h, vgrid.nv, vgrid.vmax, q.data_ptr(), w.data_ptr(),
                                                         u.data_ptr(), nc, st.data_ptr()))
    if check:
        _check_cells(st, "remove_invariant_moments")
    return q


def _eps_arg(eps, nc, dev):
    if isinstance(eps, torch.Tensor):
        e = eps.to(device=dev, dtype=torch.float64).contiguous()
        assert e.numel() == nc
        return e, 0.0
    return None, float(eps)


def esbgk_stage_solve(f_star, a: float, eps, params: EsbgkParams, vgrid: VelocityGrid, *, check=True, ctx=None):
    """esbgk_stage_solve (src/esbgk.cpp:9-45), batched.  Returns (out, info) with
    info = status | (gaussian_fallback << 8) per cell."""
    ctx = ctx or default_context(f_star.device.index or 0)
    f_star, nc = _cells(f_star, vgrid.nv)
    e, es = _eps_arg(eps, nc, f_star.device)
    out = torch.empty_like(f_star)
    info = torch.empty(nc, dtype=torch.int32, device=f_star.device)
    ctx.check(ctx._lib.hk_esbgk_stage_batch(ctx.h, vgrid.nv, vgrid.vmax, f_star.data_ptr(), out.data_ptr(), nc, a,
                                            _ptr(e), es, params.beta, params.nu_coeff, info.data_ptr(), None))
    if check:
        _check_cells(info, "esbgk_stage_solve")
    return out, info


def penalized_stage_solve(f_star, a: float, eps, rule: PenalizationRule, vgrid: VelocityGrid, *, check=True,
                          ctx=None):
    """penalized_stage_solve (src/boltzmann.cpp:29-45), batched."""
    ctx = ctx or default_context(f_star.device.index or 0)
    f_star, nc = _cells(f_star, vgrid.nv)
    e, es = _eps_arg(eps, nc, f_star.device)
    out = torch.empty_like(f_star)
    info = torch.empty(nc, dtype=torch.int32, device=f_star.device)
    ctx.check(ctx._lib.hk_penalized_stage_batch(ctx.h, vgrid.nv, vgrid.vmax, f_star.data_ptr(), out.data_ptr(), nc, a,
                                                _ptr(e), es, rule.coeff, info.data_ptr(), None))
    if check:
        _check_cells(info, "penalized_stage_solve")
    return out, info


def penalized_residual(f, kernel: SpectralKernel, vgrid: VelocityGrid, rule: PenalizationRule = PenalizationRule(),
                       *, exact=False, check=True):
    """penalized_residual (src/boltzmann.cpp:9-27), batched (collision incl.)."""
    ctx = kernel.ctx
    f, nc = _cells(f, vgrid.nv)
    out = torch.empty_like(f)
    st = torch.empty(nc, dtype=torch.int32, device=f.device)
    flags = _abi.HK_COLL_EXACT if exact else 0
    ctx.check(ctx._lib.hk_penalized_residual_batch(ctx.h, kernel.h, f.data_ptr(), out.data_ptr(), nc, rule.coeff,
                                                   flags, st.data_ptr(), None))
    if check:
        _check_cells(st, "penalized_residual")
    return out


def classify(moments, nx: int, ny: int, dx: float, dy: float, eps_cell, r_in, th: Thresholds = Thresholds(),
             l1=None, mu0=1.0, kappa0=1.0, signed_sum=False, ctx=None):
    """Indicators + Algorithm 1 over a periodic grid of kinetic cells.
    Returns (r_out int8 [cells], indicators [cells,4] = (la, lb, lc, lambda_B), status)."""
    ctx = ctx or default_context(moments.device.index or 0)
    dev = moments.device
    nc = nx * ny
    r_out = torch.empty(nc, dtype=torch.int8, device=dev)
    ind = torch.empty((nc, 4), dtype=torch.float64, device=dev)
    st = torch.empty(nc, dtype=torch.int32, device=dev)
    e = eps_cell.to(device=dev, dtype=torch.float64).contiguous()
    ctx.check(ctx._lib.hk_classify(ctx.h, nx, ny, dx, dy, moments.contiguous().data_ptr(), e.data_ptr(), _ptr(l1),
                                   r_in.to(device=dev, dtype=torch.int8).contiguous().data_ptr(), r_out.data_ptr(),
                                   ind.data_ptr(), st.data_ptr(), th.eta0, th.eta1, th.delta0, mu0, kappa0,
                                   int(signed_sum)))
    return r_out, ind, st


def kinetic_transport_rhs_periodic(f, nx: int, ny: int, vgrid: VelocityGrid, dx: float, dy: float,
                                   eps_weno: float = 1e-6, x_halo: int = 0, ctx=None):
    """kinetic_transport_rhs_periodic (src/transport.cpp:51-66); with x_halo >= 2 the
    input carries ghost columns (x-slab of a partitioned grid)."""
    ctx = ctx or default_context(f.device.index or 0)
    f = f.contiguous()
    out = torch.empty((nx * ny, vgrid.nv ** 3), dtype=torch.float64, device=f.device)
    ctx.check(ctx._lib.hk_transport_rhs(ctx.h, vgrid.nv, vgrid.vmax, f.data_ptr(), out.data_ptr(), nx, ny, x_halo, dx,
                                        dy, eps_weno))
    return out


def esbgk_imex_step(f, nx, ny, vgrid: VelocityGrid, dx, dy, dt, eps_cell, params: EsbgkParams = EsbgkParams(),
                    ctx=None):
    """esbgk_imex_step (src/esbgk.cpp:47-99), in place on the device slab."""
    ctx = ctx or default_context(f.device.index or 0)
    assert f.is_contiguous()
    e = eps_cell.to(device=f.device, dtype=torch.float64).contiguous()
    ctx.check(ctx._lib.hk_esbgk_imex_step(ctx.h, vgrid.nv, vgrid.vmax, f.data_ptr(), nx, ny, dx, dy, dt, e.data_ptr(),
                                          params.beta, params.nu_coeff, params.eps_weno, None))
    return f


def penalized_imex_step(f, nx, ny, kernel: SpectralKernel, dx, dy, dt, eps_cell,
                        rule: PenalizationRule = PenalizationRule(), eps_weno: float = 1e-6, exact=False):
    """penalized_imex_step (src/boltzmann.cpp:47-110), in place on the device slab."""
    ctx = kernel.ctx
    assert f.is_contiguous()
    e = eps_cell.to(device=f.device, dtype=torch.float64).contiguous()
    ctx.check(ctx._lib.hk_penalized_imex_step(ctx.h, kernel.h, f.data_ptr(), nx, ny, dx, dy, dt, e.data_ptr(),
                                              rule.coeff, eps_weno, _abi.HK_COLL_EXACT if exact else 0, None))
    return f


# ---------------------------------------------------------------------------
# Layer 0 (compressible Euler) and layer transitions (SURVEY §8f "next")
# ---------------------------------------------------------------------------
def euler_rhs_periodic(u, nx: int, ny: int, dx: float, dy: float, xi: float = 5.0 / 3.0, eps_weno: float = 1e-6,
                       ctx=None):
    """euler_rhs_periodic (src/euler.cpp:159-170): u [nx*ny, 4] conserved -> rhs."""
    ctx = ctx or default_context(u.device.index or 0)
    u = u.contiguous()
    out = torch.empty_like(u)
    ctx.check(ctx._lib.hk_euler_rhs_periodic(ctx.h, u.data_ptr(), nx, ny, dx, dy, xi, eps_weno, out.data_ptr()))
    return out


def tvd_rk2_step_periodic(u, nx: int, ny: int, dx: float, dy: float, dt: float, xi: float = 5.0 / 3.0,
                          eps_weno: float = 1e-6, ctx=None):
    """tvd_rk2_step_periodic (src/euler.cpp:172-181), in place on the device field."""
    ctx = ctx or default_context(u.device.index or 0)
    assert u.is_contiguous()
    ctx.check(ctx._lib.hk_euler_tvd_rk2_step(ctx.h, u.data_ptr(), nx, ny, dx, dy, dt, xi, eps_weno, None))
    return u


def conserved_to_maxwellian(u, vgrid: VelocityGrid, heat_ratio: float = 5.0 / 3.0, ctx=None):
    """Layer 0 -> 1 (src/regime.cpp:62-65): Maxwellian of each cell's hydro state."""
    ctx = ctx or default_context(u.device.index or 0)
    u = u.contiguous()
    nc = u.shape[0]
    f = torch.empty((nc, vgrid.nv ** 3), dtype=torch.float64, device=u.device)
    ctx.check(ctx._lib.hk_conserved_to_maxwellian(ctx.h, vgrid.nv, vgrid.vmax, u.data_ptr(), nc, heat_ratio, f.data_ptr()))
    return f


def distribution_to_conserved(f, vgrid: VelocityGrid, heat_ratio: float = 5.0 / 3.0, ctx=None):
    """Layer 1 -> 0 (src/regime.cpp:66-70): hydro state of each cell's moments."""
    ctx = ctx or default_context(f.device.index or 0)
    f, nc = _cells(f, vgrid.nv)
    u = torch.empty((nc, 4), dtype=torch.float64, device=f.device)
    ctx.check(ctx._lib.hk_distribution_to_conserved(ctx.h, vgrid.nv, vgrid.vmax, f.data_ptr(), nc, heat_ratio,
                                                    u.data_ptr()))
    return u


def gather_cells(src, idx, ctx=None):
    """Dense batch of the cells `idx` (int64 device tensor) of a cell-major slab."""
    ctx = ctx or default_context(src.device.index or 0)
    idx = idx.to(device=src.device, dtype=torch.int64).contiguous()
    dst = torch.empty((idx.numel(), src.shape[1]), dtype=src.dtype, device=src.device)
    ctx.check(ctx._lib.hk_gather_cells(ctx.h, src.shape[1], src.data_ptr(), idx.data_ptr(), idx.numel(), dst.data_ptr()))
    return dst


def scatter_cells(src, idx, dst, ctx=None):
    """dst[idx[k]] = src[k] (the inverse of gather_cells), in place on `dst`."""
    ctx = ctx or default_context(src.device.index or 0)
    idx = idx.to(device=src.device, dtype=torch.int64).contiguous()
    ctx.check(ctx._lib.hk_scatter_cells(ctx.h, src.shape[1], src.contiguous().data_ptr(), idx.data_ptr(), idx.numel(),
                                        dst.data_ptr()))
    return dst


# ---- embedded obstacles (src/grid.cpp:56-110, src/coupling.cpp:95-147) -------
ObstacleSpec = _abi.ObstacleSpec


class ObstacleApplyResult(NamedTuple):  # inc/hykin/coupling.hpp:53-56
    covered: int
    vacated: int


def classify_cells(nx: int, ny: int, spec: ObstacleSpec, device=0, ctx=None):
    """CellKind per cell (uint8 device tensor [ny*nx]): 0 interior, 1 obstacle,
    2 forced ring, 3 ghost.  config_error when the obstacle or its ring
    reaches the 4-cell ghost frame."""
    ctx = ctx or default_context(device)
    kind = torch.empty(nx * ny, dtype=torch.uint8, device=f"cuda:{ctx.device}")
    ctx.check(ctx._lib.hk_classify_cells(ctx.h, nx, ny, C.byref(spec), kind.data_ptr()))
    return kind


def apply_obstacle(nx: int, ny: int, vgrid: VelocityGrid, spec: ObstacleSpec, r, kind, hydro, f,
                   heat_ratio: float = 5.0 / 3.0, ctx=None) -> ObstacleApplyResult:
    """One step of the obstacle update, in place: `spec` moves, r (int8), kind
    (uint8), hydro [cells,4] and the dense field f [cells,n^3] (device tensors)
    follow the reference; blocks of newly covered cells are left as they are."""
    for t, dt in ((r, torch.int8), (kind, torch.uint8), (hydro, torch.float64), (f, torch.float64)):
        assert t.is_cuda and t.dtype == dt and t.is_contiguous(), "device tensors of the documented dtypes"
    ctx = ctx or default_context(f.device.index or 0)
    cov, vac = C.c_int(0), C.c_int(0)
    ctx.check(ctx._lib.hk_apply_obstacle(ctx.h, vgrid.nv, vgrid.vmax, C.byref(spec), nx, ny, r.data_ptr(),
                                         kind.data_ptr(), hydro.data_ptr(), f.data_ptr(), heat_ratio, C.byref(cov),
                                         C.byref(vac)))
    return ObstacleApplyResult(cov.value, vac.value)


# ---- cross-layer stencil synthesis (src/coupling.cpp:57-93) ------------------
def _stage_view_args(r, kind, hydro, f):
    for t, dt in ((r, torch.int8), (kind, torch.uint8), (hydro, torch.float64), (f, torch.float64)):
        assert t.is_cuda and t.dtype == dt and t.is_contiguous(), "device tensors of the documented dtypes"


def synthesize_hydro_state(nx: int, ny: int, vgrid: VelocityGrid, r, kind, hydro, f, spec: ObstacleSpec = None,
                           heat_ratio: float = 5.0 / 3.0, ctx=None):
    """The conserved state a stencil sees at every cell ([cells, 4] device tensor)."""
    _stage_view_args(r, kind, hydro, f)
    ctx = ctx or default_context(f.device.index or 0)
    out = torch.empty((nx * ny, 4), dtype=torch.float64, device=f.device)
    ctx.check(ctx._lib.hk_synthesize_hydro(ctx.h, vgrid.nv, vgrid.vmax, nx, ny,
                                           C.byref(spec) if spec is not None else None, r.data_ptr(), kind.data_ptr(),
                                           hydro.data_ptr(), f.data_ptr(), heat_ratio, out.data_ptr()))
    return out


def synthesize_distribution(nx: int, ny: int, vgrid: VelocityGrid, r, kind, hydro, f, cells=None,
                            spec: ObstacleSpec = None, heat_ratio: float = 5.0 / 3.0, ctx=None):
    """cells (int64 tensor of cell indices): the blocks a stencil sees there,
    [len(cells), n^3].  cells None: fills the transport-stencil halo of the
    kinetic cells in place in f and returns the number of blocks written."""
    _stage_view_args(r, kind, hydro, f)
    ctx = ctx or default_context(f.device.index or 0)
    sp = C.byref(spec) if spec is not None else None
    filled = C.c_int64(0)
    if cells is None:
        ctx.check(ctx._lib.hk_synthesize_distributions(ctx.h, vgrid.nv, vgrid.vmax, nx, ny, sp, r.data_ptr(),
                                                       kind.data_ptr(), hydro.data_ptr(), f.data_ptr(), heat_ratio,
                                                       None, 0, None, C.byref(filled)))
        return filled.value
    idx = cells.to(device=f.device, dtype=torch.int64).contiguous()
    out = torch.empty((idx.numel(), vgrid.nv ** 3), dtype=torch.float64, device=f.device)
    ctx.check(ctx._lib.hk_synthesize_distributions(ctx.h, vgrid.nv, vgrid.vmax, nx, ny, sp, r.data_ptr(),
                                                   kind.data_ptr(), hydro.data_ptr(), f.data_ptr(), heat_ratio,
                                                   idx.data_ptr(), idx.numel(), out.data_ptr(), C.byref(filled)))
    return out


# ---------------------------------------------------------------------------
# Hybrid time step (SURVEY §8f "next" #1; contract in include/hykin_b200.h)
# ---------------------------------------------------------------------------
@dataclass
class HybridParams:
    """Thresholds + physics of one hybrid step (ScenarioConfig, inc/hykin/scenario.hpp:39-63)."""
    eta0: float = 1e-3
    eta1: float = 1e-2
    delta0: float = 1e-3
    mu0: float = 1.0
    kappa0: float = 1.0
    signed_sum: bool = False
    update_regimes: bool = True
    heat_ratio: float = 5.0 / 3.0
    esbgk_beta: float = -0.5
    nu_coeff: float = 0.5 * math.pi
    pen_coeff: float = 2.0 * math.pi
    eps_weno: float = 1e-6
    exact: bool = False  # collision of the residuals on the exact (two-transform) path
    ghost_x: int = 0     # x-slab ghost columns per side (partition.hybrid_step_slab)

    def to_c(self) -> "_abi.HybridParams":
        return _abi.HybridParams(self.eta0, self.eta1, self.delta0, self.mu0, self.kappa0, int(self.signed_sum),
                                 int(self.update_regimes), self.heat_ratio, self.esbgk_beta, self.nu_coeff,
                                 self.pen_coeff, self.eps_weno, _abi.HK_COLL_EXACT if self.exact else 0,
                                 int(self.ghost_x), None, None)


class _DeviceArray:
    """A raw device pointer as a CUDA-array-interface object (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None, "stream": None}


def device_view(ptr: int, shape, dtype=torch.float64, device=None) -> torch.Tensor:
    """torch tensor over `ptr` (no copy); empty when shape has a zero."""
    if not ptr or 0 in tuple(shape):
        return torch.empty(tuple(shape), dtype=dtype, device=device or "cuda")
    typestr = {torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_DeviceArray(ptr, shape, typestr), device=device or "cuda")


def penalized_residual_rows(kernel: SpectralKernel, y: torch.Tensor, pen_coeff: float = 2.0 * math.pi,
                            exact: bool = False, out=None, status=None):
    """penalized_residual (src/boltzmann.cpp:9-27) of the rows of y [m, n^3] ->
    (res [m, n^3], status int32 [m]) without raising (the hybrid step's hook form);
    out / status: preallocated destinations (no allocation on the hook path)."""
    ctx = kernel.ctx
    out = torch.empty_like(y) if out is None else out
    st = torch.zeros(y.shape[0], dtype=torch.int32, device=y.device) if status is None else status
    if y.shape[0]:
        ctx.check(ctx._lib.hk_penalized_residual_batch(ctx.h, kernel.h, y.data_ptr(), out.data_ptr(), y.shape[0],
                                                       pen_coeff, _abi.HK_COLL_EXACT if exact else 0, st.data_ptr(),
                                                       None))
    return out, st


class HybridCounts(NamedTuple):
    layer0: int
    layer1: int
    layer2: int
    to_kinetic: int   # 0 -> 1 transitions
    to_fluid: int     # 1 -> 0 transitions
    halo_blocks: int  # layer-0 Maxwellian blocks synthesized for the transport stencil


def _hybrid_call(kernel: SpectralKernel, nx: int, ny: int, eps_cell, r, hydro, f, params: HybridParams,
                 residual_hook, call):
    """Argument checks, the residual hook as a C callback, then call(e, hp) (hk_hybrid_step[_slab])."""
    ctx = kernel.ctx
    cells = nx * ny
    for name, t, dt_, width in (("r", r, torch.int8, 1), ("hydro", hydro, torch.float64, 4),
                                ("f", f, torch.float64, kernel.modes())):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt_ and t.is_contiguous()):
            raise contract_violation(f"hybrid_step: {name} must be a contiguous {dt_} CUDA tensor")
        if t.numel() != cells * width:
            raise contract_violation(f"hybrid_step: {name} has {t.numel()} elements, expected {cells * width}")
    e = eps_cell.to(device=f.device, dtype=torch.float64).contiguous()
    if e.numel() != cells:
        raise contract_violation(f"hybrid_step: eps_cell has {e.numel()} elements, expected {cells}")
    hp = params.to_c()
    errors = []
    if residual_hook is not None:
        nb = kernel.modes()

        def _hook(user, y_ptr, res_ptr, m2, st_ptr, stream):
            try:
                residual_hook(device_view(y_ptr, (m2, nb), device=f.device), device_view(res_ptr, (m2, nb), device=f.device),
                              device_view(st_ptr, (m2,), torch.int32, device=f.device))
                return 0
            except Exception as exc:  # reported after the call (a C frame cannot unwind Python)
                errors.append(exc)
                return _abi.HK_CONTRACT

        cb = _abi.RESIDUAL_FN(_hook)
        hp.residual_fn = C.cast(cb, C.c_void_p)
    import gc
    gc_was = gc.isenabled()
    if residual_hook is not None:
        gc.disable()  # no collector pause inside the hook while the step's kernels wait on it
    try:
        st = call(e, hp)
    finally:
        if gc_was:
            gc.enable()
    if errors:
        raise errors[0]
    ctx.check(st)


def hybrid_step(kernel: SpectralKernel, nx: int, ny: int, dx: float, dy: float, dt: float, eps_cell, r, hydro, f,
                params: HybridParams = HybridParams(), residual_hook=None) -> HybridCounts:
    """One hybrid step in place on device tensors: r [cells] int8, hydro [cells, 4]
    conserved, f [cells, n^3] dense, eps_cell [cells].  Algorithm 1 regime update,
    convert_on_transition, Euler TVD-RK2 on layer 0, PR(2,2,2) ES-BGK / penalized
    Boltzmann on layers 1 / 2 with the cross-layer transport halo.

    residual_hook(y, res, status): optional evaluator of the layer-2 residuals
    (hk_hybrid_params.residual_fn): y / res [m2, n^3] and status int32 [m2]
    device views; called twice per step, also with m2 = 0."""
    ctx = kernel.ctx
    counts = (C.c_int64 * 6)()
    _hybrid_call(kernel, nx, ny, eps_cell, r, hydro, f, params, residual_hook,
                 lambda e, hp: ctx._lib.hk_hybrid_step(ctx.h, kernel.h, nx, ny, dx, dy, dt, e.data_ptr(), r.data_ptr(),
                                                      hydro.data_ptr(), f.data_ptr(), C.byref(hp), counts))
    return HybridCounts(*[int(c) for c in counts])


def hybrid_step_slab_native(kernel: SpectralKernel, nx_local: int, ny: int, dx: float, dy: float, dt: float, eps_cell,
                            r, hydro, f, params: HybridParams = HybridParams(), ghost: int = 8,
                            residual_hook=None) -> list:
    """hk_hybrid_step_slab: the x-slab hybrid step with its host logic in C++ (the
    ghost columns of r, eps, hydro, f exchanged over the context's NCCL
    communicator into a padded copy, or the slab's own wrap without one; the step
    on the padded torus; the interior copied back).  Returns the global layer
    counts [n0, n1, n2] after the step."""
    ctx = kernel.ctx
    counts = (C.c_int64 * 3)()
    _hybrid_call(kernel, nx_local, ny, eps_cell, r, hydro, f, params, residual_hook,
                 lambda e, hp: ctx._lib.hk_hybrid_step_slab(ctx.h, kernel.h, nx_local, ny, dx, dy, dt, e.data_ptr(),
                                                           r.data_ptr(), hydro.data_ptr(), f.data_ptr(), C.byref(hp),
                                                           ghost, counts))
    return [int(c) for c in counts]


# ---- snapshot I/O -----------------------------------------
def write_snapshot(directory: str, step: int, time: float, vgrid: VelocityGrid, nx: int, ny: int, dx: float, dy: float,
                   r, hydro, f, kind=None, heat_ratio: float = 5.0 / 3.0, config: dict = None, ctx=None):
    """write_snapshot: moments_<step>.csv (i,j,x,y,rho,ux,uy,T,P), regimes_<step>.txt
    (layers, -1 = obstacle) and meta_<step>.json in `directory` (hk_write_snapshot).
    Raises io_error when the files cannot be written."""
    import json
    ctx = ctx or default_context(f.device.index or 0)
    for name, t, dt_ in (("r", r, torch.int8), ("hydro", hydro, torch.float64), ("f", f, torch.float64)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt_ and t.is_contiguous()):
            raise contract_violation(f"write_snapshot: {name} must be a contiguous {dt_} CUDA tensor")
    if kind is not None and not (kind.is_cuda and kind.dtype == torch.uint8 and kind.is_contiguous()):
        raise contract_violation("write_snapshot: kind must be a contiguous uint8 CUDA tensor")
    cfg = json.dumps(config).encode() if config is not None else None
    ctx.check(ctx._lib.hk_write_snapshot(ctx.h, vgrid.nv, vgrid.vmax, nx, ny, dx, dy, r.data_ptr(), _ptr(kind),
                                         hydro.data_ptr(), f.data_ptr(), heat_ratio, int(step), float(time),
                                         str(directory).encode(), cfg))
