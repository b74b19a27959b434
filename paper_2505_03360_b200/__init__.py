"""hykin-b200: B200-native fast-spectral collision path of arXiv 2505.03360.

Python mirror of the reference's operator interface (namespace ``hykin``,
/root/reference/proj/core/include/hykin): same function names, argument
meaning and error classes, running on the sm_100a kernels of
``lib/libhykin_b200.so`` through the C-ABI of ``include/hykin_b200.h``.

    vgrid  = make_velocity_grid(32, 8.0)                 # src/grid.cpp:18
    kernel = precompute_kernel(vgrid, 32, 8, 8, r_phys)  # src/spectral.cpp:53
    q      = spectral_collision(f, kernel)               # src/spectral.cpp:114 (batched)

``f`` is a cell-major slab ``[cells, n^3]`` (or ``[n^3]`` for one cell):
a CUDA torch tensor (device path) or a numpy array (host path, H2D/D2H
inside the call).  fp64 only.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi

__all__ = [
    "error", "config_error", "aliasing_config_error", "degenerate_state_error",
    "positivity_error", "contract_violation", "numerical_consistency_error", "scenario_end_error",
    "VelocityGrid", "make_velocity_grid", "SpectralKernel", "precompute_kernel",
    "precompute_kernel_from_tables", "spectral_collision", "Context", "default_context",
]


# ---- exception hierarchy of inc/errors.hpp:9-61 ----------------------------
class error(RuntimeError):
    pass


class config_error(error):
    pass


class aliasing_config_error(config_error):
    pass


class degenerate_state_error(error):
    pass


class positivity_error(error):
    pass


class contract_violation(error):
    pass


class numerical_consistency_error(error):
    def __init__(self, msg, cell=-1):
        super().__init__(msg)
        self.cell = cell


class scenario_end_error(error):
    """A moving obstacle left the domain (src/coupling.cpp:113-118)."""


class io_error(error):
    """hykin::io_error (inc/errors.hpp)."""


class device_error(error):
    """CUDA failure (no reference analogue; the reference is CPU-only)."""


_STATUS_EXC = {
    _abi.HK_CONFIG: config_error,
    _abi.HK_ALIASING: aliasing_config_error,
    _abi.HK_DEGENERATE: degenerate_state_error,
    _abi.HK_NUMERICAL_CONSISTENCY: numerical_consistency_error,
    _abi.HK_CONTRACT: contract_violation,
    _abi.HK_CUDA: device_error,
    _abi.HK_NCCL: device_error,
    _abi.HK_POSITIVITY: positivity_error,
    _abi.HK_UNSUPPORTED: config_error,
    _abi.HK_SCENARIO_END: scenario_end_error,
    _abi.HK_IO: io_error,
}


class Context:
    """One hk_ctx per (process, device); all calls are ordered on `stream`."""

    def __init__(self, device: int = 0, stream=None):
        self._lib = _abi.lib()
        h = C.c_void_p()
        st = self._lib.hk_ctx_create(device, C.byref(h))
        if st:
            raise device_error(f"hk_ctx_create(device={device}) failed with status {st}: "
                               "no usable sm_100 device (there is no CPU fallback)")
        self.h = h
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream):
        ptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._lib.hk_ctx_set_stream(self.h, C.c_void_p(ptr))

    def check(self, st: int):
        if st == _abi.HK_OK:
            return
        cell = C.c_int64(-1)
        buf = C.create_string_buffer(512)
        self._lib.hk_last_error(self.h, C.byref(cell), buf, 512)
        exc = _STATUS_EXC.get(st, error)
        msg = buf.value.decode() or f"status {st}"
        if exc is numerical_consistency_error:
            raise exc(msg, cell.value)
        raise exc(msg)

    def trim(self):
        """Frees the context's cached device workspaces (hk_ctx_trim)."""
        self.check(self._lib.hk_ctx_trim(self.h))

    @property
    def launches(self) -> int:
        return int(self._lib.hk_launch_count(self.h))

    def fp64_peak_tflops(self) -> float:
        return float(self._lib.hk_measure_fp64_peak(self.h))

    # ---- native NCCL communicator (hk_comm.cu) ----
    @staticmethod
    def comm_unique_id() -> bytes:
        """128 opaque bytes (ncclGetUniqueId) that rank 0 ships to every rank."""
        buf = C.create_string_buffer(_abi.HK_COMM_ID_BYTES)
        st = _abi.lib().hk_comm_unique_id(buf)
        if st:
            raise device_error(f"hk_comm_unique_id failed with status {st} (libnccl.so.2 missing?)")
        return buf.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        if len(uid) != _abi.HK_COMM_ID_BYTES:
            raise contract_violation("communicator id must be 128 bytes")
        self.check(self._lib.hk_ctx_comm_init(self.h, nranks, rank, C.c_char_p(uid)))

    def halo_exchange(self, f, n: int, nx_local: int, ny: int, left, right):
        """x-slab halos over the context's communicator: f [ny][nx_local][n^3],
        left/right [ny][2][n^3] (torch CUDA tensors, fp64, contiguous)."""
        self.check(self._lib.hk_halo_exchange(self.h, n, C.c_void_p(f.data_ptr()), nx_local, ny,
                                              C.c_void_p(left.data_ptr()), C.c_void_p(right.data_ptr())))

    def allreduce_(self, buf, op: str = "sum"):
        """In-place all-reduce of a CUDA fp64 tensor over the context's ranks."""
        code = {"sum": _abi.HK_REDUCE_SUM, "max": _abi.HK_REDUCE_MAX}[op]
        self.check(self._lib.hk_allreduce_scalars(self.h, C.c_void_p(buf.data_ptr()), buf.numel(), code))
        return buf

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self._lib.hk_ctx_destroy(self.h)
            except Exception:
                pass
            self.h = None


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        import torch

        ctx = Context(device)
        ctx.set_stream(torch.cuda.current_stream(device))
        _default_ctx[device] = ctx
    return _default_ctx[device]


# ---- grids (inc/grid.hpp:45-56, src/grid.cpp:18-33) ------------------------
@dataclass
class VelocityGrid:
    nv: int
    vmax: float
    dv1: float = 0.0
    dvk: float = 0.0
    nodes: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return self.nv ** 3

    def index(self, k1: int, k2: int, k3: int) -> int:
        return (k1 * self.nv + k2) * self.nv + k3


def make_velocity_grid(nv: int, vmax: float) -> VelocityGrid:
    if nv < 2:
        raise config_error(f"velocity grid needs at least 2 nodes per axis, got {nv}")
    if vmax <= 0.0:
        raise config_error("velocity cutoff must be positive")
    dv = 2.0 * vmax / nv
    g = VelocityGrid(nv, vmax, dv, dv * dv * dv)
    g.nodes = -vmax + (np.arange(nv) + 0.5) * dv
    return g


# ---- spectral kernel (inc/spectral.hpp:15-56) ------------------------------
class SpectralKernel:
    """Device-resident weight tables; mirrors hykin::SpectralKernel's scalars."""

    def __init__(self, ctx: Context, handle: C.c_void_p, n: int, a1: int, a2: int, vmax: float):
        self.ctx, self.h = ctx, handle
        self.n, self.a1, self.a2, self.vmax = n, a1, a2, vmax
        info = (C.c_double * 6)()
        ctx._lib.hk_kernel_info(handle, info)
        self.r, self.jacobian, self.weight, self.r_phys = info[0], info[1], info[2], info[3]
        self.distinct_dirs = int(info[4])

    def dirs(self) -> int:
        return self.a1 * self.a2

    def modes(self) -> int:
        return self.n ** 3

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.ctx._lib.hk_kernel_destroy(self.h)
            except Exception:
                pass
            self.h = None


def precompute_kernel(vgrid: VelocityGrid, n: int, a1: int, a2: int, r_phys: float,
                      ctx: Context | None = None) -> SpectralKernel:
    """src/spectral.cpp:53-112 — same validation, tables built on the device."""
    if n != vgrid.nv:
        raise config_error(f"spectral mode count must match the velocity grid ({n} vs {vgrid.nv})")
    ctx = ctx or default_context()
    h = C.c_void_p()
    ctx.check(ctx._lib.hk_kernel_create(ctx.h, n, a1, a2, vgrid.vmax, r_phys, C.byref(h)))
    return SpectralKernel(ctx, h, n, a1, a2, vgrid.vmax)


def precompute_kernel_from_tables(vgrid: VelocityGrid, n: int, a1: int, a2: int, r_phys: float,
                                  alpha, alpha_prime, loss_diag,
                                  ctx: Context | None = None) -> SpectralKernel:
    """Uses the reference's own tables (SpectralKernel::alpha/alpha_prime/loss_diag)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    ap = np.ascontiguousarray(alpha_prime, dtype=np.float64)
    ld = np.ascontiguousarray(loss_diag, dtype=np.float64)
    assert a.size == a1 * a2 * n ** 3 and ap.size == a.size and ld.size == n ** 3
    h = C.c_void_p()
    ctx.check(ctx._lib.hk_kernel_create_from_tables(
        ctx.h, n, a1, a2, vgrid.vmax, r_phys, a.ctypes.data, ap.ctypes.data, ld.ctypes.data,
        C.byref(h)))
    return SpectralKernel(ctx, h, n, a1, a2, vgrid.vmax)


def _status_array_np(ncells: int) -> np.ndarray:
    return np.zeros(ncells, dtype=np.dtype([("max_re", "f8"), ("max_im", "f8"), ("q_norm2", "f8"),
                                            ("nyq_bound", "f8"), ("flags", "u4"), ("reserved", "u4"),
                                            ("loss_norm2", "f8")]))


def spectral_collision(f, kernel: SpectralKernel, out=None, *, exact: bool = False,
                       strict: bool = False, guard: bool = True, return_status: bool = False):
    """Batched Q(f) — src/spectral.cpp:114-154.

    strict=True reproduces the reference's throw: numerical_consistency_error
    (with ``.cell`` = lowest failing cell) when max|Im Q| > 1e-10 max|Re Q|,
    raised after `out` was written.  exact=True forces the full-complex path.
    """
    ctx = kernel.ctx
    flags = (_abi.HK_COLL_EXACT if exact else 0) | (_abi.HK_COLL_STRICT if strict else 0) | \
        (0 if guard else _abi.HK_COLL_NOGUARD)
    nb = kernel.modes()
    if isinstance(f, np.ndarray):
        fh = np.ascontiguousarray(f, dtype=np.float64)
        if fh.size % nb:
            raise contract_violation("f is not a whole number of velocity blocks")
        ncells = fh.size // nb
        if out is None:
            q = np.empty_like(fh)
        else:
            q = out
            if not (isinstance(q, np.ndarray) and q.dtype == np.float64 and q.flags["C_CONTIGUOUS"]
                    and q.flags["WRITEABLE"] and q.size == fh.size):
                raise contract_violation("out must be a writeable C-contiguous float64 array of f's size")
        sth = _status_array_np(ncells)
        st = ctx._lib.hk_collision_batch_host(ctx.h, kernel.h, fh.ctypes.data, q.ctypes.data,
                                              ncells, flags, sth.ctypes.data)
        ctx.check(st)
        return (q, sth) if return_status else q
    import torch

    if not (isinstance(f, torch.Tensor) and f.is_cuda and f.dtype == torch.float64):
        raise contract_violation("f must be a float64 CUDA tensor or a numpy array")
    f = f.contiguous()
    if f.numel() % nb:
        raise contract_violation("f is not a whole number of velocity blocks")
    ncells = f.numel() // nb
    if out is None:
        q = torch.empty_like(f)
    else:
        q = out
        if not (isinstance(q, torch.Tensor) and q.dtype == torch.float64 and q.is_contiguous()
                and q.device == f.device and q.numel() == f.numel()):
            raise contract_violation("out must be a contiguous float64 tensor of f's size on f's device")
    # every field is written by the library (zeroed or computed): no fill launch here
    stt = torch.empty(ncells * _abi.CELL_STATUS_BYTES // 8, dtype=torch.float64, device=f.device)
    st = ctx._lib.hk_collision_batch(ctx.h, kernel.h, f.data_ptr(), q.data_ptr(), ncells, flags,
                                     stt.data_ptr())
    ctx.check(st)
    if return_status:
        return q, status_to_numpy(stt, ncells)
    return q


def status_to_numpy(stt, ncells: int) -> np.ndarray:
    raw = stt.detach().cpu().numpy().view(np.uint8)[: ncells * _abi.CELL_STATUS_BYTES]
    return raw.view(_status_array_np(0).dtype).copy()
