"""ctypes binding of the C-ABI in include/hykin_b200.h.

The product path: every call here lands in paper_2505_03360_b200/lib/
libhykin_b200.so (hand-written sm_100a CUDA).  There is no CPU fallback —
if the library or a usable B200 is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HK_LIB") or os.path.join(HERE, "lib", "libhykin_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "hykin_b200.h")

HK_OK = 0
HK_CONFIG = 1
HK_ALIASING = 2
HK_DEGENERATE = 3
HK_NUMERICAL_CONSISTENCY = 4
HK_CONTRACT = 5
HK_CUDA = 6
HK_NCCL = 7
HK_POSITIVITY = 8
HK_UNSUPPORTED = 9
HK_SCENARIO_END = 10
HK_IO = 11

HK_COMM_ID_BYTES = 128
HK_IPC_HANDLE_BYTES = 64
HK_REDUCE_SUM = 0
HK_REDUCE_MAX = 1

HK_CELL_EXACT = 1
HK_CELL_RESIDUE = 2
HK_CELL_GUARD_REROUTED = 4

HK_COLL_EXACT = 1
HK_COLL_STRICT = 2
HK_COLL_NOGUARD = 4


class CellStatus(C.Structure):
    _fields_ = [
        ("max_re", C.c_double),
        ("max_im", C.c_double),
        ("q_norm2", C.c_double),
        ("nyq_bound", C.c_double),
        ("flags", C.c_uint32),
        ("reserved", C.c_uint32),
        ("loss_norm2", C.c_double),
    ]


CELL_STATUS_BYTES = C.sizeof(CellStatus)  # 40

HK_OBSTACLE_NONE, HK_OBSTACLE_RECTANGLE, HK_OBSTACLE_DISK = 0, 1, 2
HK_CELL_INTERIOR, HK_CELL_OBSTACLE, HK_CELL_FORCED_RING, HK_CELL_GHOST = 0, 1, 2, 3


class ObstacleSpec(C.Structure):
    """hk_obstacle_spec == ObstacleSpec (inc/hykin/obstacle.hpp:9-34)."""
    _fields_ = [("shape", C.c_int), ("center_i", C.c_int), ("center_j", C.c_int), ("half_i", C.c_int),
                ("half_j", C.c_int), ("radius", C.c_int), ("rho", C.c_double), ("pressure", C.c_double),
                ("ux", C.c_double), ("uy", C.c_double), ("move_di", C.c_int), ("move_dj", C.c_int)]

    def __init__(self, shape=HK_OBSTACLE_NONE, center_i=0, center_j=0, half_i=0, half_j=0, radius=0, rho=1.0,
                 pressure=1.0, ux=0.0, uy=0.0, move_di=0, move_dj=0):
        super().__init__(shape, center_i, center_j, half_i, half_j, radius, rho, pressure, ux, uy, move_di, move_dj)

    def enabled(self) -> bool:
        return self.shape != HK_OBSTACLE_NONE

    def temperature(self) -> float:
        return self.pressure / self.rho

class HybridParams(C.Structure):
    """hk_hybrid_params (include/hykin_b200.h): thresholds, physics and collision flags of hk_hybrid_step."""
    _fields_ = [("eta0", C.c_double), ("eta1", C.c_double), ("delta0", C.c_double), ("mu0", C.c_double),
                ("kappa0", C.c_double), ("signed_sum", C.c_int), ("update_regimes", C.c_int),
                ("heat_ratio", C.c_double), ("esbgk_beta", C.c_double), ("nu_coeff", C.c_double),
                ("pen_coeff", C.c_double), ("eps_weno", C.c_double), ("coll_flags", C.c_uint32),
                ("ghost_x", C.c_int), ("residual_fn", C.c_void_p), ("residual_user", C.c_void_p)]


# int (*)(void* user, const double* y, double* res, int64_t m2, int* status, void* stream)
RESIDUAL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


_lib = None


def lib() -> C.CDLL:
    """Loads libhykin_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2505_03360_b200/csrc` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, u32, dbl = C.c_void_p, C.c_int64, C.c_uint32, C.c_double
    sig = {
        "hk_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "hk_ctx_destroy": (C.c_int, [vp]),
        "hk_ctx_set_stream": (C.c_int, [vp, vp]),
        "hk_ctx_trim": (C.c_int, [vp]),
        "hk_last_error": (C.c_int, [vp, C.POINTER(i64), C.c_char_p, C.c_size_t]),
        "hk_launch_count": (i64, [vp]),
        "hk_ctx_set_timing": (C.c_int, [vp, C.c_int]),
        "hk_device_alloc": (C.c_int, [vp, C.c_size_t, C.POINTER(vp)]),
        "hk_device_free": (C.c_int, [vp, vp]),
        "hk_copy_to_device": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "hk_copy_to_host": (C.c_int, [vp, vp, vp, C.c_size_t]),
        "hk_ctx_synchronize": (C.c_int, [vp]),
        "hk_ctx_timing_report": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(i64)]),
        "hk_kernel_create": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dbl, dbl, C.POINTER(vp)]),
        "hk_kernel_create_from_tables": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dbl, dbl, vp, vp, vp,
                                                   C.POINTER(vp)]),
        "hk_kernel_destroy": (C.c_int, [vp]),
        "hk_kernel_info": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "hk_collision_batch": (C.c_int, [vp, vp, vp, vp, i64, u32, vp]),
        "hk_collision_batch_host": (C.c_int, [vp, vp, vp, vp, i64, u32, vp]),
        "hk_measure_fp64_peak": (dbl, [vp]),
        "hk_moments_batch": (C.c_int, [vp, C.c_int, dbl, vp, i64, vp, vp, vp, vp, vp]),
        "hk_maxwellian_batch": (C.c_int, [vp, C.c_int, dbl, vp, i64, vp, vp]),
        "hk_anisotropic_gaussian_batch": (C.c_int, [vp, C.c_int, dbl, vp, vp, dbl, i64, vp, vp]),
        "hk_match_moments_batch": (C.c_int, [vp, C.c_int, dbl, vp, vp, i64, vp]),
        "hk_remove_invariant_moments_batch": (C.c_int, [vp, C.c_int, dbl, vp, vp, vp, i64, vp]),
        "hk_esbgk_stage_batch": (C.c_int, [vp, C.c_int, dbl, vp, vp, i64, dbl, vp, dbl, dbl, dbl, vp, vp]),
        "hk_penalized_stage_batch": (C.c_int, [vp, C.c_int, dbl, vp, vp, i64, dbl, vp, dbl, dbl, vp, vp]),
        "hk_penalized_residual_batch": (C.c_int, [vp, vp, vp, vp, i64, dbl, u32, vp, vp]),
        "hk_classify": (C.c_int, [vp, C.c_int, C.c_int, dbl, dbl, vp, vp, vp, vp, vp, vp, vp, dbl, dbl, dbl, dbl,
                                  dbl, C.c_int]),
        "hk_transport_rhs": (C.c_int, [vp, C.c_int, dbl, vp, vp, C.c_int, C.c_int, C.c_int, dbl, dbl, dbl]),
        "hk_esbgk_imex_step": (C.c_int, [vp, C.c_int, dbl, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, dbl, dbl, dbl,
                                         vp]),
        "hk_penalized_imex_step": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, dbl, dbl, u32, vp]),
        "hk_penalized_imex_step_slab": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, dbl, dbl, u32, vp]),
        "hk_esbgk_imex_step_slab": (C.c_int, [vp, C.c_int, dbl, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, dbl, dbl, dbl,
                                              vp]),
        "hk_axpby": (C.c_int, [vp, i64, vp, vp, dbl, vp, dbl, vp]),
        "hk_transport_rhs_slab": (C.c_int, [vp, C.c_int, dbl, vp, vp, vp, vp, C.c_int, C.c_int, dbl, dbl, dbl]),
        "hk_imex_combine": (C.c_int, [vp, C.c_int, i64, i64, dbl, vp, vp, vp, vp, vp, vp, vp, vp]),
        "hk_euler_rhs_periodic": (C.c_int, [vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, vp]),
        "hk_euler_tvd_rk2_step": (C.c_int, [vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl, vp]),
        "hk_conserved_to_maxwellian": (C.c_int, [vp, C.c_int, dbl, vp, i64, dbl, vp]),
        "hk_distribution_to_conserved": (C.c_int, [vp, C.c_int, dbl, vp, i64, dbl, vp]),
        "hk_gather_cells": (C.c_int, [vp, i64, vp, vp, i64, vp]),
        "hk_scatter_cells": (C.c_int, [vp, i64, vp, vp, i64, vp]),
        "hk_transport_rhs_peer": (C.c_int, [vp, C.c_int, dbl, vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
                                            dbl, dbl, dbl]),
        "hk_ipc_handle": (C.c_int, [vp, vp, vp, C.POINTER(C.c_int64)]),
        "hk_ipc_open": (C.c_int, [vp, vp, C.POINTER(C.c_void_p)]),
        "hk_ipc_close": (C.c_int, [vp, vp]),
        "hk_comm_unique_id": (C.c_int, [vp]),
        "hk_ctx_comm_init": (C.c_int, [vp, C.c_int, C.c_int, vp]),
        "hk_ctx_comm_info": (C.c_int, [vp, vp, vp]),
        "hk_halo_exchange": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp]),
        "hk_allreduce_scalars": (C.c_int, [vp, vp, i64, C.c_int]),
        "hk_classify_cells": (C.c_int, [vp, i64, i64, C.POINTER(ObstacleSpec), vp]),
        "hk_synthesize_hydro": (C.c_int, [vp, C.c_int, dbl, i64, i64, C.POINTER(ObstacleSpec), vp, vp, vp, vp, dbl,
                                          vp]),
        "hk_synthesize_distributions": (C.c_int, [vp, C.c_int, dbl, i64, i64, C.POINTER(ObstacleSpec), vp, vp, vp, vp,
                                                  dbl, vp, i64, vp, C.POINTER(C.c_int64)]),
        "hk_write_snapshot": (C.c_int, [vp, C.c_int, dbl, i64, i64, dbl, dbl, vp, vp, vp, vp, dbl, i64, dbl,
                                        C.c_char_p, C.c_char_p]),
        "hk_hybrid_step": (C.c_int, [vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, vp, vp, vp, C.POINTER(HybridParams),
                                     C.POINTER(C.c_int64)]),
        "hk_hybrid_step_slab": (C.c_int, [vp, vp, C.c_int, C.c_int, dbl, dbl, dbl, vp, vp, vp, vp,
                                          C.POINTER(HybridParams), C.c_int, C.POINTER(C.c_int64)]),
        "hk_apply_obstacle": (C.c_int, [vp, C.c_int, dbl, C.POINTER(ObstacleSpec), i64, i64, vp, vp, vp, vp, dbl,
                                        C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols_from_header(path: str = HEADER) -> list[str]:
    """Function names declared in include/hykin_b200.h."""
    import re

    text = open(path).read()
    return sorted(set(re.findall(r"\b(hk_[a-z0-9_]+)\s*\(", text)))
