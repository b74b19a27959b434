"""ctypes front-end for the CPU checker — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2505_03360_b200) never does.

Two libraries are exposed:

* :class:`Oracle`  — ``oracle/liboracle.so``, the C restatement
  (``oracle/hk_oracle.c``), each function citing the reference file:line.
* :class:`RefLib`  — ``oracle/_ref/libhykin_ref.so``, the reference's own
  sources compiled with the FFTW3/Eigen API shims (``oracle/Makefile``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhykin_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.int32:
        return a.ctypes.data_as(_ip)
    raise TypeError(a.dtype)


class _Kernel(C.Structure):
    _fields_ = [
        ("n", C.c_int), ("a1", C.c_int), ("a2", C.c_int),
        ("vmax", C.c_double), ("r_phys", C.c_double), ("r", C.c_double),
        ("jacobian", C.c_double), ("weight", C.c_double),
        ("alpha", _dp), ("alpha_prime", _dp), ("loss_diag", _dp),
    ]


class _Moments(C.Structure):
    _fields_ = [("rho", C.c_double), ("u", C.c_double * 3), ("T", C.c_double)]


class Obstacle(C.Structure):
    """hko_obstacle / ObstacleSpec (inc/hykin/obstacle.hpp); shape 0 none, 1 rectangle, 2 disk."""
    _fields_ = [("shape", C.c_int), ("center_i", C.c_int), ("center_j", C.c_int), ("half_i", C.c_int),
                ("half_j", C.c_int), ("radius", C.c_int), ("rho", C.c_double), ("pressure", C.c_double),
                ("ux", C.c_double), ("uy", C.c_double), ("move_di", C.c_int), ("move_dj", C.c_int)]

    def copy(self):
        o = Obstacle()
        C.pointer(o)[0] = self
        return o


def build(quiet: bool = True) -> None:
    """Builds liboracle.so (and _ref when /root/reference is present)."""
    import subprocess

    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class OracleKernel:
    """Owns an ``hko_kernel`` (weight tables of src/spectral.cpp:53-112)."""

    def __init__(self, lib, n, vmax, a1, a2, r_phys, closed_form=True, nthreads=8):
        self._lib = lib
        self._k = _Kernel()
        st = lib.hko_precompute(n, C.c_double(vmax), a1, a2, C.c_double(r_phys),
                                int(bool(closed_form)), nthreads, C.byref(self._k))
        self.status = st
        if st:
            self._k = None
            return
        self.n, self.a1, self.a2, self.vmax = n, a1, a2, vmax
        total = n ** 3
        d = a1 * a2
        self.alpha = np.ctypeslib.as_array(self._k.alpha, shape=(d, total)).copy()
        self.alpha_prime = np.ctypeslib.as_array(self._k.alpha_prime, shape=(d, total)).copy()
        self.loss_diag = np.ctypeslib.as_array(self._k.loss_diag, shape=(total,)).copy()
        self.r, self.jacobian, self.weight = self._k.r, self._k.jacobian, self._k.weight

    def __del__(self):
        if getattr(self, "_k", None) is not None:
            self._lib.hko_kernel_free(C.byref(self._k))
            self._k = None

    @property
    def ref(self):
        return C.byref(self._k)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.hko_precompute.restype = C.c_int
        L.hko_spectral_collision.restype = C.c_int
        L.hko_collision_batch.restype = C.c_int
        L.hko_closed_radial.restype = C.c_double
        L.hko_closed_planar.restype = C.c_double
        L.hko_gk15_radial.restype = C.c_double
        L.hko_gk15_planar.restype = C.c_double
        L.hko_node.restype = C.c_double
        L.hko_lambda_b.restype = C.c_double
        for fn in ("hko_closed_radial", "hko_closed_planar", "hko_gk15_radial", "hko_gk15_planar"):
            getattr(L, fn).argtypes = [C.c_double, C.c_double, C.c_double]

    # --- kernel / collision -------------------------------------------------
    def kernel(self, n, vmax, a1, a2, r_phys, closed_form=True, nthreads=8):
        return OracleKernel(self.lib, n, vmax, a1, a2, r_phys, closed_form, nthreads)

    def collision(self, k: OracleKernel, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.empty_like(f)
        res = C.c_double(0.0)
        st = self.lib.hko_spectral_collision(k.ref, _ptr(f), _ptr(out), C.byref(res))
        return out, st, res.value

    def collision_batch(self, k: OracleKernel, f, nthreads=8):
        f = np.ascontiguousarray(f, dtype=np.float64)
        nb = k.n ** 3
        ncells = f.size // nb
        q = np.empty_like(f)
        st = np.zeros(ncells, np.int32)
        res = np.zeros(ncells, np.float64)
        self.lib.hko_collision_batch(k.ref, _ptr(f), _ptr(q), C.c_long(ncells), nthreads,
                                     _ptr(st), _ptr(res))
        return q, st, res

    def fft3d(self, x, sign):
        x = np.ascontiguousarray(x, dtype=np.complex128).copy()
        n = round(x.size ** (1 / 3))
        self.lib.hko_fft_3d(n, x.ctypes.data_as(_dp), sign)
        return x

    # --- moments ------------------------------------------------------------
    def moments(self, n, vmax, f):
        m = _Moments()
        f = np.ascontiguousarray(f, dtype=np.float64)
        st = self.lib.hko_moments_of(n, C.c_double(vmax), _ptr(f), C.byref(m))
        return st, (m.rho, m.u[0], m.u[1], m.u[2], m.T)

    def second_moment(self, n, vmax, f):
        s = np.zeros(9)
        self.lib.hko_second_moment(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f)), _ptr(s))
        return s.reshape(3, 3)

    def maxwellian(self, n, vmax, mom5):
        m = _Moments(mom5[0], (C.c_double * 3)(*mom5[1:4]), mom5[4])
        out = np.empty(n ** 3)
        st = self.lib.hko_maxwellian(C.byref(m), n, C.c_double(vmax), _ptr(out))
        return st, out

    def realizability(self, n, vmax, f):
        st, mom = self.moments(n, vmax, f)
        m = _Moments(mom[0], (C.c_double * 3)(*mom[1:4]), mom[4])
        a = np.zeros(9); b = np.zeros(3); c = C.c_double(0.0)
        self.lib.hko_realizability_matrix(_ptr(np.ascontiguousarray(f)), n, C.c_double(vmax),
                                          C.byref(m), _ptr(a), _ptr(b), C.byref(c))
        return st, a.reshape(3, 3), b, c.value

    def match_moments(self, n, vmax, f, rho, mom3, energy):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        m3 = np.ascontiguousarray(mom3, dtype=np.float64)
        st = self.lib.hko_match_moments(_ptr(f), n, C.c_double(vmax), C.c_double(rho), _ptr(m3),
                                        C.c_double(energy))
        return st, f

    def stress_tensor(self, n, vmax, f, mom5):
        m = _Moments(mom5[0], (C.c_double * 3)(*mom5[1:4]), mom5[4])
        th = np.zeros(9)
        self.lib.hko_stress_tensor(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f, dtype=np.float64)),
                                   C.byref(m), _ptr(th))
        return th.reshape(3, 3)

    def anisotropic_gaussian(self, n, vmax, mom5, theta, beta):
        m = _Moments(mom5[0], (C.c_double * 3)(*mom5[1:4]), mom5[4])
        out = np.empty(n ** 3)
        fb = C.c_int(0)
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(9)
        st = self.lib.hko_anisotropic_gaussian(C.byref(m), _ptr(th), C.c_double(beta), n, C.c_double(vmax),
                                               _ptr(out), C.byref(fb))
        return st, out, fb.value

    def remove_invariant_moments(self, n, vmax, q, weight, uc):
        q = np.ascontiguousarray(q, dtype=np.float64).copy()
        st = self.lib.hko_remove_invariant_moments(_ptr(q), _ptr(np.ascontiguousarray(weight, dtype=np.float64)), n,
                                                   C.c_double(vmax), _ptr(np.ascontiguousarray(uc, dtype=np.float64)))
        return st, q

    def penalized_residual(self, k: OracleKernel, f, pen_coeff=2 * np.pi):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.empty_like(f)
        res = C.c_double(0.0)
        st = self.lib.hko_penalized_residual(k.ref, _ptr(f), C.c_double(pen_coeff), _ptr(out),
                                             C.byref(res))
        return out, st, res.value

    def penalized_stage_solve(self, n, vmax, f_star, a, eps, pen_coeff=2 * np.pi):
        f_star = np.ascontiguousarray(f_star, dtype=np.float64)
        out = np.empty_like(f_star)
        m = _Moments()
        st = self.lib.hko_penalized_stage_solve(_ptr(f_star), C.c_double(a), C.c_double(eps),
                                                C.c_double(pen_coeff), n, C.c_double(vmax),
                                                _ptr(out), C.byref(m))
        return out, st

    def esbgk_stage_solve(self, n, vmax, f_star, a, eps, beta=-0.5, nu_coeff=0.5 * np.pi):
        f_star = np.ascontiguousarray(f_star, dtype=np.float64)
        out = np.empty_like(f_star)
        m = _Moments()
        fb = C.c_int(0)
        st = self.lib.hko_esbgk_stage_solve(_ptr(f_star), C.c_double(a), C.c_double(eps),
                                            C.c_double(beta), C.c_double(nu_coeff), n,
                                            C.c_double(vmax), _ptr(out), C.byref(m), C.byref(fb))
        return out, st, fb.value

    def l1_distance(self, n, vmax, f):
        out = C.c_double(0.0)
        st = self.lib.hko_l1_distance(_ptr(np.ascontiguousarray(f)), n, C.c_double(vmax),
                                      C.byref(out))
        return st, out.value

    def indicators(self, prim5x4, dx, dy, eps, mu0=1.0, kappa0=1.0, signed_sum=False):
        p = np.ascontiguousarray(prim5x4, dtype=np.float64).reshape(5, 4)
        d = np.zeros(11)
        rows = [np.ascontiguousarray(p[i]) for i in range(5)]
        self.lib.hko_spatial_derivatives(*[_ptr(r) for r in rows], C.c_double(dx), C.c_double(dy),
                                         _ptr(d))
        lam = np.zeros(3)
        self.lib.hko_v_eps1_eigenvalues(_ptr(d), _ptr(rows[0]), C.c_double(eps), C.c_double(mu0),
                                        C.c_double(kappa0), _ptr(lam))
        lb = self.lib.hko_lambda_b(_ptr(d), _ptr(rows[0]), C.c_double(eps), int(signed_sum))
        return d, lam, lb

    def regime_update(self, r, lam=None, lambda_b=None, l1=None, eta0=1e-3, eta1=1e-2,
                      delta0=1e-3):
        lam_a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
        lb = None if lambda_b is None else C.byref(C.c_double(lambda_b))
        l1p = None if l1 is None else C.byref(C.c_double(l1))
        out = C.c_int(-1)
        st = self.lib.hko_regime_update(r, _ptr(lam_a) if lam_a is not None else None, lb, l1p,
                                        C.c_double(eta0), C.c_double(eta1), C.c_double(delta0),
                                        C.byref(out))
        return st, out.value

    def transport_rhs_periodic(self, f, nx, ny, n, vmax, dx, dy, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.empty_like(f)
        self.lib.hko_transport_rhs_periodic(_ptr(f), nx, ny, n, C.c_double(vmax), C.c_double(dx),
                                            C.c_double(dy), C.c_double(eps_weno), _ptr(out))
        return out

    # ---- Layer-0 Euler (src/euler.cpp:159-181), transitions (src/coupling.cpp:7-22) ----
    def euler_rhs_periodic(self, u, nx, ny, dx, dy, xi=5.0 / 3.0, eps_weno=1e-6):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        bad = C.c_long(-1)
        st = self.lib.hko_euler_rhs_periodic(_ptr(u), nx, ny, C.c_double(dx), C.c_double(dy), C.c_double(xi),
                                             C.c_double(eps_weno), _ptr(out), C.byref(bad))
        return st, out, bad.value

    def tvd_rk2_step_periodic(self, u, nx, ny, dx, dy, dt, xi=5.0 / 3.0, eps_weno=1e-6):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        bad = C.c_long(-1)
        st = self.lib.hko_tvd_rk2_step_periodic(_ptr(u), nx, ny, C.c_double(dx), C.c_double(dy), C.c_double(dt),
                                                C.c_double(xi), C.c_double(eps_weno), C.byref(bad))
        return st, u

    def moments_from_conserved(self, u4, heat_ratio=5.0 / 3.0):
        u4 = np.ascontiguousarray(u4, dtype=np.float64)
        m = np.zeros(5)
        st = self.lib.hko_moments_from_conserved(_ptr(u4), C.c_double(heat_ratio), _ptr(m))
        return st, m

    def conserved_from_moments(self, mom5, heat_ratio=5.0 / 3.0):
        mom5 = np.ascontiguousarray(mom5, dtype=np.float64)
        u = np.zeros(4)
        self.lib.hko_conserved_from_moments(_ptr(mom5), C.c_double(heat_ratio), _ptr(u))
        return u

    # --- obstacles (src/grid.cpp:56-110, src/coupling.cpp:95-147) -----------
    def classify_cells(self, nx, ny, spec):
        kind = np.zeros(nx * ny, dtype=np.uint8)
        bad = C.c_long(-1)
        st = self.lib.hko_classify_cells(nx, ny, C.byref(spec), kind.ctypes.data_as(C.c_void_p), C.byref(bad))
        return st, kind, bad.value

    def apply_obstacle(self, nx, ny, n, vmax, spec, r, kind, hydro, f, heat_ratio=5.0 / 3.0):
        """In-place on copies; returns (status, spec, r, kind, hydro, f, covered, vacated)."""
        spec = spec.copy()
        r = np.ascontiguousarray(r, dtype=np.int8).copy()
        kind = np.ascontiguousarray(kind, dtype=np.uint8).copy()
        hydro = np.ascontiguousarray(hydro, dtype=np.float64).copy()
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        cov, vac = C.c_int(0), C.c_int(0)
        st = self.lib.hko_apply_obstacle(nx, ny, n, C.c_double(vmax), C.byref(spec), r.ctypes.data_as(C.c_void_p),
                                         kind.ctypes.data_as(C.c_void_p), _ptr(hydro), _ptr(f),
                                         C.c_double(heat_ratio), C.byref(cov), C.byref(vac))
        return st, spec, r, kind, hydro, f, cov.value, vac.value

    def synthesize(self, which, nx, ny, n, vmax, spec, r, kind, hydro, f, cells, heat_ratio=5.0 / 3.0):
        """synthesize_hydro_state (which 0, -> [k,4]) / synthesize_distribution (which 1,
        -> [k,n^3]) at the (i, j) pairs `cells`; returns (first failing status, out)."""
        r = np.ascontiguousarray(r, dtype=np.int8)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        hydro = np.ascontiguousarray(hydro, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        width = 4 if which == 0 else n ** 3
        out = np.zeros((len(cells), width))
        fn = self.lib.hko_synthesize_hydro_state if which == 0 else self.lib.hko_synthesize_distribution
        sp = C.byref(spec) if spec is not None else None
        for k, (i, j) in enumerate(cells):
            row = np.zeros(width)
            st = fn(nx, ny, n, C.c_double(vmax), sp, r.ctypes.data_as(C.c_void_p), kind.ctypes.data_as(C.c_void_p),
                    _ptr(hydro), _ptr(f), C.c_double(heat_ratio), int(i), int(j), _ptr(row))
            if st:
                return st, out
            out[k] = row
        return 0, out

    def penalized_imex_step(self, k: OracleKernel, f, nx, ny, dx, dy, dt, eps_cell,
                            pen_coeff=2 * np.pi, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        e = np.ascontiguousarray(eps_cell, dtype=np.float64)
        st = self.lib.hko_penalized_imex_step(_ptr(f), nx, ny, k.ref, C.c_double(dx),
                                              C.c_double(dy), C.c_double(dt), _ptr(e),
                                              C.c_double(pen_coeff), C.c_double(eps_weno), 1)
        return f, st

    def esbgk_imex_step(self, f, nx, ny, n, vmax, dx, dy, dt, eps_cell, beta=-0.5,
                        nu_coeff=0.5 * np.pi, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        e = np.ascontiguousarray(eps_cell, dtype=np.float64)
        st = self.lib.hko_esbgk_imex_step(_ptr(f), nx, ny, n, C.c_double(vmax), C.c_double(dx),
                                          C.c_double(dy), C.c_double(dt), _ptr(e),
                                          C.c_double(beta), C.c_double(nu_coeff),
                                          C.c_double(eps_weno), 1)
        return f, st

    def hybrid_step(self, k: OracleKernel, nx, ny, dx, dy, dt, eps_cell, r, hydro, f, params):
        """hko_hybrid_step on copies; params = paper_2505_03360_b200.HybridParams-like object
        with the hko_hybrid_params fields.  Returns (status, r, hydro, f, counts[6])."""
        r = np.ascontiguousarray(r, dtype=np.int8).copy()
        hydro = np.ascontiguousarray(hydro, dtype=np.float64).copy()
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        e = np.ascontiguousarray(eps_cell, dtype=np.float64)
        hp = HkoHybridParams(params.eta0, params.eta1, params.delta0, params.mu0, params.kappa0,
                             int(params.signed_sum), int(params.update_regimes), params.heat_ratio,
                             params.esbgk_beta, params.nu_coeff, params.pen_coeff, params.eps_weno)
        counts = np.zeros(6, dtype=np.int64)
        st = self.lib.hko_hybrid_step(nx, ny, k.ref, C.c_double(dx), C.c_double(dy), C.c_double(dt), _ptr(e),
                                      r.ctypes.data_as(C.c_void_p), _ptr(hydro), _ptr(f), C.byref(hp),
                                      counts.ctypes.data_as(C.c_void_p))
        return st, r, hydro, f, counts


class HkoHybridParams(C.Structure):
    """hko_hybrid_params (oracle/hk_oracle.h)."""
    _fields_ = [("eta0", C.c_double), ("eta1", C.c_double), ("delta0", C.c_double), ("mu0", C.c_double),
                ("kappa0", C.c_double), ("signed_sum", C.c_int), ("update_regimes", C.c_int),
                ("heat_ratio", C.c_double), ("esbgk_beta", C.c_double), ("nu_coeff", C.c_double),
                ("pen_coeff", C.c_double), ("eps_weno", C.c_double)]


class RefKernel:
    def __init__(self, lib, n, vmax, a1, a2, r_phys, tables=None):
        self._lib = lib
        st = C.c_int(0)
        if tables is None:
            lib.href_kernel_create.restype = C.c_void_p
            self.h = lib.href_kernel_create(n, C.c_double(vmax), a1, a2, C.c_double(r_phys),
                                            C.byref(st))
        else:  # (alpha [d, n^3], alpha_prime [d, n^3], loss [n^3]) supplied, e.g. OracleKernel's
            a, ap, ld = (np.ascontiguousarray(x, dtype=np.float64) for x in tables)
            lib.href_kernel_from_tables.restype = C.c_void_p
            self.h = lib.href_kernel_from_tables(n, C.c_double(vmax), a1, a2, C.c_double(r_phys),
                                                 _ptr(a), _ptr(ap), _ptr(ld))
        self.status = st.value
        self.n, self.a1, self.a2, self.vmax = n, a1, a2, vmax

    def tables(self):
        d, total = self.a1 * self.a2, self.n ** 3
        a = np.empty((d, total)); ap = np.empty((d, total)); ld = np.empty(total)
        self._lib.href_kernel_tables(C.c_void_p(self.h), _ptr(a), _ptr(ap), _ptr(ld))
        sc = np.empty(4)
        self._lib.href_kernel_scalars(C.c_void_p(self.h), _ptr(sc))
        return a, ap, ld, sc

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.href_kernel_free(C.c_void_p(self.h))
            self.h = None


class RefLib:
    """The reference's own code (oracle/_ref/libhykin_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)

    def kernel(self, n, vmax, a1, a2, r_phys, tables=None):
        return RefKernel(self.lib, n, vmax, a1, a2, r_phys, tables)

    def collision_batch(self, k: RefKernel, f, nthreads=1):
        f = np.ascontiguousarray(f, dtype=np.float64)
        ncells = f.size // k.n ** 3
        q = np.empty_like(f)
        st = np.zeros(ncells, np.int32)
        self.lib.href_collision_batch(C.c_void_p(k.h), _ptr(f), _ptr(q), C.c_int64(ncells),
                                      nthreads, _ptr(st))
        return q, st

    def penalized_residual_batch(self, k: RefKernel, f, pen_coeff=2 * np.pi, nthreads=1):
        f = np.ascontiguousarray(f, dtype=np.float64)
        ncells = f.size // k.n ** 3
        out = np.empty_like(f)
        st = np.zeros(ncells, np.int32)
        self.lib.href_penalized_residual_batch(C.c_void_p(k.h), _ptr(f), _ptr(out),
                                               C.c_int64(ncells), C.c_double(pen_coeff), nthreads,
                                               _ptr(st))
        return out, st

    def moments(self, n, vmax, f):
        m = np.zeros(5)
        st = self.lib.href_moments(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f)), _ptr(m))
        return st, tuple(m)

    def second_moment(self, n, vmax, f):
        s = np.zeros(9)
        self.lib.href_second_moment(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f)), _ptr(s))
        return s.reshape(3, 3)

    def maxwellian(self, n, vmax, mom5):
        out = np.empty(n ** 3)
        st = self.lib.href_maxwellian(n, C.c_double(vmax), _ptr(np.asarray(mom5, np.float64)),
                                      _ptr(out))
        return st, out

    def realizability(self, n, vmax, f):
        o = np.zeros(13)
        st = self.lib.href_realizability(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f)), _ptr(o))
        return st, o[:9].reshape(3, 3), o[9:12], o[12]

    def match_moments(self, n, vmax, f, rho, mom3, energy):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        st = self.lib.href_match_moments(n, C.c_double(vmax), _ptr(f), C.c_double(rho),
                                         _ptr(np.asarray(mom3, np.float64)), C.c_double(energy))
        return st, f

    def penalized_stage_solve(self, n, vmax, f_star, a, eps, pen_coeff=2 * np.pi):
        f_star = np.ascontiguousarray(f_star, dtype=np.float64)
        out = np.empty_like(f_star)
        m = np.zeros(5)
        st = self.lib.href_penalized_stage_solve(n, C.c_double(vmax), _ptr(f_star), C.c_double(a),
                                                 C.c_double(eps), C.c_double(pen_coeff), _ptr(out),
                                                 _ptr(m))
        return out, st

    def esbgk_stage_solve(self, n, vmax, f_star, a, eps, beta=-0.5, nu_coeff=0.5 * np.pi):
        f_star = np.ascontiguousarray(f_star, dtype=np.float64)
        out = np.empty_like(f_star)
        m = np.zeros(5)
        fb = C.c_int(0)
        st = self.lib.href_esbgk_stage_solve(n, C.c_double(vmax), _ptr(f_star), C.c_double(a),
                                             C.c_double(eps), C.c_double(beta),
                                             C.c_double(nu_coeff), _ptr(out), _ptr(m), C.byref(fb))
        return out, st, fb.value

    def esbgk_stage_batch(self, n, vmax, f_star, a, eps_cell, beta=-0.5, nu_coeff=0.5 * np.pi,
                          nthreads=1):
        f_star = np.ascontiguousarray(f_star, dtype=np.float64)
        ncells = f_star.size // n ** 3
        out = np.empty_like(f_star)
        st = np.zeros(ncells, np.int32)
        fb = np.zeros(ncells, np.int32)
        self.lib.href_esbgk_stage_batch(n, C.c_double(vmax), _ptr(f_star), _ptr(out),
                                        C.c_int64(ncells), C.c_double(a),
                                        _ptr(np.ascontiguousarray(eps_cell, dtype=np.float64)),
                                        C.c_double(beta), C.c_double(nu_coeff), nthreads,
                                        _ptr(st), _ptr(fb))
        return out, st, fb

    def l1_distance(self, n, vmax, f):
        out = C.c_double(0.0)
        st = self.lib.href_l1_distance(n, C.c_double(vmax), _ptr(np.ascontiguousarray(f)),
                                       C.byref(out))
        return st, out.value

    def indicators(self, prim5x4, dx, dy, eps, mu0=1.0, kappa0=1.0, signed_sum=False):
        lam = np.zeros(3)
        lb = C.c_double(0.0)
        self.lib.href_indicators(_ptr(np.ascontiguousarray(prim5x4, dtype=np.float64).ravel()),
                                 C.c_double(dx), C.c_double(dy), C.c_double(eps), C.c_double(mu0),
                                 C.c_double(kappa0), int(signed_sum), _ptr(lam), C.byref(lb))
        return lam, lb.value

    def regime_update(self, r, lam=None, lambda_b=None, l1=None, eta0=1e-3, eta1=1e-2,
                      delta0=1e-3):
        mask = (lam is not None) | ((lambda_b is not None) << 1) | ((l1 is not None) << 2)
        lam_a = np.asarray(lam if lam is not None else [0, 0, 0], np.float64)
        out = C.c_int(-1)
        st = self.lib.href_regime_update(r, mask, _ptr(lam_a), C.c_double(lambda_b or 0.0),
                                         C.c_double(l1 or 0.0), C.c_double(eta0), C.c_double(eta1),
                                         C.c_double(delta0), C.byref(out))
        return st, out.value

    def transport_rhs_periodic(self, f, nx, ny, n, vmax, dx, dy, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.empty_like(f)
        self.lib.href_transport_rhs_periodic(n, C.c_double(vmax), _ptr(f), nx, ny, C.c_double(dx),
                                             C.c_double(dy), C.c_double(eps_weno), _ptr(out))
        return out

    # ---- Layer-0 Euler and transitions, the reference's own code ----
    def euler_rhs_periodic(self, u, nx, ny, dx, dy, xi=5.0 / 3.0, eps_weno=1e-6):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        st = self.lib.href_euler_rhs_periodic(_ptr(u), nx, ny, C.c_double(dx), C.c_double(dy), C.c_double(xi),
                                              C.c_double(eps_weno), _ptr(out))
        return st, out

    def tvd_rk2_step_periodic(self, u, nx, ny, dx, dy, dt, xi=5.0 / 3.0, eps_weno=1e-6):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        st = self.lib.href_tvd_rk2_step_periodic(_ptr(u), nx, ny, C.c_double(dx), C.c_double(dy), C.c_double(dt),
                                                 C.c_double(xi), C.c_double(eps_weno))
        return st, u

    def moments_from_conserved(self, u4, heat_ratio=5.0 / 3.0):
        u4 = np.ascontiguousarray(u4, dtype=np.float64)
        m = np.zeros(5)
        st = self.lib.href_moments_from_conserved(_ptr(u4), C.c_double(heat_ratio), _ptr(m))
        return st, m

    def conserved_from_moments(self, mom5, heat_ratio=5.0 / 3.0):
        mom5 = np.ascontiguousarray(mom5, dtype=np.float64)
        u = np.zeros(4)
        self.lib.href_conserved_from_moments(_ptr(mom5), C.c_double(heat_ratio), _ptr(u))
        return u

    # --- obstacles ------------------------------------------------------------
    def classify_cells(self, nx, ny, spec):
        kind = np.zeros(nx * ny, dtype=np.uint8)
        st = self.lib.href_classify_cells(nx, ny, C.byref(spec), kind.ctypes.data_as(C.c_void_p))
        return st, kind

    def apply_obstacle(self, nx, ny, n, vmax, spec, r, kind, hydro, f, has, heat_ratio=5.0 / 3.0):
        """`has` marks the cells owning a distribution block (DistributionField::has)."""
        spec = spec.copy()
        r = np.ascontiguousarray(r, dtype=np.int8).copy()
        kind = np.ascontiguousarray(kind, dtype=np.uint8).copy()
        hydro = np.ascontiguousarray(hydro, dtype=np.float64).copy()
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        has = np.ascontiguousarray(has, dtype=np.uint8).copy()
        cov, vac = C.c_int(0), C.c_int(0)
        st = self.lib.href_apply_obstacle(nx, ny, n, C.c_double(vmax), C.byref(spec), r.ctypes.data_as(C.c_void_p),
                                          kind.ctypes.data_as(C.c_void_p), _ptr(hydro), _ptr(f),
                                          has.ctypes.data_as(C.c_void_p), C.c_double(heat_ratio), C.byref(cov),
                                          C.byref(vac))
        return st, spec, r, kind, hydro, f, has, cov.value, vac.value

    def synthesize(self, which, nx, ny, n, vmax, spec, r, kind, hydro, f, has, cells, heat_ratio=5.0 / 3.0):
        r = np.ascontiguousarray(r, dtype=np.int8)
        kind = np.ascontiguousarray(kind, dtype=np.uint8)
        hydro = np.ascontiguousarray(hydro, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        has = np.ascontiguousarray(has, dtype=np.uint8)
        ij = np.ascontiguousarray(np.asarray(cells, dtype=np.int32).reshape(-1, 2))
        ii, jj = np.ascontiguousarray(ij[:, 0]), np.ascontiguousarray(ij[:, 1])
        out = np.zeros((len(ij), 4 if which == 0 else n ** 3))
        st = self.lib.href_synthesize(which, nx, ny, n, C.c_double(vmax), C.byref(spec) if spec is not None else None,
                                      r.ctypes.data_as(C.c_void_p), kind.ctypes.data_as(C.c_void_p), _ptr(hydro),
                                      _ptr(f), has.ctypes.data_as(C.c_void_p), C.c_double(heat_ratio), _ptr(ii),
                                      _ptr(jj), len(ij), _ptr(out))
        return st, out

    def penalized_imex_step(self, k: RefKernel, f, nx, ny, dx, dy, dt, eps_cell,
                            pen_coeff=2 * np.pi, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        st = self.lib.href_penalized_imex_step(C.c_void_p(k.h), _ptr(f), nx, ny, C.c_double(dx),
                                               C.c_double(dy), C.c_double(dt),
                                               _ptr(np.ascontiguousarray(eps_cell, np.float64)),
                                               C.c_double(pen_coeff), C.c_double(eps_weno))
        return f, st

    def esbgk_imex_step(self, f, nx, ny, n, vmax, dx, dy, dt, eps_cell, beta=-0.5,
                        nu_coeff=0.5 * np.pi, eps_weno=1e-6):
        f = np.ascontiguousarray(f, dtype=np.float64).copy()
        st = self.lib.href_esbgk_imex_step(n, C.c_double(vmax), _ptr(f), nx, ny, C.c_double(dx),
                                           C.c_double(dy), C.c_double(dt),
                                           _ptr(np.ascontiguousarray(eps_cell, np.float64)),
                                           C.c_double(beta), C.c_double(nu_coeff),
                                           C.c_double(eps_weno))
        return f, st
