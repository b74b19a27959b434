"""Generates the golden fixtures from the REFERENCE's own code.

Run in the container that has /root/reference (oracle/_ref built by
`make -C oracle ref`): the reference sources, unmodified, compiled against
the FFTW3/Eigen API shims.  The fixtures are committed; the GPU box (no
/root/reference) checks the oracle and the CUDA path against them.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib  # noqa: E402
from paper_2505_03360_b200 import inputs  # noqa: E402

VMAX = 8.0


def euler(R):
    """Layer-0 Euler (src/euler.cpp:159-181) on config 4's smoothed quadrants."""
    nx, ny = 24, 20
    u = inputs.config4_conserved(nx, ny)
    st, rhs = R.euler_rhs_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny)
    st2, u1 = R.tvd_rk2_step_periodic(u, nx, ny, 1.0 / nx, 1.0 / ny, 2e-3)
    assert st == st2 == 0
    np.savez_compressed(os.path.join(HERE, "euler_cfg4.npz"), u=u, rhs=rhs, step=u1, nx=nx, ny=ny, dt=2e-3,
                        xi=5.0 / 3.0, eps_weno=1e-6)


def main():
    R = RefLib()
    if "--only-euler" in sys.argv:
        euler(R)
        return
    euler(R)
    # config 1 shapes: 16^3, M = 4 x 8, R = 2L/(3+sqrt2), hard spheres
    k = R.kernel(16, VMAX, 4, 8, inputs.R_PHYS_MAX)
    f = inputs.config1_cells(4, 16)
    q, st = R.collision_batch(k, f)
    res, rst = R.penalized_residual_batch(k, f)
    np.savez_compressed(os.path.join(HERE, "collision_n16_cfg1.npz"), f=f, q=q, status=st, residual=res,
                        residual_status=rst, n=16, a1=4, a2=8, vmax=VMAX, r_phys=inputs.R_PHYS_MAX)
    # config 2 shapes: 32^3, M = 8 x 8
    k = R.kernel(32, VMAX, 8, 8, inputs.R_PHYS_MAX)
    f = inputs.config2_cells(2, 32)
    q, st = R.collision_batch(k, f, nthreads=2)
    np.savez_compressed(os.path.join(HERE, "collision_n32_cfg2.npz"), f=f, q=q, status=st, n=32, a1=8, a2=8,
                        vmax=VMAX, r_phys=inputs.R_PHYS_MAX)
    # config 3 shapes at 16^3: moments, realizability, ES-BGK stage (a = dt = 1e-3, eps = 1e-2)
    n = 16
    f, fl = inputs.config3_cells(8, 8, n, cells=[0, 9, 27, 63])
    mom, real, es, fb, l1 = [], [], [], [], []
    for c in range(len(f)):
        mom.append(R.moments(n, VMAX, f[c])[1])
        _, a, b, cc = R.realizability(n, VMAX, f[c])
        real.append(np.concatenate([a.ravel(), b, [cc]]))
        out, s, fbk = R.esbgk_stage_solve(n, VMAX, f[c], 1e-3, 1e-2)
        es.append(out)
        fb.append(fbk)
        l1.append(R.l1_distance(n, VMAX, f[c])[1])
    np.savez_compressed(os.path.join(HERE, "esbgk_cfg3_n16.npz"), f=f, moments=np.array(mom),
                        realizability=np.array(real), esbgk=np.array(es), fallback=np.array(fb),
                        l1=np.array(l1), n=n, vmax=VMAX, a=1e-3, eps=1e-2, beta=-0.5, nu_coeff=0.5 * np.pi)
    # transport + ES-BGK IMEX step on a small periodic field (8^3 velocity grid)
    n, nx, ny = 8, 5, 4
    f, _ = inputs.config3_cells(nx, ny, n)
    t = R.transport_rhs_periodic(f, nx, ny, n, VMAX, 0.2, 0.25)
    eps = np.full(nx * ny, 1e-2)
    step, s = R.esbgk_imex_step(f, nx, ny, n, VMAX, 0.2, 0.25, 1e-3, eps)
    np.savez_compressed(os.path.join(HERE, "transport_n8.npz"), f=f, rhs=t, esbgk_step=step, nx=nx, ny=ny, n=n,
                        vmax=VMAX, dx=0.2, dy=0.25, dt=1e-3, eps=eps)
    # Algorithm 1 truth table (src/regime.cpp:25-52)
    rows = []
    for r in (0, 1, 2, 3):
        for lam in (None, [1.0, 1.0, 1.0], [1.0, 1.5, 1.0], [1.0005, 0.9995, 1.0]):
            for lb in (None, 0.0, 0.02, -0.02):
                for l1v in (None, 0.0, 0.5e-3, 2e-3):
                    st, out = R.regime_update(r, lam, lb, l1v, 1e-3, 1e-2, 1e-3)
                    rows.append(dict(r=r, lam=lam, lambda_b=lb, l1=l1v, status=st, out=out if st == 0 else None))
    with open(os.path.join(HERE, "regime_truth_table.json"), "w") as fh:
        json.dump(dict(eta0=1e-3, eta1=1e-2, delta0=1e-3, rows=rows), fh, indent=0)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
