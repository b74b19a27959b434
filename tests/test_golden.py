"""The oracle against the golden fixtures generated from the reference's own
code (tests/golden/make_golden.py).  CPU only; runs on the GPU box too."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def test_collision_n16(oracle):
    g = load("collision_n16_cfg1.npz")
    k = oracle.kernel(int(g["n"]), float(g["vmax"]), int(g["a1"]), int(g["a2"]), float(g["r_phys"]), closed_form=False)
    q, st, _ = oracle.collision_batch(k, g["f"])
    assert np.array_equal(q, g["q"])  # bitwise: same arithmetic, same stand-in FFT
    assert np.array_equal(st, g["status"])
    for c in range(len(g["f"])):
        r, s, _ = oracle.penalized_residual(k, g["f"][c])
        assert s == g["residual_status"][c] and rel(r, g["residual"][c]) < 1e-13


@pytest.mark.slow
def test_collision_n32(oracle):
    g = load("collision_n32_cfg2.npz")
    k = oracle.kernel(int(g["n"]), float(g["vmax"]), int(g["a1"]), int(g["a2"]), float(g["r_phys"]), closed_form=False)
    q, st, _ = oracle.collision_batch(k, g["f"], nthreads=2)
    assert np.array_equal(q, g["q"]) and np.array_equal(st, g["status"])


def test_esbgk_cfg3(oracle):
    g = load("esbgk_cfg3_n16.npz")
    n, vmax = int(g["n"]), float(g["vmax"])
    for c in range(len(g["f"])):
        s, m = oracle.moments(n, vmax, g["f"][c])
        assert s == 0 and np.allclose(m, g["moments"][c], rtol=1e-14, atol=1e-16)
        _, a, b, cc = oracle.realizability(n, vmax, g["f"][c])
        assert np.allclose(np.concatenate([a.ravel(), b, [cc]]), g["realizability"][c], atol=1e-13)
        out, s, fb = oracle.esbgk_stage_solve(n, vmax, g["f"][c], float(g["a"]), float(g["eps"]))
        assert s == 0 and fb == g["fallback"][c] and rel(out, g["esbgk"][c]) < 1e-13
        assert abs(oracle.l1_distance(n, vmax, g["f"][c])[1] - g["l1"][c]) < 1e-13


def test_transport_and_imex(oracle):
    g = load("transport_n8.npz")
    nx, ny, n, vmax = int(g["nx"]), int(g["ny"]), int(g["n"]), float(g["vmax"])
    t = oracle.transport_rhs_periodic(g["f"], nx, ny, n, vmax, float(g["dx"]), float(g["dy"]))
    assert np.array_equal(t, g["rhs"])
    s, st = oracle.esbgk_imex_step(g["f"], nx, ny, n, vmax, float(g["dx"]), float(g["dy"]), float(g["dt"]), g["eps"])
    assert st == 0 and rel(s, g["esbgk_step"]) < 1e-13


def test_regime_truth_table(oracle):
    with open(os.path.join(GOLD, "regime_truth_table.json")) as fh:
        t = json.load(fh)
    for row in t["rows"]:
        st, out = oracle.regime_update(row["r"], row["lam"], row["lambda_b"], row["l1"], t["eta0"], t["eta1"],
                                       t["delta0"])
        assert st == row["status"], row
        if st == 0:
            assert out == row["out"], row


def test_euler_cfg4(oracle):
    """Layer-0 Euler residual and TVD-RK2 step, bitwise the reference's."""
    g = load("euler_cfg4.npz")
    nx, ny = int(g["nx"]), int(g["ny"])
    st, rhs, _ = oracle.euler_rhs_periodic(g["u"], nx, ny, 1.0 / nx, 1.0 / ny, float(g["xi"]), float(g["eps_weno"]))
    assert st == 0 and np.array_equal(rhs, g["rhs"])
    st, u1 = oracle.tvd_rk2_step_periodic(g["u"], nx, ny, 1.0 / nx, 1.0 / ny, float(g["dt"]), float(g["xi"]),
                                          float(g["eps_weno"]))
    assert st == 0 and np.array_equal(u1, g["step"])
