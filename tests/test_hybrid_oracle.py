"""CPU checks of the hybrid-step restatement (oracle/hk_oracle.c:hko_hybrid_step).

The reference ships no step driver, so the restatement is pinned through its
limits: with the layer map frozen, a single-layer field must reproduce the
already-pinned single-layer steps bit for bit (TVD-RK2 src/euler.cpp:172-181,
ES-BGK PR(2,2,2) src/esbgk.cpp:47-99, penalized PR(2,2,2)
src/boltzmann.cpp:47-110), and with Algorithm 1 on, the transitions must be
the ones PAPER.md Algorithm 1 allows (no 0 <-> 2 jump)."""
import numpy as np
import pytest

from paper_2505_03360_b200 import inputs
from paper_2505_03360_b200.kinetic import HybridParams

NX, NY, N = 6, 5, 16


def _state(layer):
    rng = np.random.default_rng(11)
    cells = NX * NY
    rho = rng.uniform(0.6, 1.4, cells)
    T = rng.uniform(0.7, 1.3, cells)
    ux = rng.uniform(-0.2, 0.2, cells)
    uy = rng.uniform(-0.2, 0.2, cells)
    hydro = np.stack([rho, rho * ux, rho * uy, 1.5 * rho * T + 0.5 * rho * (ux * ux + uy * uy)], -1)
    f = np.stack([inputs.maxwellian(N, rho[c], (ux[c], uy[c], 0.0), T[c]) *
                  (1 + 0.05 * np.sin(np.arange(N ** 3) * (c + 1) * 1e-3)) for c in range(cells)])
    eps = rng.uniform(0.05, 0.2, cells)
    return hydro, eps, np.full(cells, layer, np.int8), f


@pytest.fixture(scope="module")
def okern(oracle):
    return oracle.kernel(N, inputs.VMAX, 4, 4, inputs.R_PHYS_MAX)


def _step(oracle, okern, layer, update=False):
    hydro, eps, r, f = _state(layer)
    dx, dy, dt = 1.0 / NX, 1.0 / NY, 2e-3
    p = HybridParams(update_regimes=update)
    st, r2, h2, f2, counts = oracle.hybrid_step(okern, NX, NY, dx, dy, dt, eps, r, hydro, f, p)
    return (hydro, eps, r, f, dx, dy, dt), (st, r2, h2, f2, counts)


def test_layer0_is_tvd_rk2(oracle, okern):
    (hydro, eps, r, f, dx, dy, dt), (st, r2, h2, f2, counts) = _step(oracle, okern, 0)
    assert st == 0 and list(counts[:3]) == [NX * NY, 0, 0]
    st_e, u = oracle.tvd_rk2_step_periodic(hydro, NX, NY, dx, dy, dt)
    assert st_e == 0
    assert np.array_equal(h2, u)
    assert np.array_equal(f2, f)  # no kinetic cell: no halo either


def test_layer1_is_esbgk_imex(oracle, okern):
    (hydro, eps, r, f, dx, dy, dt), (st, r2, h2, f2, counts) = _step(oracle, okern, 1)
    assert st == 0 and list(counts[:3]) == [0, NX * NY, 0] and counts[5] == 0
    ref, st_r = oracle.esbgk_imex_step(f, NX, NY, N, inputs.VMAX, dx, dy, dt, eps)
    assert st_r == 0
    assert np.array_equal(f2, ref)
    assert np.array_equal(h2, hydro)  # kinetic cells' hydro is not authoritative: untouched


def test_layer2_is_penalized_imex(oracle, okern):
    (hydro, eps, r, f, dx, dy, dt), (st, r2, h2, f2, counts) = _step(oracle, okern, 2)
    assert st == 0 and list(counts[:3]) == [0, 0, NX * NY]
    ref, st_r = oracle.penalized_imex_step(okern, f, NX, NY, dx, dy, dt, eps)
    assert st_r in (0, 4)  # numerical_consistency is reported, not fatal
    assert np.array_equal(f2, ref)


def test_algorithm1_transitions(oracle):
    nx, ny, n = 16, 12, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / 16)
    k = oracle.kernel(n, inputs.VMAX, 4, 4, inputs.R_PHYS_MAX)
    dx, dy = 1.0 / nx, 1.0 / ny
    dt = 0.5 * dx / (inputs.VMAX - inputs.VMAX / n)
    p = HybridParams()
    seen = set()
    for _ in range(2):
        st, r2, hydro, f, counts = oracle.hybrid_step(k, nx, ny, dx, dy, dt, eps, r, hydro, f, p)
        assert st == 0
        assert sum(counts[:3]) == nx * ny
        assert np.array_equal(np.bincount(r2, minlength=3), counts[:3])
        pairs = set(zip(r.tolist(), r2.tolist()))
        assert (0, 2) not in pairs and (2, 0) not in pairs  # Algorithm 1 moves one layer at a time
        assert counts[3] == int(np.sum((r == 0) & (r2 != 0))) and counts[4] == int(np.sum((r != 0) & (r2 == 0)))
        seen |= pairs
        r = r2
        kin = r2 != 0
        assert np.all(np.isfinite(f[kin])) and np.all(hydro[~kin, 0] > 0)
    assert (0, 1) in seen  # the run exercises a transition
