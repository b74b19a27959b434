"""Snapshot I/O: moments CSV, regime grid, metadata JSON of a
hybrid state, against the oracle's moments and the conserved-state primitives."""
import json
import os

import numpy as np
import pytest

from paper_2505_03360_b200 import inputs

pytestmark = pytest.mark.gpu


def test_snapshot_files(hk, oracle, tmp_path):
    import torch
    from paper_2505_03360_b200 import kinetic
    nx, ny, n = 8, 6, 16
    hydro, eps, r, f = inputs.config4_hybrid_state(nx, ny, n, half_width=1.0 / nx)
    vg = hk.make_velocity_grid(n, inputs.VMAX)
    kind = np.zeros(nx * ny, np.uint8)
    kind[3] = 1  # an obstacle cell (HK_CELL_OBSTACLE) -> -1 in the regime file
    rd, hd, fd = (torch.from_numpy(x.copy()).cuda() for x in (r, hydro, f))
    kd = torch.from_numpy(kind).cuda()
    kinetic.write_snapshot(tmp_path, 7, 0.125, vg, nx, ny, 1 / nx, 1 / ny, rd, hd, fd, kind=kd,
                           config={"scenario": 4, "eps_band": 0.1})
    rows = np.loadtxt(tmp_path / "moments_7.csv", delimiter=",", skiprows=1)
    assert rows.shape == (nx * ny, 9)
    for c in range(nx * ny):
        i, j = c % nx, c // nx
        ri, rj, x, y, rho, ux, uy, T, P = rows[c]
        assert (ri, rj) == (i, j) and np.isclose(x, (i + 0.5) / nx) and np.isclose(y, (j + 0.5) / ny)
        if r[c] != 0:
            st, m = oracle.moments(n, inputs.VMAX, f[c])
            ref = (m[0], m[1], m[2], m[4])
        else:
            u = hydro[c]
            p = (5.0 / 3.0 - 1.0) * (u[3] - 0.5 * (u[1] ** 2 + u[2] ** 2) / u[0])
            ref = (u[0], u[1] / u[0], u[2] / u[0], p / u[0])
        np.testing.assert_allclose([rho, ux, uy, T], ref, rtol=1e-12, atol=1e-15)
        assert np.isclose(P, rho * T, rtol=1e-14)
    reg = np.loadtxt(tmp_path / "regimes_7.txt", dtype=int)
    expect = r.reshape(ny, nx).astype(int)
    expect.ravel()[3] = -1
    assert np.array_equal(reg, expect)
    meta = json.load(open(tmp_path / "meta_7.json"))
    assert meta["step"] == 7 and meta["time"] == 0.125 and meta["nx"] == nx and meta["config"]["scenario"] == 4
    with pytest.raises(hk.io_error):
        kinetic.write_snapshot(os.path.join(tmp_path, "missing", "dir"), 8, 0.0, vg, nx, ny, 1 / nx, 1 / ny, rd, hd, fd)
