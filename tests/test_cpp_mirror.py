"""The C++ mirror (include/hykin_b200.hpp) of every §8(b) reference signature,
driven by a reference-style C++ caller (tests/cpp/mirror_demo.cpp) on the GPU:
collision and residual with the reference's throw semantics, the moments
family, both stage solves, transport (field and single cell), both PR(2,2,2)
steps on a DistributionField, the indicators and Algorithm 1 — each compared
with the reference-generated golden fixtures or the oracle."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2505_03360_b200", "lib")
GOLD = os.path.join(ROOT, "tests", "golden")


def build(tmp_path):
    exe = str(tmp_path / "mirror_demo")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "mirror_demo.cpp"), "-L", LIBDIR, "-lhykin_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_mirror_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.gpu
def test_mirror_against_golden_and_oracle(tmp_path, oracle):
    exe = build(tmp_path)
    d = tmp_path
    w = lambda name, a: np.ascontiguousarray(a, dtype=np.float64).tofile(str(d / name))  # noqa: E731
    r = lambda name: np.fromfile(str(d / name), dtype=np.float64)  # noqa: E731
    gc = np.load(os.path.join(GOLD, "collision_n16_cfg1.npz"))
    ge = np.load(os.path.join(GOLD, "esbgk_cfg3_n16.npz"))
    gt = np.load(os.path.join(GOLD, "transport_n8.npz"))
    vmax = float(gc["vmax"])
    w("params.bin", np.array([vmax, float(gc["r_phys"]), int(gc["a1"]), int(gc["a2"])] + [0] * 12))
    w("coll_f.bin", gc["f"])
    w("mom_f.bin", ge["f"])
    w("mom_params.bin", [float(ge["a"]), float(ge["eps"]), float(ge["beta"]), float(ge["nu_coeff"])])
    nx, ny, n = int(gt["nx"]), int(gt["ny"]), int(gt["n"])
    w("tr_params.bin", [nx, ny, float(gt["dx"]), float(gt["dy"]), float(gt["dt"]), n])
    w("tr_f.bin", gt["f"])
    w("tr_eps.bin", gt["eps"])
    from paper_2505_03360_b200 import inputs
    fpen, _ = inputs.config3_cells(4, 3, 16)
    epen = np.array([1e-2, 1e-1, 1.0, 3e-2] * 3)
    w("pen_f.bin", fpen)
    w("pen_eps.bin", epen)
    rng = np.random.default_rng(5)
    prim = np.stack([[1.0 + 0.1 * rng.uniform(), 0.1 * rng.uniform(-1, 1), 0.1 * rng.uniform(-1, 1),
                      1.0 + 0.1 * rng.uniform()] for _ in range(5)])
    w("ind_prim.bin", np.concatenate([prim.ravel(), [0.02, 0.03, 1e-2]]))
    tt = json.load(open(os.path.join(GOLD, "regime_truth_table.json")))
    rows = []
    for row in tt["rows"]:
        lam = row["lam"]
        rows.append([row["r"], 0 if lam is None else 1, *(lam or [0, 0, 0]),
                     math.nan if row["lambda_b"] is None else row["lambda_b"],
                     math.nan if row["l1"] is None else row["l1"], 0])
    w("regime_rows.bin", rows)

    out = subprocess.run([exe, str(d)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr

    nb16 = 16 ** 3
    # collision / residual: values (written before the throw) and the throw itself
    q, res, threw = r("out_coll_q.bin").reshape(4, nb16), r("out_coll_res.bin").reshape(4, nb16), r("out_coll_threw.bin")
    for c in range(4):
        assert rel(q[c], gc["q"][c]) < 1e-10, c
        assert rel(res[c], gc["residual"][c]) < 1e-10, c
        assert (int(threw[c]) & 1) == (gc["status"][c] == 4), c          # spectral_collision throws iff the reference did
        assert bool(int(threw[c]) & 2) == (gc["status"][c] == 4), c      # penalized_residual propagates it
    # moments family vs golden / oracle
    mom = r("out_mom.bin").reshape(4, 5)
    np.testing.assert_allclose(mom, ge["moments"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r("out_real.bin").reshape(4, 13), ge["realizability"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(r("out_l1.bin"), ge["l1"], rtol=1e-12, atol=1e-15)
    sig, maxw = r("out_sigma.bin").reshape(4, 9), r("out_maxw.bin").reshape(4, nb16)
    gauss, gfb = r("out_gauss.bin").reshape(4, nb16), r("out_gauss_fb.bin")
    matched, removed = r("out_matched.bin").reshape(4, nb16), r("out_removed.bin").reshape(4, nb16)
    for c in range(4):
        f = ge["f"][c]
        np.testing.assert_allclose(sig[c], oracle.second_moment(16, vmax, f).ravel(), rtol=1e-12, atol=1e-15)
        assert rel(maxw[c], oracle.maxwellian(16, vmax, tuple(mom[c]))[1]) < 1e-13
        th = oracle.stress_tensor(16, vmax, f, mom[c])
        st, g_ref, fb_ref = oracle.anisotropic_gaussian(16, vmax, tuple(mom[c]), th, -0.5)
        assert rel(gauss[c], g_ref) < 1e-12 and int(gfb[c]) == fb_ref, c
        E = 0.5 * mom[c, 0] * (mom[c, 1:4] ** 2).sum() + 1.5 * mom[c, 0] * mom[c, 4]
        st, m_ref = oracle.match_moments(16, vmax, g_ref, mom[c, 0], mom[c, 0] * mom[c, 1:4], E)
        assert rel(matched[c], m_ref) < 1e-12, c
        st, rm_ref = oracle.remove_invariant_moments(16, vmax, f - m_ref, m_ref, mom[c, 1:4])
        assert np.abs(removed[c] - rm_ref).max() <= 1e-12 * np.abs(f - m_ref).max(), c
    es = r("out_esbgk.bin").reshape(4, nb16)
    for c in range(4):
        assert rel(es[c], ge["esbgk"][c]) < 1e-11, c
    assert np.array_equal(r("out_esbgk_fb.bin").astype(int), ge["fallback"])
    pen = r("out_pen.bin").reshape(4, nb16)
    for c in range(4):
        ref, st = oracle.penalized_stage_solve(16, vmax, ge["f"][c], float(ge["a"]), float(ge["eps"]))
        assert rel(pen[c], ref) < 1e-11, c
    # transport and the two PR(2,2,2) steps on a DistributionField
    assert rel(r("out_tr_rhs.bin"), gt["rhs"]) < 1e-13
    assert rel(r("out_tr_cell.bin"), gt["rhs"][2 * nx + 1]) < 1e-13
    assert rel(r("out_esbgk_step.bin"), gt["esbgk_step"]) < 1e-11
    ko = oracle.kernel(16, vmax, 2, 4, float(gc["r_phys"]))
    ref, st = oracle.penalized_imex_step(ko, fpen, 4, 3, 0.25, 1.0 / 3.0, 1e-3, epen)
    got = r("out_pen_step.bin").reshape(-1, nb16)
    for c in range(12):
        assert rel(got[c], ref[c]) < 1e-10, c
    assert r("out_tableau_rejected.bin")[0] == 1.0
    # indicators and Algorithm 1
    _, lam, lb = oracle.indicators(prim, 0.02, 0.03, 1e-2)
    ind = r("out_ind.bin")
    np.testing.assert_allclose(ind[:3], lam, rtol=1e-13)
    assert math.isclose(ind[3], lb, rel_tol=1e-12)
    reg = r("out_regime.bin").astype(int)
    for k, row in enumerate(tt["rows"]):
        expect = -1 if row["status"] != 0 else row["out"]
        assert reg[k] == expect, (k, row)
