"""Alpha sweep: grid/format helpers on the CPU; on the GPU the
batched sweep (one filter grid per image) against one d_landweber run per
alpha, divergent cells flagged like the reference's run_cell, and the
experiment files in the reference's formats (experiment.hpp:126-164, 271-307)."""
import math
import os

import numpy as np
import pytest

from paper_1211_0393_b200 import experiment as ex


def test_alpha_grid_and_formats():
    g = ex.alpha_grid(1e-6, 1e-1, 6)
    la, lb = math.log(1e-6), math.log(1e-1)
    assert g == [math.exp(la + (lb - la) * i / 5) for i in range(6)]
    assert ex.alpha_grid(0.5, 0.5, 1) == [0.5]
    with pytest.raises(ValueError):
        ex.alpha_grid(0.0, 1.0, 3)
    with pytest.raises(ValueError):
        ex.alpha_grid(1e-3, 1e-2, 0)
    assert ex.format_alpha(g[1]) == "1e-05" and ex.format_double(0.1) == "0.10000000000000001"
    run = ex.RestorationRun(rre_history=[0.5, 0.25], residual_history=[2.0, 1.0])
    assert ex.history_csv(run) == "iter,rre,residual\n1,0.5,2\n2,0.25,1\n"
    cell = ex.CellResult("d-landweber", 0.01, run, 0.0)
    assert cell.stem() == "antireflective_d-landweber_alpha0.01"
    assert ex.CellResult("landweber", 0.0, run, 0.0).stem() == "antireflective_landweber"


@pytest.mark.gpu
def test_batched_sweep_matches_single_runs(dbx):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C2"]  # motion mask: small alphas diverge with tau = 1
    n, iters = 64, 12
    f, g, taps = cf.make_problem(c, n=n)
    alphas = [1e-4, 0.3, 1.0, 3.0]
    cells = ex.sweep_d_landweber(taps, g, f, alphas, iters)
    op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.AntiReflective, n, n)
    for a, cell in zip(alphas, cells):
        d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, a), n, n)
        cfg = dbx.SolverConfig(max_iters=iters, track_rre_against=f)
        try:
            ref = dbx.d_landweber(op, d, g, cfg)
        except dbx.SolverDivergence:
            assert cell.diverged, a
            continue
        assert not cell.diverged, a
        assert cell.run.iterations_executed == ref.iterations_executed
        assert cell.run.best_iteration == ref.best_iteration
        np.testing.assert_allclose(cell.run.residual_history, ref.residual_history, rtol=1e-12, atol=0)
        np.testing.assert_allclose(cell.run.rre_history, ref.rre_history, rtol=1e-12, atol=0)
        assert np.abs(cell.run.restored - ref.restored).max() <= 1e-12 * np.abs(ref.restored).max()
    assert any(c.diverged for c in cells) and not all(c.diverged for c in cells)


@pytest.mark.gpu
def test_run_experiment_writes_reference_files(dbx, tmp_path):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C1"]
    f, g, taps = cf.make_problem(c, n=48)
    res = ex.run_experiment(taps, g, f, ex.alpha_grid(1e-3, 1e-1, 3), max_iters=10, out_dir=str(tmp_path))
    names = sorted(os.listdir(tmp_path))
    assert "summary.csv" in names and "metadata.txt" in names and "antireflective_landweber.csv" in names
    assert sum(n.startswith("antireflective_d-landweber_alpha") for n in names) == 3
    rows = open(tmp_path / "summary.csv").read().splitlines()
    assert rows[0] == "bc,method,alpha,best_rre,best_iter,seconds" and len(rows) == 3
    best = min((cc for cc in res.cells if cc.method == "d-landweber"),
               key=lambda cc: cc.run.rre_history[cc.run.best_iteration - 1])
    assert res.summary[1].alpha == best.alpha
    hist = open(tmp_path / (best.stem() + ".csv")).read().splitlines()
    assert hist[0] == "iter,rre,residual" and len(hist) == 11


@pytest.mark.gpu
@pytest.mark.parametrize("bc", ["AntiReflective", "Reflective"])
def test_sweep_cells_match_oracle(dbx, oracle, bc):
    """Every alpha cell of the batched GPU sweep against the CPU oracle's own
    D-Landweber run for that alpha (experiment.hpp:209-232 run_cell): identical
    divergence verdict, iteration count and best iteration; histories and the
    restored image within the 1e-10 parity bar."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C1"]
    n, iters = 64, 15
    f, g, taps = cf.make_problem(c, n=n)
    alphas = ex.alpha_grid(1e-3, 0.3, 4)
    bcv = int(getattr(dbx.BoundaryCondition, bc))
    cells = ex.sweep_d_landweber(taps, g, f, alphas, iters, bc=bcv)
    for a, cell in zip(alphas, cells):
        assert cell.bc == bcv and cell.stem().startswith(ex.bc_name(bcv) + "_d-landweber_alpha")
        try:
            ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, a, n, n, bc=bcv), f_true=f,
                                   max_iters=iters, bc=bcv)
        except oracle.OracleDivergence:
            assert cell.diverged, a
            continue
        assert not cell.diverged, a
        assert cell.run.iterations_executed == ref["iterations_executed"]
        assert cell.run.best_iteration == ref["best_iteration"]
        np.testing.assert_allclose(cell.run.rre_history, ref["rre_history"], rtol=1e-10, atol=0)
        np.testing.assert_allclose(cell.run.residual_history, ref["residual_history"], rtol=1e-10, atol=0)
        r = ref["restored"]
        assert np.linalg.norm(cell.run.restored - r) <= 1e-10 * np.linalg.norm(r)


@pytest.mark.gpu
def test_run_experiment_both_bcs_writes_pgms(dbx, tmp_path):
    """Per-BC cell blocks and the restored PGMs of experiment.hpp:242-244, 266-268."""
    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200 import io as dio
    c = cf.CONFIGS["C1"]
    f, g, taps = cf.make_problem(c, n=48)
    f, g = 200.0 * f, 200.0 * g  # PGM range: the writer rounds and clamps to [0, 255]
    bcs = (dbx.BoundaryCondition.AntiReflective, dbx.BoundaryCondition.Reflective)
    res = ex.run_experiment(taps, g, f, ex.alpha_grid(1e-3, 1e-1, 3), max_iters=8, out_dir=str(tmp_path), bcs=bcs)
    names = set(os.listdir(tmp_path))
    for b in ("antireflective", "reflective"):
        assert {b + "_landweber.csv", b + "_landweber.pgm", b + "_d-landweber.pgm"} <= names
        assert sum(nm.startswith(b + "_d-landweber_alpha") for nm in names) == 3
    rows = open(tmp_path / "summary.csv").read().splitlines()
    assert [r.split(",")[0] for r in rows[1:]] == ["antireflective"] * 2 + ["reflective"] * 2
    assert "bcs=antireflective,reflective" in open(tmp_path / "metadata.txt").read()
    for b, bcv in zip(("antireflective", "reflective"), bcs):
        plain = next(cc for cc in res.cells if cc.bc == bcv and cc.method == "landweber")
        px, mx = dio.read_pgm(str(tmp_path / (b + "_landweber.pgm")))
        assert mx == 255 and px.shape == (48, 48)
        assert np.array_equal(px, np.clip(np.round(plain.run.restored), 0, 255))
        row = next(r for r in res.summary if r.bc == bcv and r.method == "d-landweber")
        best = next(cc for cc in res.cells if cc.bc == bcv and cc.method == "d-landweber" and cc.alpha == row.alpha)
        px, _ = dio.read_pgm(str(tmp_path / (b + "_d-landweber.pgm")))
        assert np.array_equal(px, np.clip(np.round(best.run.restored), 0, 255))


def test_bc_names_and_refusal():
    from paper_1211_0393_b200 import BoundaryCondition as BC
    assert ex.bc_name(BC.AntiReflective) == "antireflective" and ex.bc_name(BC.Reflective) == "reflective"
    with pytest.raises(ValueError):
        ex.bc_name(BC.Zero)
    run = ex.RestorationRun(rre_history=[0.5], residual_history=[1.0])
    assert ex.CellResult("d-landweber", 0.1, run, 0.0, bc=BC.Reflective).stem() == "reflective_d-landweber_alpha0.1"
