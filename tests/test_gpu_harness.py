"""The reference's acceptance checks that exercise the whole solver
(proj/tests/acceptance.cpp:170-237), on the GPU engine."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpu(sg):
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")


def test_heat_converges_at_second_order(sg):
    """Acceptance check 5 (acceptance.cpp:170-177) / run_verify heat."""
    _gpu(sg)
    from paper_2105_10332_b200 import harness
    rep = harness.run_verify("heat", [32, 64, 128])
    assert rep.observed_order >= 1.9 and rep.passed


def test_euler_vortex_error_shrinks_and_conserves(sg):
    """Acceptance check 6 (acceptance.cpp:179-205): monotone error, drift <= 1e-11."""
    _gpu(sg)
    from paper_2105_10332_b200 import harness
    rep = harness.run_verify("euler", [64, 128, 256])
    assert rep.passed
    cfg = sg.SolverConfig(problem="euler", nx=64, block=8, steps=100, engine="standard")
    res = sg.run(cfg)
    init = sg.Solver(cfg)
    full = np.empty((4, 64, 64))
    init.initial(full)
    init.close()
    drift = max(abs(res.final_field.data[v].sum() - full[v].sum()) / np.abs(full[v]).sum() for v in range(4))
    assert drift <= 1e-11


def test_step_rounding(sg):
    """Acceptance check 8 (acceptance.cpp:228-237): 500 -> 497, 10 -> 7."""
    _gpu(sg)
    assert sg.run(sg.SolverConfig(problem="heat", nx=96, block=16, steps=500)).record.actual_steps == 497
    assert sg.run(sg.SolverConfig(problem="heat", nx=32, block=16, steps=10)).record.actual_steps == 7


def test_sweep_csv_schema(sg, tmp_path):
    """run_sweep CSV (bench.cpp:60-63, 138-206): header, one row per cell,
    standard run at the swept actual steps, resumable."""
    _gpu(sg)
    from paper_2105_10332_b200 import harness
    spec = harness.SweepSpec(problems=["heat"], array_sizes=[48], block_sizes=[8, 16], shares=[0.0, 1.0], steps=20)
    path = tmp_path / "sweep.csv"
    harness.run_sweep(spec, str(path))
    rows = harness.load_bench_csv(str(path))
    assert path.read_text().splitlines()[0] == harness.BENCH_CSV_HEADER
    assert len(rows) == 4 and all(r["error"] == "" and float(r["speedup"]) > 0 for r in rows)
    harness.run_sweep(spec, str(path))  # resume: nothing new
    assert len(harness.load_bench_csv(str(path))) == 4


def test_weak_scaling_csv(sg, tmp_path):
    """run_weak_scaling CSV (bench.cpp:208-244): the reference's rank ladder
    (1, 192) .. (4, 384), block 16, share 0.9, standard then swept per rung;
    points per rank, per-step seconds and bytes per exchange event derived
    from the record exactly as the reference does."""
    _gpu(sg)
    import csv
    from paper_2105_10332_b200 import harness
    spec = harness.SweepSpec(problems=["heat", "euler"], array_sizes=[], block_sizes=[16], shares=[0.9], steps=20)
    path = tmp_path / "weak.csv"
    harness.run_weak_scaling(spec, str(path))
    rows = list(csv.DictReader(open(path)))
    assert list(rows[0]) == ["problem", "ranks", "nx", "points_per_rank", "engine", "actual_steps", "seconds",
                             "seconds_per_step", "messages", "bytes", "bytes_per_event"]
    assert len(rows) == 2 * 4 * 2
    for r in rows:
        ranks, nx = int(r["ranks"]), int(r["nx"])
        assert (ranks, nx) in ((1, 192), (2, 288), (3, 336), (4, 384))
        assert int(r["points_per_rank"]) == nx * nx // ranks
        assert float(r["seconds"]) > 0
        assert float(r["seconds_per_step"]) == pytest.approx(float(r["seconds"]) / int(r["actual_steps"]))
        if ranks > 1:
            assert int(r["messages"]) > 0 and int(r["bytes"]) > 0 and float(r["bytes_per_event"]) > 0
        else:
            assert int(r["messages"]) == 0
        # schedule arithmetic of the reference: swept 20 -> 21 levels (heat, k=7) / 20 steps (euler, k=3)
        if r["engine"] == "standard":
            assert int(r["actual_steps"]) == 20
    sw = {(r["problem"], r["ranks"]): int(r["actual_steps"]) for r in rows if r["engine"] == "swept"}
    assert set(sw.values()) <= {sg.build_schedule(20, 16, 1, 1)["completed_steps"],
                                sg.build_schedule(20, 16, 2, 2)["completed_steps"]}
