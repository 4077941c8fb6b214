"""Host-side swept plan + schedule arithmetic of the product library (no GPU).

Mirrors proj/tests/test_geometry.cpp: the k table, rounding golden values,
and the coverage replay (compile_swept_plan replays the schedule on a periodic
tile and fails on any cell computed twice, read before written, or read from
a concurrent instance -- the reference CoverageOracle's checks,
proj/tests/oracle.hpp:58-87).  Also pins the per-block dependency counts to
SURVEY.md §8d.
"""
import json
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())


def test_max_levels_table(sg):
    assert [sg.max_levels(b, 1) for b in (8, 12, 16, 24, 32)] == [3, 5, 7, 11, 15]
    assert [sg.max_levels(b, 2) for b in (8, 12, 16, 24, 32)] == [1, 2, 3, 5, 7]
    for b, n in ((10, 2), (9, 1), (4, 2)):
        with pytest.raises(sg.InvalidArgument):
            sg.max_levels(b, n)


def test_schedule_rounding(sg):
    """test_geometry.cpp:76-99."""
    s = sg.build_schedule(500, 16, 1, 1)
    assert (s["flat_level"], s["octahedra"], s["communicates"], s["completed_steps"]) == (497, 70, 71, 497)
    s = sg.build_schedule(10, 16, 1, 1)
    assert (s["flat_level"], s["octahedra"], s["completed_steps"]) == (7, 0, 7)
    s = sg.build_schedule(10, 16, 2, 2)
    assert (s["k"], s["octahedra"], s["flat_level"], s["completed_steps"]) == (3, 6, 21, 10)


@pytest.mark.parametrize("entry", [e for e in GOLD["schedule"] if "error" not in e],
                         ids=lambda e: f"b{e['b']}n{e['n']}s{e['steps']}")
def test_schedule_matches_reference(sg, entry):
    s = sg.build_schedule(entry["steps"], entry["b"], entry["n"], entry["S"])
    assert s["octahedra"] == entry["octahedra"] and s["flat_level"] == entry["flat_level"]


@pytest.mark.parametrize("problem", ["heat", "euler"])
@pytest.mark.parametrize("b", [8, 12, 16, 24, 32])
@pytest.mark.parametrize("steps", [1, 3, 10, 40, 200, 10000])
def test_plan_compiles_and_proves_coverage(sg, problem, b, steps):
    try:
        sg.build_schedule(steps, b, 1 if problem == "heat" else 2, 1 if problem == "heat" else 2)
    except sg.InvalidArgument:
        return  # nearest achievable step count is 0
    d = sg.plan_info(problem, b, steps)
    S = 1 if problem == "heat" else 2
    assert d["launches"] == 3 + 3 * d["m"] + 1
    assert d["ghost"] == 1           # instances only ever read their 8 neighbours
    assert 1 <= d["slots"] <= 7      # records live at most two cycles
    assert d["flat"] == d["k"] * (d["m"] + 1)
    # a long run collapses onto a fixed number of launch classes
    assert d["classes"] <= 14
    if d["m"] > 9:
        assert d["replay_cycles"] in (8, 9)
    del S


def test_heat_b16_dependency_counts_match_survey(sg):
    """SURVEY.md §8d, heat b16 per block: Octahedron 1120 updates / 476
    imported / 392 exported; YBridge 336 / 252 / 196."""
    d = sg.plan_info("heat", 16, 500)
    assert (d["oct_updates"], d["oct_imports"], d["oct_exports"]) == (1120, 476, 392)
    assert (d["yb_updates"], d["yb_imports"], d["yb_exports"]) == (336, 252, 196)
    # minimum inter-phase traffic per update over a steady cycle: 7.875 B
    bytes_per_update = 8 * (476 + 392 + 2 * (252 + 196)) / (1120 + 2 * 336)
    assert bytes_per_update == pytest.approx(7.875)


@pytest.mark.parametrize("b,expect", [(8, 15.5), (12, 10.44), (16, 7.88), (24, 5.28), (32, 3.97)])
def test_swept_traffic_per_update_table(sg, b, expect):
    """SURVEY.md §8d table of minimum swept bytes/update (heat)."""
    d = sg.plan_info("heat", b, 500)
    byt = 8 * (d["oct_imports"] + d["oct_exports"] + 2 * (d["yb_imports"] + d["yb_exports"]))
    upd = d["oct_updates"] + 2 * d["yb_updates"]
    assert byt / upd == pytest.approx(expect, abs=0.01)


@pytest.mark.parametrize("b", [8, 12, 16, 24, 32])
def test_column_layout_covers_the_replayed_reads_exactly(sg, b):
    """The closed-form import/export sets of the register-tile kernels
    (colgeom.hpp) cover every cross-instance read of the schedule replay and,
    in the steady state, nothing more (overexport = 0)."""
    d = sg.plan_info("heat", b, 40 * b)
    assert "heat_kernel=column" in d["text"] and "overexport=0" in d["text"]


def test_generic_kernels_for_euler(sg):
    assert "heat_kernel=generic" in sg.plan_info("euler", 16, 200)["text"]
