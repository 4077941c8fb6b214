"""CPU oracle checks (no GPU): the C restatement (oracle/sgoracle.c) is pinned
to the reference's own outputs before anything is compared against it.

* golden.json  -- FNV-1a-64 hashes of final fields produced by the reference
                  library itself (tests/golden/gen_golden.py), including the
                  SURVEY.md §8c fingerprints;
* oracle/_ref  -- the reference built from its own sources, when present here;
* known answers of the reference's unit tests (proj/tests/test_physics.cpp,
  test_geometry.cpp).
"""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())


def _P(oracle, problem):
    return oracle.HEAT if problem == "heat" else oracle.EULER


@pytest.mark.parametrize("case", [c for c in GOLD["runs"] if c["cfg"]["nx"] <= 384],
                         ids=lambda c: f"{c['cfg']['problem']}{c['cfg']['nx']}b{c['cfg']['block']}s{c['cfg']['steps']}")
def test_restated_standard_matches_reference_hash(oracle, case):
    cfg = case["cfg"]
    P = _P(oracle, cfg["problem"])
    init, params = oracle.params(P, cfg["nx"])
    out = oracle.standard_solve(P, init, case["record"]["final_level"], params)
    assert oracle.fnv1a(out) == case["fnv1a64"]
    assert float(np.abs(out).max()) == case["max_abs"]


@pytest.mark.parametrize("case", GOLD["setup"], ids=lambda c: f"{c['cfg']['problem']}{c['cfg']['nx']}")
def test_restated_setup_matches_reference(oracle, case):
    P = _P(oracle, case["cfg"]["problem"])
    init, dt, dx, dy = oracle.setup(P, case["cfg"]["nx"])
    assert (dt, dx, dy) == (case["dt"], case["dx"], case["dy"])
    assert oracle.fnv1a(init) == case["fnv1a64"]


def test_c1_and_c2_fingerprints_present():
    """heat 384^2 b16 req 500 and Euler 960^2 b16 req 10."""
    h = {(c["cfg"]["problem"], c["cfg"]["nx"], c["cfg"]["block"], c["cfg"]["steps"]): c["fnv1a64"]
         for c in GOLD["runs"]}
    assert h[("heat", 384, 16, 500)] == "267c1269b2cb2b1a"
    assert h[("euler", 960, 16, 10)] == "aeafdd9a9c7a87b3"


@pytest.mark.parametrize("problem,nx,b,steps", [("heat", 64, 8, 20), ("heat", 96, 16, 50), ("heat", 64, 32, 40),
                                                ("euler", 32, 16, 5), ("euler", 96, 8, 20), ("euler", 48, 24, 9)])
def test_restated_swept_equals_standard(oracle, problem, nx, b, steps):
    """Swept == standard bit for bit; also pins the frame
    recipe (physical = template + origin - {0, b/2}) that replaces the shift."""
    P = _P(oracle, problem)
    n, S = (1, 1) if problem == "heat" else (2, 2)
    m, flat = oracle.schedule(steps, b, n, S)
    init, params = oracle.params(P, nx)
    final = (flat // S) * S
    a = oracle.swept_solve(P, init, b, m, final, params)
    c = oracle.standard_solve(P, init, final, params)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("entry", GOLD["schedule"], ids=lambda e: f"b{e['b']}n{e['n']}s{e['steps']}")
def test_restated_schedule_matches_reference(oracle, entry):
    if "error" in entry:
        with pytest.raises(Exception):
            oracle.schedule(entry["steps"], entry["b"], entry["n"], entry["S"])
        return
    m, flat = oracle.schedule(entry["steps"], entry["b"], entry["n"], entry["S"])
    assert m == entry["octahedra"] and flat == entry["flat_level"]


def test_schedule_golden_values(oracle):
    """test_geometry.cpp:76-99."""
    assert oracle.schedule(500, 16, 1, 1) == (70, 497)
    assert oracle.schedule(10, 16, 1, 1) == (0, 7)
    assert oracle.schedule(10, 16, 2, 2) == (6, 21)
    assert [oracle.max_levels(b, 1) for b in (8, 12, 16, 24, 32)] == [3, 5, 7, 11, 15]
    assert [oracle.max_levels(b, 2) for b in (8, 12, 16, 24, 32)] == [1, 2, 3, 5, 7]
    assert oracle.max_levels(10, 2) < 0 and oracle.max_levels(9, 1) < 0 and oracle.max_levels(4, 2) < 0


def test_physics_known_answers(oracle):
    """test_physics.cpp:86-119."""
    from oracle_bind import OracleError
    assert oracle.pressure([1.0, 0.0, 0.0, 1.0]) == pytest.approx(0.4)
    for bad in ([-1.0, 0, 0, 1.0], [0.0, 0, 0, 1.0], [1.0, 10.0, 0, 1.0]):
        with pytest.raises(OracleError):
            oracle.pressure(bad)
    q = np.array([1.2, 0.4, -0.2, 3.0])
    p = oracle.pressure(q)
    fx = np.array([q[1], q[1] * (q[1] / q[0]) + p, q[2] * (q[1] / q[0]), (q[3] + p) * (q[1] / q[0])])
    assert np.array_equal(oracle.interface_flux(q, q, 0), fx)
    a, b, c, d = [1.0, 0.1, 0.0, 2.0], [1.1, 0.1, 0.0, 2.2], [1.05, 0.1, 0.0, 2.1], [1.2, 0.1, 0.0, 2.4]
    ql, qr = oracle.minmod(np.array([a, b, c, d]), [1.0, 1.2, 1.1, 1.3])
    assert list(ql) == b and list(qr) == c
    ql, qr = oracle.minmod(np.array([a, b, c, d]), [1.0, 1.1, 1.2, 1.3])
    for v in range(4):
        assert ql[v] == b[v] + 0.5 * (c[v] - b[v])


def test_restated_matches_reference_library(oracle, reference):
    """Direct comparison with the reference library built from its sources."""
    for cfg in ({"problem": "heat", "nx": 48, "block": 8, "steps": 17},
                {"problem": "euler", "nx": 48, "block": 8, "steps": 7},
                {"problem": "euler", "nx": 64, "block": 16, "steps": 11, "engine": "standard"}):
        field, rec = reference.run(cfg)
        P = _P(oracle, cfg["problem"])
        init, params = oracle.params(P, cfg["nx"])
        assert np.array_equal(oracle.standard_solve(P, init, rec["final_level"], params), field)
        rinit, dt, dx, dy = reference.setup(cfg)
        assert np.array_equal(rinit, init)


def test_restated_substep_matches_reference_on_fuzzed_fields(oracle, reference):
    """run_substep_serial on the xorshift-perturbed vortex of test_physics.cpp:24-41."""
    nx = 48
    init, _ = oracle.params(oracle.EULER, nx)
    s = 0x9E3779B97F4A7C15
    f = init.reshape(-1).copy()
    for i in range(f.size):
        s ^= (s << 13) & 0xFFFFFFFFFFFFFFFF
        s ^= s >> 7
        s ^= (s << 17) & 0xFFFFFFFFFFFFFFFF
        f[i] *= 1.0 + 0.01 * ((s % 10000) / 10000.0 - 0.5)
    f = f.reshape(init.shape)
    rects = [[4, 20, 2, 30], [20, 44, 0, 48]]
    ep = [1.4, 0.05, 0.05, 1e-4]
    for stage in (0, 1):
        a, b = np.zeros_like(f), np.zeros_like(f)
        oracle.substep(oracle.EULER, stage, f, init, a, rects, np.array(ep))
        reference.substep(1, stage, f, init, b, rects, [1.0, 0.05, 0.05, 1e-4], ep + [0.4])
        assert np.array_equal(a, b)
