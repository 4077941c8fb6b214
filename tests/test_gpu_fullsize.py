"""GPU parity with the reference at BASELINE's own sizes (configs[1]-[4]).

tests/golden/golden_large.json holds FNV-1a-64 hashes of the final fields the
unmodified reference (oracle/_ref/ref_run, reference run() at
proj/src/engine.cpp:493-568) produced for the bench grid (heat 8192^2, b16 and
b32), the 4128^2 block sweep (b 8/12/16/24/32), Euler 960^2 (b16, b32) and
Euler 8192^2 (b16, the 2D-partitioned multi-GPU config).  The GPU engines --
swept and standard, single partition and 2D partitions emulated on one GPU --
must reproduce them byte for byte.
"""
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_large.json").read_text())["runs"]


def _case(problem, nx, block):
    for c in GOLD:
        if (c["cfg"]["problem"], c["cfg"]["nx"], c["cfg"]["block"]) == (problem, nx, block):
            return c
    raise KeyError((problem, nx, block))


def _check(sg, case, engine, **over):
    if sg.device_count() < 1:
        pytest.fail("no CUDA device visible: the -m gpu suite must run on a B200")
    cfg = dict(case["cfg"], engine=engine)
    cfg.pop("ranks")
    if engine == "standard":
        cfg["steps"] = case["record"]["actual_steps"]
    cfg.update(over)
    res = sg.run(sg.SolverConfig(**cfg))
    assert res.final_field.level == case["record"]["final_level"]
    if engine == "swept":
        for k in ("actual_steps", "total_levels", "octahedra", "communicates", "cell_updates"):
            assert getattr(res.record, k) == case["record"][k], k
    got = sg.fnv1a64(res.final_field.data)
    assert got == case["fnv1a64"], f"{cfg}: GPU {got} != reference {case['fnv1a64']}"


@pytest.mark.parametrize("block", [16, 32])
@pytest.mark.parametrize("engine", ["swept", "standard"])
def test_bench_grid_8192(sg, engine, block):
    """configs[4] grid: the bench's own 21-step (b16) / 45-step (b32) sample."""
    _check(sg, _case("heat", 8192, block), engine)


@pytest.mark.parametrize("block", [8, 12, 16, 24, 32])
@pytest.mark.parametrize("engine", ["swept", "standard"])
def test_block_sweep_4128(sg, engine, block):
    """configs[2]: every block of the sweep, 100 requested steps."""
    _check(sg, _case("heat", 4128, block), engine)


@pytest.mark.parametrize("block", [16, 32])
@pytest.mark.parametrize("engine", ["swept", "standard"])
def test_euler_960(sg, engine, block):
    """configs[1]: Euler 960^2, b16 (100 requested steps) and b32 (40)."""
    _check(sg, _case("euler", 960, block), engine)


@pytest.mark.parametrize("px,py", [(1, 1), (2, 1), (2, 2), (4, 2)])
def test_euler_8192_partitioned(sg, px, py):
    """configs[3]: Euler 8192^2 b16 on a px x py partition grid (emulated on
    one GPU: partition-edge records go through the same push path)."""
    _check(sg, _case("euler", 8192, 16), "swept", ranks=px * py, px=px, py=py)


def test_euler_8192_standard_partitioned(sg):
    _check(sg, _case("euler", 8192, 16), "standard", ranks=4, px=2, py=2)


@pytest.mark.parametrize("cfg", [
    {"problem": "heat", "nx": 384, "block": 16, "steps": 500, "engine": "swept"},
    {"problem": "heat", "nx": 96, "block": 8, "steps": 50, "engine": "standard", "ranks": 2},
    {"problem": "euler", "nx": 96, "block": 16, "steps": 20, "engine": "swept", "ranks": 2},
])
def test_reference_side_dropin(sg, cfg):
    """The reference's own SolverConfig/RunRecord code calling the GPU through
    include/sweptgrid_gpu.hpp (oracle/_ref/shim_run) prints the same record
    and final-field hash as the unmodified CPU reference (oracle/_ref/ref_run)."""
    import subprocess
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    root = Path(__file__).resolve().parents[1]
    shim, ref = root / "oracle" / "_ref" / "shim_run", root / "oracle" / "_ref" / "ref_run"
    if not shim.exists() or not ref.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    a = json.loads(subprocess.run([str(shim), json.dumps(cfg)], capture_output=True, text=True,
                                  timeout=300).stdout.strip().splitlines()[-1])
    b = json.loads(subprocess.run([str(ref), json.dumps(cfg), "1"], capture_output=True, text=True,
                                  timeout=300).stdout.strip().splitlines()[-1])
    assert "error" not in a, a
    for k in ("engine", "problem", "nx", "block", "ranks", "steps_requested", "actual_steps", "total_levels",
              "octahedra", "communicates", "dt", "cell_updates", "final_level", "fnv1a64"):
        assert a[k] == b[k], (k, a[k], b[k])
    assert len(a["per_rank"]) == cfg.get("ranks", 1)
