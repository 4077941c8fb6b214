"""bench.py keeps the driver's JSON-line contract (task statement + SURVEY.md
§8d): one line on rank 0 with the metric, whole-job value, e2e through the
C-ABI with host copies, kernel launch count, roofline of the dominant kernel,
the §8d whole-solve roofline, CPU baseline and clocks.  Tiny workload."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(900)
def test_bench_json_line_contract(sg):
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    p = subprocess.run([sys.executable, "bench.py", "--per-gpu", "1024", "--req-steps", "100", "--steps", "2",
                        "--warmup", "3", "--no-extra", "--ref-sample-steps", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=850)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "solve_roofline",
              "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 1024 * 1024 * 8
    assert 0 < d["roofline"]["frac"] < 1 and d["roofline"]["bound"] == "hbm"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("heat2d-swept-weak-1024sq")
