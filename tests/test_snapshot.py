"""SWPT2D snapshots (reference snapshot.cpp:11-153; engine tests
test_engine.cpp:234-289): GPU-written files are byte-identical to the files the
reference itself writes (sha256 in tests/golden/golden.json)."""
import hashlib
import json
import struct
from pathlib import Path

import numpy as np
import pytest

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())


def test_reader_rejects_foreign_files(sg, tmp_path):
    p = tmp_path / "bogus.bin"
    p.write_bytes(b"definitely not a snapshot")
    with pytest.raises(sg.SnapshotIOError):
        sg.SnapshotReader(str(p))


def test_reader_parses_handmade_stream(sg, tmp_path):
    hdr = json.dumps({"block": 8, "dt": 0.1, "dx": 0.5, "dy": 0.5, "nvars": 1, "nx": 2, "ny": 2,
                      "params": {"alpha": 1.0, "gamma": 1.4}, "problem": "heat"}).encode()
    raw = b"SWPT2D\0\0" + struct.pack("<IQ", 1, len(hdr)) + hdr
    for lev in (0, 2):
        raw += struct.pack("<Q", lev) + np.arange(4, dtype="<f8").tobytes()
    p = tmp_path / "s.bin"
    p.write_bytes(raw)
    r = sg.SnapshotReader(str(p))
    assert r.meta()["problem"] == "heat" and [f.level for f in r.frames()] == [0, 2]
    assert r.frames()[1].data.shape == (1, 2, 2)
    p.write_bytes(raw[:-3])
    with pytest.raises(sg.SnapshotIOError):
        sg.SnapshotReader(str(p))


HEAT_SWEPT = [c for c in GOLD["snapshots"]
              if c["cfg"]["problem"] == "heat" and c["cfg"].get("engine", "swept") == "swept"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["snapshots"], ids=lambda c: json.dumps(c["cfg"], sort_keys=True))
def test_snapshot_stream_is_byte_identical_to_reference(sg, tmp_path, case):
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    _check_snapshot(sg, tmp_path, case)


@pytest.mark.gpu
@pytest.mark.parametrize("case", HEAT_SWEPT, ids=lambda c: json.dumps(c["cfg"], sort_keys=True))
def test_register_tile_snapshot_stream_is_byte_identical(sg, tmp_path, monkeypatch, case):
    """The same reference streams written by the register-tile heat kernels
    (every snapshot level leaves through their stash / put_cells path)."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    monkeypatch.setenv("SG_HEAT_KERNEL", "column")
    _check_snapshot(sg, tmp_path, case)


def _check_snapshot(sg, tmp_path, case):
    path = tmp_path / "snap.bin"
    cfg = dict(case["cfg"], snapshot=str(path))
    res = sg.run(sg.SolverConfig.from_json(cfg))
    data = path.read_bytes()
    assert res.record.snapshot_frames == case["frames"]
    assert len(data) == case["bytes"]
    assert hashlib.sha256(data).hexdigest() == case["sha256"]


@pytest.mark.gpu
def test_swept_snapshot_holds_every_level(sg, oracle, tmp_path):
    """test_engine.cpp:234-252: flat+1 frames, first = initial condition,
    last = the returned field; a rewrite round-trips."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    path = tmp_path / "s.bin"
    res = sg.run(sg.SolverConfig(problem="heat", nx=64, block=8, steps=20, snapshot_path=str(path)))
    r = sg.SnapshotReader(str(path))
    assert res.record.snapshot_frames == res.record.total_levels + 1
    assert [f.level for f in r.frames()] == list(range(res.record.total_levels + 1))
    init, params = oracle.params(oracle.HEAT, 64)
    assert np.array_equal(r.frames()[0].data, init)
    assert np.array_equal(r.frames()[-1].data, res.final_field.data)
    for f in r.frames()[1:]:  # every frame is the standard solve at that level
        assert np.array_equal(f.data, oracle.standard_solve(oracle.HEAT, init, f.level, params))


def _cli(*args):
    import subprocess
    import sys
    root = Path(__file__).resolve().parents[1]
    return subprocess.run([sys.executable, "-m", "paper_2105_10332_b200", "run", *args], cwd=root,
                          capture_output=True, text=True, timeout=300)


def test_cli_rejects_bad_grid():
    """tests/CMakeLists.txt:13-15 (WILL_FAIL): nx=100 is not a multiple of 16."""
    p = _cli("--problem", "heat", "--nx", "100", "--block", "16")
    assert p.returncode == 1 and p.stderr.startswith("error:")


@pytest.mark.gpu
def test_cli_standard_and_swept_step_counts():
    """tests/CMakeLists.txt:17-26: standard prints "actual_steps": 10, swept 10 -> 7."""
    p = _cli("--problem", "heat", "--nx", "32", "--block", "8", "--steps", "10", "--engine", "standard")
    assert p.returncode == 0 and '"actual_steps": 10' in p.stdout
    p = _cli("--problem", "heat", "--nx", "32", "--block", "16", "--steps", "10")
    assert p.returncode == 0 and '"actual_steps": 7' in p.stdout
