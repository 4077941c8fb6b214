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


def _snap_worker(rank, world, port, cfgd, path, q):
    import os
    import sys
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2105_10332_b200 as sg
        res = sg.run_distributed(sg.SolverConfig(**dict(cfgd, snapshot_path=path)))
        if rank == 0:
            q.put(("ok", res.record.snapshot_frames))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e)))


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", [c for c in GOLD["snapshots"] if c["cfg"]["nx"] % 2 == 0],
                         ids=lambda c: json.dumps(c["cfg"], sort_keys=True))
def test_distributed_snapshot_is_byte_identical(sg, tmp_path, case):
    """FrameCollector (snapshot.cpp:122-153) for one process per GPU: rank 0
    assembles every partition's strip of each snapshot level (peers' frames
    through their IPC-mapped buffers) -- the stream equals the reference's."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    import socket
    import torch.multiprocessing as mp
    c = dict(case["cfg"])
    b = c.get("block", 8)
    if (c["nx"] // b) % 2:
        pytest.skip("2x1 partition needs an even number of block columns")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    every = c.pop("snapshot_every", 1)
    c.pop("ranks", None)
    cfgd = dict(problem=c["problem"], nx=c["nx"], block=b, steps=c["steps"], engine=c.get("engine", "swept"),
                ranks=2, px=2, py=1, snapshot_every=every)
    path = str(tmp_path / "d.bin")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_snap_worker, args=(r, 2, port, cfgd, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, frames = q.get(timeout=500)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", frames
    data = Path(path).read_bytes()
    assert frames == case["frames"]
    assert hashlib.sha256(data).hexdigest() == case["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["snapshots"], ids=lambda c: json.dumps(c["cfg"], sort_keys=True))
def test_partitioned_snapshot_is_byte_identical(sg, tmp_path, monkeypatch, case):
    """One process, 2x2 partitions on (aliased) devices: every frame is drained
    asynchronously (copy streams, pinned host frames) and still byte-identical."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    c = dict(case["cfg"])
    b = c.get("block", 8)
    if (c["nx"] // b) % 2:
        pytest.skip("2x2 partition needs an even number of blocks per axis")
    monkeypatch.setenv("SG_DEVICE_ALIAS", "1")
    path = tmp_path / "p.bin"
    c.pop("ranks", None)
    res = sg.run(sg.SolverConfig.from_json(dict(c, snapshot=str(path), ranks=4, px=2, py=2, devices=2)))
    data = path.read_bytes()
    assert res.record.snapshot_frames == case["frames"]
    assert hashlib.sha256(data).hexdigest() == case["sha256"]
