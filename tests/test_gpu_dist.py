"""One process per partition (the torchrun layout) exercised on ONE GPU: two
processes each own one partition of a 2x1 / 1x2 grid, exchange CUDA IPC
handles through torch.distributed (gloo), push partition-edge cells into each
other's buffers from inside the kernels and order launches with the
device-side epoch barrier.  On a multi-GPU box the same code path uses
NVLink P2P.  Result must equal the CPU oracle bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfgd, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2105_10332_b200 as sg
        res = sg.run_distributed(sg.SolverConfig(**cfgd))
        if rank == 0:
            q.put(("ok", res.final_field.data, res.final_field.level, res.record.messages))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e), None, None))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("engine,kernel", [("swept", "generic"), ("swept", "column"), ("standard", "generic")])
@pytest.mark.parametrize("problem,px,py", [("heat", 2, 1), ("heat", 1, 2), ("euler", 2, 1)])
def test_two_process_partitions_bitwise(sg, oracle, monkeypatch, engine, kernel, problem, px, py):
    """kernel: the swept heat phase kernels (SG_HEAT_KERNEL, inherited by the
    spawned ranks); "column" = the register-tile kernels, whose partition-edge
    instances push their records into the other rank's ghost ring."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    if kernel == "column" and problem != "heat":
        pytest.skip("register-tile kernels are heat-only")
    monkeypatch.setenv("SG_HEAT_KERNEL", kernel)
    import torch.multiprocessing as mp
    nx = 64
    cfgd = dict(problem=problem, nx=nx, block=16 if problem == "heat" else 8, steps=12, engine=engine,
                ranks=px * py, px=px, py=py)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfgd, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, data, level, msgs = q.get(timeout=500)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", data
    P = oracle.HEAT if problem == "heat" else oracle.EULER
    init, params = oracle.params(P, nx)
    want = oracle.standard_solve(P, init, level, params)
    assert np.array_equal(data, want)
    assert msgs > 0


@pytest.mark.timeout(600)
@pytest.mark.parametrize("engine,kernel,problem", [("swept", "column", "heat"), ("swept", "generic", "heat"),
                                                   ("standard", "generic", "heat"), ("swept", "generic", "euler")])
def test_four_process_2x2_partitions_bitwise(sg, oracle, monkeypatch, engine, kernel, problem):
    """2 x 2 partitions, one process each: partition-corner instances push
    their records to the diagonal neighbour's ghost ring too (three peers)."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    monkeypatch.setenv("SG_HEAT_KERNEL", kernel)
    import torch.multiprocessing as mp
    nx = 64
    cfgd = dict(problem=problem, nx=nx, block=16 if problem == "heat" else 8, steps=12, engine=engine,
                ranks=4, px=2, py=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, cfgd, q)) for r in range(4)]
    for p in procs:
        p.start()
    status, data, level, msgs = q.get(timeout=500)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", data
    P = oracle.HEAT if problem == "heat" else oracle.EULER
    init, params = oracle.params(P, nx)
    want = oracle.standard_solve(P, init, level, params)
    assert np.array_equal(data, want)
    assert msgs > 0


@pytest.mark.parametrize("engine", ["swept", "standard"])
@pytest.mark.parametrize("problem,px,py,devices", [("heat", 2, 1, 2), ("heat", 2, 2, 4), ("euler", 2, 2, 2)])
def test_one_process_multi_device_path(sg, oracle, monkeypatch, engine, problem, px, py, devices):
    """One process driving several devices (partitions spread over `devices`
    CUDA devices: per-device streams, cross-device event waits before every
    dependent launch, run_ranks of engine.cpp:427-457).  SG_DEVICE_ALIAS=1
    maps every logical device onto the one GPU of the test box so the path
    runs here; on a multi-GPU box it is the same code with distinct devices."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    monkeypatch.setenv("SG_DEVICE_ALIAS", "1")
    nx = 128 if problem == "heat" else 64
    block = 16 if problem == "heat" else 8
    res = sg.run(sg.SolverConfig(problem=problem, nx=nx, block=block, steps=12, engine=engine, ranks=px * py,
                                 px=px, py=py, devices=devices))
    P = oracle.HEAT if problem == "heat" else oracle.EULER
    init, params = oracle.params(P, nx)
    want = oracle.standard_solve(P, init, res.final_field.level, params)
    assert np.array_equal(res.final_field.data, want)


def _bench(args, env_extra, nproc=None):
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, **env_extra)
    if nproc:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py"] + args
    else:
        cmd = [sys.executable, "bench.py"] + args
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=800, env=env)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(900)
@pytest.mark.parametrize("n", [2, 4])
def test_bench_torchrun_n_ranks(sg, n):
    """bench.py under torchrun with N ranks (the driver's N>1 launch), all
    ranks on the one GPU of the test box (SG_BENCH_SAME_DEVICE=1, gloo): the
    JSON line is produced by rank 0 and the assembled global field equals a
    1-process solve of the same global grid bit for bit."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    per = 1024
    args = ["--gpus", str(n), "--per-gpu", str(per), "--req-steps", "100", "--steps", "2", "--warmup", "3",
            "--no-extra", "--no-cpu", "--hash"]
    d = _bench(args, {"SG_BENCH_SAME_DEVICE": "1", "SG_BENCH_BACKEND": "gloo"}, nproc=n)
    px, py = {2: (2, 1), 4: (2, 2)}[n]
    assert d["n_gpus"] == n and d["config"]["partition"] == f"{px}x{py}"
    assert d["config"]["nx"] == per * px and d["config"]["ny"] == per * py
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    with sg.Solver(sg.SolverConfig(problem="heat", nx=per * px, ny=per * py, block=16, steps=100)) as s:
        s.reset()
        s.solve()
        want = sg.fnv1a64(s.fetch().final_field.data)
    assert d["final_fnv1a64"] == want


def _worker_repeat(rank, world, port, cfgd, q):
    """Three solves on one DistSolver: the first captures the rank's launches
    (phase kernels + epoch barriers) in a CUDA graph, the others replay it."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2105_10332_b200 as sg
        s = sg.DistSolver(sg.SolverConfig(**cfgd))
        outs = []
        for _ in range(3):
            s.reset()
            s.solve()
            r = s.gather(0)
            if r is not None:
                outs.append((r.final_field.data.copy(), r.final_field.level))
        s.close()
        if rank == 0:
            q.put(("ok", outs))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e)))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("engine,problem", [("swept", "heat"), ("standard", "euler")])
def test_distributed_graph_replay(sg, oracle, engine, problem):
    """Repeated solves of one process per partition (graph replay with the
    device-side barrier epoch) stay bitwise equal to the oracle."""
    if sg.device_count() < 1:
        pytest.fail("no CUDA device")
    import torch.multiprocessing as mp
    nx = 64
    cfgd = dict(problem=problem, nx=nx, block=16 if problem == "heat" else 8, steps=20, engine=engine,
                ranks=2, px=2, py=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_repeat, args=(r, 2, port, cfgd, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=500)
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ok", res[1]
    outs = res[1]
    assert len(outs) == 3
    P = oracle.HEAT if problem == "heat" else oracle.EULER
    init, params = oracle.params(P, nx)
    want = oracle.standard_solve(P, init, outs[0][1], params)
    for data, level in outs:
        assert level == outs[0][1]
        assert np.array_equal(data, want)
