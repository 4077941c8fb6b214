"""Host-side mirror of the reference's public API for the swept hot path.

Reference (C++, /root/reference/proj):
    SolverConfig            include/sweptgrid/config.hpp:28-56 (+ from_json/to_json config.cpp:79-125)
    RunRecord / RunResult   include/sweptgrid/engine.hpp:35-64 (to_json engine.cpp:461-491)
    run(const SolverConfig&) -> RunResult                          engine.hpp:61
    run_substep_serial/omp(SubstepArgs, span<CellBlock>)           physics.hpp:132-134
    max_levels / build_schedule                                    geometry.hpp:41-103
    NonPhysicalState / std::invalid_argument / TransportError      physics.hpp:18, transport.hpp:62

Same names, argument meaning and error behaviour; every call goes through the
C-ABI of libsweptgpu.so (no CPU path).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi as _c


# ----------------------------------------------------------------- errors --
class SweptError(RuntimeError):
    code = _c.SG_ELOGIC


class InvalidArgument(SweptError, ValueError):  # std::invalid_argument
    code = _c.SG_EINVAL


class NonPhysicalState(SweptError):  # physics.hpp:18-20
    code = _c.SG_ENONPHYS


class TransportError(SweptError):  # transport.hpp:62-64
    code = _c.SG_ETRANSPORT


class SnapshotIOError(SweptError, OSError):  # std::runtime_error (I/O)
    code = _c.SG_EIO


class LogicError(SweptError):  # std::logic_error
    code = _c.SG_ELOGIC


class CudaError(SweptError):
    code = _c.SG_ECUDA


_ERRORS = {c.code: c for c in (InvalidArgument, NonPhysicalState, TransportError, SnapshotIOError, LogicError,
                               CudaError)}


def _check(rc: int, err) -> None:
    if rc != _c.SG_OK:
        msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
        raise _ERRORS.get(rc, SweptError)(msg)


# ----------------------------------------------------------------- config --
PROBLEMS = {"heat": _c.SG_HEAT, "euler": _c.SG_EULER}
ENGINES = {"swept": _c.SG_SWEPT, "standard": _c.SG_STANDARD}
MODES = {"wall": _c.SG_WALL, "virtual": _c.SG_VIRTUAL}


def _name(table, v):
    for k, x in table.items():
        if x == v:
            return k
    raise InvalidArgument(f"unknown enum value {v}")


@dataclass
class PoolSpec:  # config.hpp:23-26
    workers: int = 1
    cost: float = 1.0


@dataclass
class LinkModel:  # transport.hpp:22-33
    latency: float = 0.0
    bandwidth: float = math.inf


@dataclass
class SolverConfig:
    """config.hpp:28-56; defaults config.hpp:29-48.  GPU extensions: ny, px,
    py (partition grid; default ranks x 1 like the reference's x-only
    decomposition) and devices (CUDA devices to spread partitions over)."""
    problem: str = "heat"
    nx: int = 64
    block: int = 8
    share: float = 1.0
    steps: int = 10
    ranks: int = 1
    engine: str = "swept"
    mode: str = "wall"
    link: LinkModel = field(default_factory=LinkModel)
    pool_a: PoolSpec = field(default_factory=PoolSpec)
    pool_b: PoolSpec = field(default_factory=PoolSpec)
    cell_cost: float = 5.0e-8
    heat_alpha: float = 1.0
    heat_fourier: float = 0.2
    gamma: float = 1.4
    cfl: float = 0.4
    snapshot_path: str = ""
    snapshot_every: int = 1
    ny: int = 0
    px: int = 0
    py: int = 0
    devices: int = 0

    def ny_(self) -> int:
        return self.ny or self.nx

    def _c(self) -> _c.sg_config:
        c = _c.sg_config()
        _c.load().sg_config_default(C.byref(c))
        if self.problem not in PROBLEMS:
            raise InvalidArgument(f"unknown problem: {self.problem}")
        if self.engine not in ENGINES:
            raise InvalidArgument(f"unknown engine: {self.engine}")
        if self.mode not in MODES:
            raise InvalidArgument(f"unknown transport mode: {self.mode}")
        c.problem = PROBLEMS[self.problem]
        c.nx, c.ny, c.block = int(self.nx), int(self.ny), int(self.block)
        c.share, c.steps, c.ranks = float(self.share), int(self.steps), int(self.ranks)
        c.engine, c.mode = ENGINES[self.engine], MODES[self.mode]
        c.link_latency, c.link_bandwidth = float(self.link.latency), float(self.link.bandwidth)
        c.pool_a_workers, c.pool_a_cost = int(self.pool_a.workers), float(self.pool_a.cost)
        c.pool_b_workers, c.pool_b_cost = int(self.pool_b.workers), float(self.pool_b.cost)
        c.cell_cost = float(self.cell_cost)
        c.heat_alpha, c.heat_fourier = float(self.heat_alpha), float(self.heat_fourier)
        c.gamma, c.cfl = float(self.gamma), float(self.cfl)
        self._path = self.snapshot_path.encode() if self.snapshot_path else None
        c.snapshot_path = self._path
        c.snapshot_every = int(self.snapshot_every)
        c.px, c.py, c.devices = int(self.px), int(self.py), int(self.devices)
        return c

    def validate(self) -> None:
        """SolverConfig::validate (config.cpp:31-62) + partition checks."""
        err = _c.errbuf()
        _check(_c.load().sg_validate(C.byref(self._c()), err, len(err)), err)

    # config.cpp:79-101
    @classmethod
    def from_json(cls, j: dict) -> "SolverConfig":
        c = cls()
        if "problem" in j:
            if j["problem"] not in PROBLEMS:
                raise InvalidArgument(f"unknown problem: {j['problem']}")
            c.problem = j["problem"]
        c.nx = j.get("nx", c.nx)
        c.block = j.get("block", c.block)
        c.share = j.get("share", c.share)
        c.steps = j.get("steps", c.steps)
        c.ranks = j.get("ranks", c.ranks)
        if "engine" in j:
            if j["engine"] not in ENGINES:
                raise InvalidArgument(f"unknown engine: {j['engine']}")
            c.engine = j["engine"]
        if "mode" in j:
            if j["mode"] not in MODES:
                raise InvalidArgument(f"unknown transport mode: {j['mode']}")
            c.mode = j["mode"]
        c.link = LinkModel(j.get("latency", 0.0), j.get("bandwidth", math.inf))
        if "pool_a" in j:
            c.pool_a = PoolSpec(j["pool_a"].get("workers", 1), j["pool_a"].get("cost", 1.0))
        if "pool_b" in j:
            c.pool_b = PoolSpec(j["pool_b"].get("workers", 1), j["pool_b"].get("cost", 1.0))
        c.cell_cost = j.get("cell_cost", c.cell_cost)
        c.heat_alpha = j.get("heat_alpha", c.heat_alpha)
        c.heat_fourier = j.get("heat_fourier", c.heat_fourier)
        c.gamma = j.get("gamma", c.gamma)
        c.cfl = j.get("cfl", c.cfl)
        c.snapshot_path = j.get("snapshot", c.snapshot_path)
        c.snapshot_every = j.get("snapshot_every", c.snapshot_every)
        c.ny = j.get("ny", 0)
        c.px = j.get("px", 0)
        c.py = j.get("py", 0)
        c.devices = j.get("devices", 0)
        return c

    # config.cpp:103-125
    def to_json(self) -> dict:
        j = {"problem": self.problem, "nx": self.nx, "block": self.block, "share": self.share,
             "steps": self.steps, "ranks": self.ranks, "engine": self.engine, "mode": self.mode,
             "latency": self.link.latency}
        if math.isfinite(self.link.bandwidth):
            j["bandwidth"] = self.link.bandwidth
        j["pool_a"] = {"workers": self.pool_a.workers, "cost": self.pool_a.cost}
        j["pool_b"] = {"workers": self.pool_b.workers, "cost": self.pool_b.cost}
        j.update(cell_cost=self.cell_cost, heat_alpha=self.heat_alpha, heat_fourier=self.heat_fourier,
                 gamma=self.gamma, cfl=self.cfl)
        if self.snapshot_path:
            j["snapshot"] = self.snapshot_path
        j["snapshot_every"] = self.snapshot_every
        if self.ny and self.ny != self.nx:
            j["ny"] = self.ny
        if self.px or self.py:
            j["px"], j["py"] = self.px, self.py
        return j

    @classmethod
    def load(cls, path: str) -> "SolverConfig":
        try:
            with open(path) as f:
                return cls.from_json(json.load(f))
        except OSError as e:
            raise SnapshotIOError(f"config: cannot open {path}") from e


# ---------------------------------------------------------------- results --
@dataclass
class FieldState:  # field.hpp:44-64, layout [var][y][x]
    nvars: int
    nx: int
    ny: int
    level: int
    data: np.ndarray  # shape (nvars, ny, nx), float64

    def at(self, v: int, x: int, y: int) -> float:
        return float(self.data[v, y, x])


@dataclass
class RunRecord:  # engine.hpp:35-59
    engine: str = ""
    problem: str = ""
    mode: str = "wall"
    nx: int = 0
    block: int = 0
    ranks: int = 0
    steps_requested: int = 0
    actual_steps: int = 0
    total_levels: int = 0
    octahedra: int = 0
    communicates: int = 0
    dt: float = 0.0
    setup_seconds: float = 0.0
    wall_seconds: float = 0.0
    modeled_seconds: float = 0.0
    messages: int = 0
    bytes: int = 0
    cell_updates: int = 0
    snapshot_frames: int = 0
    # GPU extras (not in the reference JSON unless asked)
    ny: int = 0
    px: int = 1
    py: int = 1
    solve_seconds: float = 0.0
    kernel_launches: int = 0
    final_level: int = 0
    part_messages: list = field(default_factory=list)
    part_bytes: list = field(default_factory=list)

    def to_json(self, gpu_extras: bool = False) -> dict:
        """engine.cpp:461-491 key set and order."""
        j = {k: getattr(self, k) for k in (
            "engine", "problem", "mode", "nx", "block", "ranks", "steps_requested", "actual_steps",
            "total_levels", "octahedra", "communicates", "dt", "setup_seconds", "wall_seconds",
            "modeled_seconds", "messages", "bytes", "cell_updates", "snapshot_frames")}
        # per_rank (engine.cpp:482-489): one entry per partition = rank, the
        # pushes it made into other partitions; the virtual clocks are 0
        pm = self.part_messages or [0] * max(1, self.ranks)
        pb = self.part_bytes or [0] * max(1, self.ranks)
        j["per_rank"] = [{"messages": int(m), "bytes": int(b), "comm_seconds": 0.0, "compute_seconds": 0.0,
                          "clock": 0.0} for m, b in zip(pm, pb)]
        if gpu_extras:
            j.update(ny=self.ny, px=self.px, py=self.py, solve_seconds=self.solve_seconds,
                     kernel_launches=self.kernel_launches, final_level=self.final_level)
        return j


@dataclass
class RunResult:  # engine.hpp:61-64
    final_field: FieldState
    record: RunRecord


def _result(r: _c.sg_result) -> RunResult:
    n = r.nvars * r.nx * r.ny
    data = np.ctypeslib.as_array(r.final_field, shape=(n,)).copy().reshape(r.nvars, r.ny, r.nx)
    rec = RunRecord(
        engine=_name(ENGINES, r.engine), problem=_name(PROBLEMS, r.problem), mode=_name(MODES, r.mode), nx=r.nx,
        block=r.block, ranks=r.ranks, steps_requested=r.steps_requested, actual_steps=r.actual_steps,
        total_levels=r.total_levels, octahedra=r.octahedra, communicates=r.communicates, dt=r.dt,
        setup_seconds=r.setup_seconds, wall_seconds=r.wall_seconds, modeled_seconds=r.modeled_seconds,
        messages=r.messages, bytes=r.bytes, cell_updates=r.cell_updates, snapshot_frames=r.snapshot_frames,
        ny=r.ny, px=r.px, py=r.py, solve_seconds=r.solve_seconds, kernel_launches=r.kernel_launches,
        final_level=r.final_level,
        part_messages=[int(r.part_messages[q]) for q in range(r.nparts)] if r.part_messages else [],
        part_bytes=[int(r.part_bytes[q]) for q in range(r.nparts)] if r.part_bytes else [])
    return RunResult(FieldState(r.nvars, r.nx, r.ny, r.final_level, data), rec)


def run(cfg: SolverConfig) -> RunResult:
    """sweptgrid::run (engine.cpp:493-568) on the GPU: synchronous, host in/out."""
    L = _c.load()
    c = cfg._c()
    res = _c.sg_result()
    err = _c.errbuf()
    rc = L.sg_run(C.byref(c), C.byref(res), err, len(err))
    try:
        _check(rc, err)
        return _result(res)
    finally:
        L.sg_free_result(C.byref(res))


def _host_f64_ptr(host, shape, what: str) -> int:
    """Address of a host float64 buffer holding exactly prod(shape) elements
    in C order (numpy array or CPU torch tensor); InvalidArgument otherwise
    -- the C side reads or writes that many doubles through the pointer."""
    n = int(np.prod(shape))
    if hasattr(host, "data_ptr"):  # torch.Tensor
        import torch
        if host.device.type != "cpu":
            raise InvalidArgument(f"{what}: host buffer expected, got a {host.device} tensor")
        if host.dtype != torch.float64:
            raise InvalidArgument(f"{what}: float64 buffer expected, got {host.dtype}")
        if not host.is_contiguous():
            raise InvalidArgument(f"{what}: buffer must be contiguous")
        if host.numel() != n:
            raise InvalidArgument(f"{what}: buffer holds {host.numel()} values, expected {n} {tuple(shape)}")
        return host.data_ptr()
    if isinstance(host, np.ndarray):
        if host.dtype != np.float64:
            raise InvalidArgument(f"{what}: float64 buffer expected, got {host.dtype}")
        if not host.flags.c_contiguous:
            raise InvalidArgument(f"{what}: buffer must be C-contiguous")
        if host.size != n:
            raise InvalidArgument(f"{what}: buffer holds {host.size} values, expected {n} {tuple(shape)}")
        if not host.flags.writeable and what != "upload":
            raise InvalidArgument(f"{what}: buffer is read-only")
        return host.ctypes.data
    raise InvalidArgument(f"{what}: numpy array or CPU torch tensor expected, got {type(host).__name__}")


def fnv1a64(data) -> str:
    """FNV-1a-64 of a float64 field's bytes (hex), the fingerprint of the
    reference's parity probes, computed by the library."""
    a = np.ascontiguousarray(data)
    return f"{_c.load().sg_fnv1a64(C.c_void_p(a.ctypes.data), a.nbytes):016x}"


class Solver:
    """Resident solver (sg_solver_*): create once, then reset/solve/fetch.
    Used by bench.py to time the solve with inputs already in HBM."""

    def __init__(self, cfg: SolverConfig, profile=False, _dist=None):
        self._L = _c.load()
        self._cfg = cfg._c()
        h = C.c_void_p()
        err = _c.errbuf()
        if _dist is None:
            _check(self._L.sg_solver_create(C.byref(self._cfg), C.byref(h), err, len(err)), err)
        else:
            rank, world = _dist
            _check(self._L.sg_dist_create(C.byref(self._cfg), rank, world, C.byref(h), err, len(err)), err)
        self._h = h
        self._dist = _dist
        if profile:  # True: the dominant kernel; an int k >= 2: swept phase kind k - 2
            self._L.sg_solver_set_profile(self._h, int(profile))

    def reset(self) -> None:
        err = _c.errbuf()
        _check(self._L.sg_solver_reset(self._h, err, len(err)), err)

    def solve(self) -> float:
        t = C.c_double(0.0)
        err = _c.errbuf()
        _check(self._L.sg_solver_solve(self._h, C.byref(t), err, len(err)), err)
        return t.value

    def fetch(self) -> RunResult:
        res = _c.sg_result()
        err = _c.errbuf()
        rc = self._L.sg_solver_fetch(self._h, C.byref(res), err, len(err))
        try:
            _check(rc, err)
            return _result(res)
        finally:
            self._L.sg_free_result(C.byref(res))

    def _piece_shape(self, whole: bool = False):
        """(nvars, rows, cols) of the host arrays upload/download take: the
        global field, or this rank's partition piece in a distributed run
        (initial() always writes the whole global field: whole=True)."""
        c = self._cfg
        nv = 1 if c.problem == _c.SG_HEAT else 4
        ny = c.ny if c.ny > 0 else c.nx
        if whole or getattr(self, "_dist", None) is None:
            return nv, ny, c.nx
        px = c.px if c.px > 0 else (c.ranks if c.py <= 0 else 1)
        py = c.py if c.py > 0 else 1
        return nv, ny // py, c.nx // px

    def _host_ptr(self, host, what: str) -> C.c_void_p:
        return C.c_void_p(_host_f64_ptr(host, self._piece_shape(whole=what == "initial"), what))

    def upload(self, host) -> None:
        """Replace level 0 from a host array [var][ny][nx] float64 (numpy, or a
        pinned torch CPU tensor): the e2e input path."""
        err = _c.errbuf()
        _check(self._L.sg_solver_upload(self._h, self._host_ptr(host, "upload"), err, len(err)), err)

    def download(self, host) -> None:
        """Final field into a host array [var][ny][nx] float64."""
        err = _c.errbuf()
        _check(self._L.sg_solver_download(self._h, self._host_ptr(host, "download"), err, len(err)), err)

    def initial(self, host) -> None:
        """The initial condition make_setup computed (engine.cpp:27-70) into a
        host array of the global field's shape (also in a distributed run)."""
        err = _c.errbuf()
        _check(self._L.sg_solver_initial(self._h, self._host_ptr(host, "initial"), err, len(err)), err)

    def kernel_stats(self) -> dict:
        s, n, b, u = C.c_double(), C.c_long(), C.c_double(), C.c_double()
        self._L.sg_solver_kernel_stats(self._h, 0, C.byref(s), C.byref(n), C.byref(b), C.byref(u))
        return {"seconds": s.value, "launches": n.value, "alg_bytes": b.value, "updates": u.value}

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.sg_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class DistSolver(Solver):
    """One process per GPU (launched by torchrun): this rank owns partition
    `rank` of the cfg.px x cfg.py grid (world size == px*py) on its current
    CUDA device.  torch.distributed is plumbing only: it all-gathers the CUDA
    IPC handles once; afterwards partition-edge cells travel as P2P stores
    from inside the phase kernels and launches are ordered by device-side
    flags (the reference's Transport::exchange, transport.hpp:78-79)."""

    def __init__(self, cfg: SolverConfig, rank: int = None, world: int = None, group=None, profile: bool = False):
        import torch.distributed as dist
        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
        if not cfg.px and not cfg.py:
            cfg.px, cfg.py = world, 1
        if cfg.ranks != cfg.px * cfg.py:
            cfg.ranks = cfg.px * cfg.py
        super().__init__(cfg, profile=profile, _dist=(rank, world))
        self.rank, self.world, self.cfg = rank, world, cfg
        err = _c.errbuf()
        n = self._L.sg_dist_blob(self._h, None, 0, err, len(err))
        if n < 0:
            _check(-n, err)
        buf = C.create_string_buffer(n)
        self._L.sg_dist_blob(self._h, buf, n, err, len(err))
        blobs = [None] * world
        dist.all_gather_object(blobs, bytes(buf.raw), group=group)
        allb = b"".join(blobs)
        _check(self._L.sg_dist_connect(self._h, allb, n, err, len(err)), err)

    def gather(self, dst: int = 0, group=None):
        """Assemble the global final field on rank `dst` (None elsewhere)."""
        import torch.distributed as dist
        res = self.fetch()
        pi, pj = self.rank % self.cfg.px, self.rank // self.cfg.px
        pw, ph = res.final_field.nx // self.cfg.px, res.final_field.ny // self.cfg.py
        piece = res.final_field.data[:, pj * ph:(pj + 1) * ph, pi * pw:(pi + 1) * pw].copy()
        pieces = [None] * self.world if self.rank == dst else None
        dist.gather_object(piece, pieces, dst=dst, group=group)
        if self.rank != dst:
            return None
        full = np.zeros_like(res.final_field.data)
        for q, pc in enumerate(pieces):
            qi, qj = q % self.cfg.px, q // self.cfg.px
            full[:, qj * ph:(qj + 1) * ph, qi * pw:(qi + 1) * pw] = pc
        res.final_field.data = full
        return res


def run_distributed(cfg: SolverConfig, group=None) -> Optional[RunResult]:
    """run() with one process per GPU (torchrun); RunResult on rank 0."""
    import time as _t
    s = DistSolver(cfg, group=group)
    t0 = _t.perf_counter()
    s.reset()
    secs = s.solve()
    out = s.gather(0, group=group)
    wall = _t.perf_counter() - t0
    s.close()
    if out is not None:
        out.record.wall_seconds = wall
        out.record.solve_seconds = secs
    return out


# --------------------------------------------------------------- snapshots --
_MAGIC = b"SWPT2D\0\0"


@dataclass
class SnapshotFrame:  # snapshot.hpp:199-202
    level: int
    data: np.ndarray  # (nvars, ny, nx)


class SnapshotReader:
    """SWPT2D v1 reader (snapshot.cpp:86-115): magic, u32 version, u64 header
    length, JSON header, then (u64 level, f64[var][y][x]) frames."""

    def __init__(self, path: str):
        import struct
        try:
            raw = open(path, "rb").read()
        except OSError as e:
            raise SnapshotIOError(f"snapshot: cannot open {path}") from e
        if raw[:8] != _MAGIC:
            raise SnapshotIOError("snapshot: bad magic")
        (version,) = struct.unpack_from("<I", raw, 8)
        if version != 1:
            raise SnapshotIOError("snapshot: unsupported version")
        (hlen,) = struct.unpack_from("<Q", raw, 12)
        if 20 + hlen > len(raw):
            raise SnapshotIOError("snapshot: truncated header")
        self._meta = json.loads(raw[20:20 + hlen].decode())
        m = self._meta
        plane = m["nvars"] * m["nx"] * m["ny"]
        off, self._frames = 20 + hlen, []
        while off < len(raw):
            if off + 8 + 8 * plane > len(raw):
                raise SnapshotIOError("snapshot: truncated frame")
            (level,) = struct.unpack_from("<Q", raw, off)
            data = np.frombuffer(raw, dtype="<f8", count=plane, offset=off + 8).reshape(m["nvars"], m["ny"], m["nx"])
            self._frames.append(SnapshotFrame(int(level), data.copy()))
            off += 8 + 8 * plane

    def meta(self) -> dict:
        return self._meta

    def frames(self) -> list:
        return self._frames


def measure_fp64_peak() -> float:
    """FP64 flop/s of cuda:0 without FMA (DADD + DMUL chains), -1 without a GPU."""
    return float(_c.load().sg_measure_fp64_peak())


# ------------------------------------------------------- geometry / plugin --
def max_levels(b: int, n: int) -> int:
    """geometry.cpp:59-66; raises InvalidArgument like the reference."""
    k = _c.load().sg_max_levels(b, n)
    if k < 0:
        raise InvalidArgument(f"max_levels: invalid block {b} for halo {n}")
    return k


def build_schedule(requested_steps: int, b: int, n: int, substeps: int) -> dict:
    """geometry.cpp:169-184 arithmetic: {k, octahedra, flat_level, completed_steps, communicates}."""
    flat = C.c_long(0)
    m = _c.load().sg_schedule(requested_steps, b, n, substeps, C.byref(flat))
    if m < 0:
        raise InvalidArgument("build_schedule: invalid request")
    return {"k": max_levels(b, n), "octahedra": m, "flat_level": flat.value,
            "completed_steps": flat.value // substeps, "communicates": m + 1}


def plan_info(problem: str, block: int, steps: int) -> dict:
    """Compile the GPU swept plan on the host (no GPU) and return its statistics."""
    stats = (C.c_long * 16)()
    text = C.create_string_buffer(1 << 16)
    err = _c.errbuf()
    _check(_c.load().sg_plan_info(PROBLEMS[problem], block, steps, stats, text, len(text), err, len(err)), err)
    keys = ("k", "m", "flat", "launches", "classes", "slots", "ghost", "max_record", "oct_imports",
            "oct_exports", "oct_updates", "yb_imports", "yb_exports", "yb_updates", "oct_smem_bytes",
            "replay_cycles")
    d = dict(zip(keys, list(stats)))
    d["text"] = text.value.decode()
    return d


def substep(problem: str, stage: int, read1, read2, out, rects, params, stream=None) -> None:
    """run_substep on DEVICE tensors (torch CUDA tensors or raw pointers):
    physics.hpp:132-134.  read1/read2/out: float64 [nvars][ny][nx] contiguous."""
    L = _c.load()
    nvars, ny, nx = (int(s) for s in read1.shape)
    r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
    err = _c.errbuf()

    if nvars != (1 if problem == "heat" else 4):
        raise InvalidArgument(f"substep: {problem} needs {1 if problem == 'heat' else 4} variables, got {nvars}")

    def ptr(t):
        if hasattr(t, "data_ptr"):  # torch tensor: a device buffer of read1's shape
            import torch
            if not t.is_cuda:
                raise InvalidArgument("substep: device (CUDA) tensors expected")
            if t.dtype != torch.float64 or not t.is_contiguous():
                raise InvalidArgument("substep: contiguous float64 tensors expected")
            if tuple(t.shape) != (nvars, ny, nx):
                raise InvalidArgument(f"substep: shape {tuple(t.shape)} != read1's {(nvars, ny, nx)}")
            return C.c_void_p(t.data_ptr())
        return C.c_void_p(int(t))  # a raw device pointer: the caller vouches for it

    s = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else (stream or 0))
    rc = L.sg_substep(PROBLEMS[problem], stage, ptr(read1), ptr(read2), ptr(out), nvars, nx, ny,
                      r.ctypes.data_as(C.POINTER(C.c_int)), r.shape[0], p.ctypes.data_as(C.POINTER(C.c_double)),
                      s, err, len(err))
    _check(rc, err)


def device_count() -> int:
    return _c.load().sg_device_count()


def version() -> str:
    return _c.load().sg_version().decode()
