"""Benchmark / verification harness around run() -- the reference's bench.cpp
(sweep CSV, weak scaling, convergence check), re-targeted at the GPU engine.

    run_sweep(spec, csv_path)          bench.cpp:138-206, CSV header bench.cpp:60-63
    run_weak_scaling(spec, csv_path)   bench.cpp:208-244
    run_verify(problem, sizes)         bench.cpp:246-310
Solver numerics all run on the GPU through run(); only the analytic reference
fields (heat_analytic / vortex_analytic, physics.cpp:47-50, 193-216) are
evaluated here with numpy to measure errors (tolerances ~1e-4, not parity).
"""
from __future__ import annotations

import csv
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api

BENCH_CSV_HEADER = ("problem,nx,block,share,ranks,mode,repetition,actual_steps,run_seconds_standard,"
                    "run_seconds_swept,modeled_seconds_standard,modeled_seconds_swept,messages_standard,"
                    "messages_swept,speedup,error")


@dataclass
class SweepSpec:  # bench.hpp SweepSpec; desk_default bench.cpp:45-51
    problems: List[str] = field(default_factory=lambda: ["heat", "euler"])
    array_sizes: List[int] = field(default_factory=lambda: [80, 120, 160, 200, 240, 280])
    block_sizes: List[int] = field(default_factory=lambda: [8, 12, 16, 24, 32])
    shares: List[float] = field(default_factory=lambda: [i / 10.0 for i in range(11)])
    steps: int = 250
    repetitions: int = 1
    ranks: int = 1
    out_dir: str = "."

    @classmethod
    def desk_default(cls) -> "SweepSpec":
        return cls()

    @classmethod
    def paper_scale(cls) -> "SweepSpec":  # bench.cpp:53-58
        return cls(array_sizes=[320, 480, 640, 800, 960, 1120], steps=500)


def _key(problem, nx, block, share, ranks, mode):
    return f"{problem}|{nx}|{block}|{share:g}|{ranks}|{mode}"


def load_bench_csv(path: str) -> list:
    if not os.path.exists(path):
        return []
    with open(path) as f:
        return list(csv.DictReader(f))


def run_sweep(spec: SweepSpec, csv_path: str, log=None) -> None:
    """Swept, then standard at the swept run's actual step count; median of
    the repetitions; speedup = standard / swept; resumable by key."""
    done = {_key(r["problem"], int(r["nx"]), int(r["block"]), float(r["share"]), int(r["ranks"]), r["mode"])
            for r in load_bench_csv(csv_path)}
    fresh = not os.path.exists(csv_path)
    with open(csv_path, "a") as out:
        if fresh:
            out.write(BENCH_CSV_HEADER + "\n")
        for problem in spec.problems:
            for nx in spec.array_sizes:
                for b in spec.block_sizes:
                    if nx % b or (nx // b) % spec.ranks:
                        continue
                    for share in spec.shares:
                        if _key(problem, nx, b, share, spec.ranks, "wall") in done:
                            continue
                        row = dict(problem=problem, nx=nx, block=b, share=f"{share:g}", ranks=spec.ranks,
                                   mode="wall", repetition=spec.repetitions, actual_steps=0,
                                   run_seconds_standard=0.0, run_seconds_swept=0.0, modeled_seconds_standard=0.0,
                                   modeled_seconds_swept=0.0, messages_standard=0, messages_swept=0, speedup=0.0,
                                   error="")
                        try:
                            sw_t, st_t = [], []
                            for _ in range(spec.repetitions):
                                cfg = api.SolverConfig(problem=problem, nx=nx, block=b, share=share,
                                                       steps=spec.steps, ranks=spec.ranks)
                                sw = api.run(cfg).record
                                cfg.engine, cfg.steps = "standard", sw.actual_steps
                                st = api.run(cfg).record
                                sw_t.append(sw.wall_seconds)
                                st_t.append(st.wall_seconds)
                            row.update(actual_steps=sw.actual_steps, messages_swept=sw.messages,
                                       messages_standard=st.messages, run_seconds_swept=float(np.median(sw_t)),
                                       run_seconds_standard=float(np.median(st_t)))
                            row["speedup"] = row["run_seconds_standard"] / row["run_seconds_swept"]
                        except Exception as e:  # noqa: BLE001 -- recorded in the CSV like the reference
                            row["error"] = str(e).replace(",", ";").replace("\n", ";")
                        out.write(",".join(str(row[k]) for k in BENCH_CSV_HEADER.split(",")) + "\n")
                        out.flush()
                        if log:
                            log(f"{problem} nx={nx} b={b} share={share:g} speedup={row['speedup']:.4g}"
                                + (f" ERROR {row['error']}" if row["error"] else ""))


def run_weak_scaling(spec: SweepSpec, csv_path: str, log=None) -> None:
    """Constant points per rank, block 16, share 0.9 (bench.cpp:208-244);
    ranks = GPU partitions (spread over the visible GPUs)."""
    ladder = [(1, 192), (2, 288), (3, 336), (4, 384)]
    with open(csv_path, "w") as out:
        out.write("problem,ranks,nx,points_per_rank,engine,actual_steps,seconds,seconds_per_step,messages,bytes,"
                  "bytes_per_event\n")
        for problem in spec.problems:
            for ranks, nx in ladder:
                for engine in ("standard", "swept"):
                    r = api.run(api.SolverConfig(problem=problem, nx=nx, block=16, share=0.9, steps=spec.steps,
                                                 ranks=ranks, engine=engine)).record
                    events = r.communicates if engine == "swept" else r.total_levels
                    out.write(f"{problem},{ranks},{nx},{nx * nx // ranks},{engine},{r.actual_steps},{r.wall_seconds},"
                              f"{r.wall_seconds / r.actual_steps},{r.messages},{r.bytes},"
                              f"{(r.bytes / events) if events else 0.0}\n")
                    if log:
                        log(f"{problem} ranks={ranks} engine={engine} s/step={r.wall_seconds / r.actual_steps:.4g}")


# ----------------------------------------------------------------- verify --
def heat_analytic(x, y, t, alpha):  # physics.cpp:47-50
    return np.sin(2.0 * np.pi * x) * np.sin(2.0 * np.pi * y) * np.exp(-8.0 * np.pi * np.pi * alpha * t)


def vortex_analytic(nx, ny, gamma, t):  # physics.cpp:193-216 (VortexSpec::standard, :28-39)
    mach = math.sqrt(2.0 / gamma)
    alpha = math.pi / 4.0
    beta = mach * (5.0 * math.sqrt(2.0) / (4.0 * math.pi)) * math.exp(0.5)
    L = 5.0
    dx, dy = 2.0 * L / nx, 2.0 * L / ny
    ux, uy = mach * math.cos(alpha), mach * math.sin(alpha)

    def wrap(c):
        c = np.fmod(c + L, 2.0 * L)
        c = np.where(c < 0, c + 2.0 * L, c)
        return c - L

    y = wrap(-L + (np.arange(ny) + 0.5) * dy - uy * t)[:, None]
    x = wrap(-L + (np.arange(nx) + 0.5) * dx - ux * t)[None, :]
    f = -0.5 * (x * x + y * y)
    omega = beta * np.exp(f)
    du, dv = -y * omega, x * omega
    base = 1.0 - 0.5 * (gamma - 1.0) * omega * omega
    rho = base ** (1.0 / (gamma - 1.0))
    u, v = ux + du, uy + dv
    p = (1.0 / gamma) * base ** (gamma / (gamma - 1.0))
    e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return np.stack([rho, rho * u, rho * v, e])


@dataclass
class VerifyRow:
    nx: int
    steps: int
    t_final: float
    err_linf: float
    err_l2: float


@dataclass
class VerifyReport:
    rows: List[VerifyRow]
    observed_order: float
    passed: bool


def run_verify(problem: str, sizes: Optional[List[int]] = None, log=None) -> VerifyReport:
    """bench.cpp:246-310: heat at a fixed final time (40 coarse steps, dt ~ dx^2)
    must converge at order >= 1.9; Euler (t = 0.5) errors must shrink."""
    sizes = sizes or ([32, 64, 128] if problem == "heat" else [64, 128, 256])
    rows = []
    for nx in sizes:
        cfg = api.SolverConfig(problem=problem, nx=nx, block=8, engine="standard", ranks=1, steps=1)
        probe = api.run(cfg).record  # dt of this grid (make_setup)
        cfg.steps = 40 * (nx // sizes[0]) ** 2 if problem == "heat" else max(1, round(0.5 / probe.dt))
        res = api.run(cfg)
        t = res.record.actual_steps * res.record.dt
        if problem == "heat":
            xs = np.arange(nx) / nx
            exact = heat_analytic(xs[None, :], xs[:, None], t, cfg.heat_alpha)
            err = res.final_field.data[0] - exact
        else:
            err = res.final_field.data[0] - vortex_analytic(nx, nx, cfg.gamma, t)[0]
        rows.append(VerifyRow(nx, res.record.actual_steps, t, float(np.abs(err).max()),
                              float(np.sqrt((err * err).sum() / (nx * nx)))))
        if log:
            log(f"nx={nx} steps={rows[-1].steps} t={t:.6g} Linf={rows[-1].err_linf:.6g} L2={rows[-1].err_l2:.6g}")
    order = math.log(rows[0].err_linf / rows[-1].err_linf) / math.log(rows[-1].nx / rows[0].nx)
    monotone = all(rows[i].err_linf < rows[i - 1].err_linf for i in range(1, len(rows)))
    return VerifyReport(rows, order, order >= 1.9 if problem == "heat" else monotone)
