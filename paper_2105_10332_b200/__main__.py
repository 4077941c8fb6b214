"""CLI: ``python -m paper_2105_10332_b200 run|sweep|weak-scaling|verify`` -- the reference's
``sweptgrid run`` (proj/tools/sweptgrid_main.cpp:48-65, 83-116): flags override
an optional JSON config, the solve runs on the GPU, and the RunRecord is
printed as 2-space-indented JSON (``record.to_json().dump(2)``).  Errors go to
stderr as ``error: ...`` with exit status 1.  ``sweep`` / ``weak-scaling`` /
``verify`` mirror bench.cpp (CSV schemas, convergence check); ``render`` (SVG
heatmaps) is out of scope.
"""
import argparse
import json
import sys

from . import api, harness


def _pool(s: str) -> api.PoolSpec:  # "workers:cost", sweptgrid_main.cpp parse_pool
    w, _, c = s.partition(":")
    return api.PoolSpec(int(w), float(c) if c else 1.0)


def build_config(a) -> api.SolverConfig:
    cfg = api.SolverConfig.load(a.config) if a.config else api.SolverConfig()
    if a.problem is not None:
        if a.problem not in api.PROBLEMS:
            raise api.InvalidArgument(f"unknown problem: {a.problem}")
        cfg.problem = a.problem
    for name in ("nx", "block", "share", "steps", "ranks", "ny", "px", "py", "devices"):
        v = getattr(a, name)
        if v is not None:
            setattr(cfg, name, v)
    if a.engine is not None:
        cfg.engine = a.engine
    if a.mode is not None:
        cfg.mode = a.mode
    if a.latency is not None:
        cfg.link.latency = a.latency
    if a.bandwidth is not None:
        cfg.link.bandwidth = a.bandwidth
    if a.pool_a:
        cfg.pool_a = _pool(a.pool_a)
    if a.pool_b:
        cfg.pool_b = _pool(a.pool_b)
    if a.out:
        cfg.snapshot_path = a.out
    return cfg


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2105_10332_b200",
                                 description="B200 swept-rule PDE solver (run subcommand)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="single solve, prints a JSON record")
    r.add_argument("--problem")
    r.add_argument("--nx", type=int)
    r.add_argument("--block", type=int)
    r.add_argument("--share", type=float)
    r.add_argument("--steps", type=int)
    r.add_argument("--ranks", type=int)
    r.add_argument("--engine", choices=["swept", "standard"])
    r.add_argument("--mode", choices=["wall", "virtual"])
    r.add_argument("--latency", type=float)
    r.add_argument("--bandwidth", type=float)
    r.add_argument("--pool-a")
    r.add_argument("--pool-b")
    r.add_argument("--config", help="JSON config file (flags override)")
    r.add_argument("--out", help="snapshot output path (SWPT2D)")
    r.add_argument("--ny", type=int, help="GPU extension: non-square grids")
    r.add_argument("--px", type=int, help="GPU extension: partition grid")
    r.add_argument("--py", type=int)
    r.add_argument("--devices", type=int)
    sw = sub.add_parser("sweep", help="parameter sweep to CSV (bench.cpp run_sweep)")
    sw.add_argument("--problem")
    sw.add_argument("--steps", type=int)
    sw.add_argument("--ranks", type=int)
    sw.add_argument("--reps", type=int)
    sw.add_argument("--paper-scale", action="store_true")
    sw.add_argument("--out", default=".")
    wk = sub.add_parser("weak-scaling", help="constant work per rank (bench.cpp run_weak_scaling)")
    wk.add_argument("--problem")
    wk.add_argument("--steps", type=int)
    wk.add_argument("--out", default=".")
    vf = sub.add_parser("verify", help="convergence vs analytic solutions (exit 0 = pass)")
    vf.add_argument("--problem", default="heat")
    vf.add_argument("--sizes", type=int, nargs="*")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            res = api.run(build_config(a))
            print(json.dumps(res.record.to_json(), indent=2))
            return 0
        if a.cmd in ("sweep", "weak-scaling"):
            import os
            spec = harness.SweepSpec.paper_scale() if getattr(a, "paper_scale", False) else harness.SweepSpec()
            if a.problem:
                spec.problems = [a.problem]
            if a.steps:
                spec.steps = a.steps
            if getattr(a, "ranks", None):
                spec.ranks = a.ranks
            if getattr(a, "reps", None):
                spec.repetitions = a.reps
            os.makedirs(a.out, exist_ok=True)
            path = os.path.join(a.out, "sweep.csv" if a.cmd == "sweep" else "weak_scaling.csv")
            log = lambda m: print(m, file=sys.stderr)  # noqa: E731
            (harness.run_sweep if a.cmd == "sweep" else harness.run_weak_scaling)(spec, path, log)
            print(path)
            return 0
        rep = harness.run_verify(a.problem, a.sizes or None, lambda m: print(m))
        print(f"observed order {rep.observed_order:.4g} ({'pass' if rep.passed else 'FAIL'})")
        return 0 if rep.passed else 1
    except Exception as e:  # noqa: BLE001 -- mirror `catch (const std::exception&)`
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
