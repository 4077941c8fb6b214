#!/usr/bin/env python3
"""A/B of kernel variants selected by environment switches (read once per
process by the library, so every variant runs in its own process).

For each variant: whole-solve rate on the graph path (the bench's headline
path), per-kind mean launch time (profiling pass, events around every launch
of that kind) and the FNV-1a-64 of the final field (all variants must agree).

    python profiles/ab_env.py --nx 8192 --steps 1000 --block 16 \
        --variant base: --variant cpl2:SG_BRIDGE_CPL=2
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(args):
    sys.path.insert(0, str(ROOT))
    import paper_2105_10332_b200 as sg
    cfg = sg.SolverConfig(problem=args.problem, nx=args.nx, block=args.block, steps=args.steps,
                          engine=args.engine)
    s = sg.Solver(cfg)
    for _ in range(2):
        s.reset()
        s.solve()
    t = []
    for _ in range(args.reps):
        s.reset()
        t.append(s.solve())
    r = s.fetch()
    s.close()
    out = {"rate": r.record.cell_updates / min(t), "ms": 1e3 * min(t), "actual_steps": r.record.actual_steps,
           "fnv1a64": sg.fnv1a64(r.final_field.data)}
    if args.engine == "swept":
        for name, kd in (("up", 0), ("yb", 1), ("xb", 2), ("oct", 3), ("down", 4)):
            p = sg.Solver(cfg, profile=2 + kd)
            p.reset()
            p.solve()
            k = p.kernel_stats()
            p.close()
            if k["launches"]:
                out[f"{name}_ms"] = round(1e3 * k["seconds"] / k["launches"], 4)
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--block", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--problem", default="heat")
    ap.add_argument("--engine", default="swept")
    ap.add_argument("--variant", action="append", default=[], help="name:K=V,K=V")
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        return child(args)
    ref = None
    for v in args.variant or ["base:"]:
        name, _, kv = v.partition(":")
        env = dict(os.environ)
        for item in filter(None, kv.split(",")):
            k, _, val = item.partition("=")
            env[k] = val
        cmd = [sys.executable, __file__, "--child", "--nx", str(args.nx), "--steps", str(args.steps), "--block",
               str(args.block), "--reps", str(args.reps), "--problem", args.problem, "--engine", args.engine]
        p = subprocess.run(cmd, env=env, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(json.dumps({"variant": name, "error": p.stderr[-1500:]}), flush=True)
            continue
        d = json.loads(line[0][7:])
        if ref is None:
            ref = d["fnv1a64"]
        d.update(variant=name, env=kv, nx=args.nx, block=args.block, same_as_first=d["fnv1a64"] == ref)
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    sys.exit(main())
