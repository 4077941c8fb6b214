#!/usr/bin/env python3
"""A/B of the swept heat phase kernels: generic table-driven (SG_HEAT_KERNEL=generic)
vs column-register (default for b in 8/16/32).  Same config, final fields
compared bit for bit, solve time (CUDA graph replay) and the dominant launch's
mean time.  One JSON line per (config, kernel).

    python profiles/ab_heat.py [--nx 8192] [--steps 1000] [--blocks 16]
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--blocks", default="16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kernels", default="generic,column")
    ap.add_argument("--problem", default="heat")
    args = ap.parse_args()
    import numpy as np
    import paper_2105_10332_b200 as sg

    for b in [int(x) for x in args.blocks.split(",")]:
        ref = None
        for kern in args.kernels.split(","):
            os.environ["SG_HEAT_KERNEL"] = kern
            cfg = sg.SolverConfig(problem=args.problem, nx=args.nx, block=b, steps=args.steps)
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
            kinds = {}
            for name, kd in (("oct", 3), ("yb", 1), ("xb", 2)):
                p = sg.Solver(cfg, profile=2 + kd)
                p.reset()
                p.solve()
                kinds[name] = p.kernel_stats()
                p.close()
            k = kinds["oct"]
            same = None
            if ref is None:
                ref = r.final_field.data
            else:
                same = bool(np.array_equal(ref, r.final_field.data))
            upd = r.record.cell_updates
            print(json.dumps({"problem": args.problem, "nx": args.nx, "block": b, "kernel": kern, "steps": r.record.actual_steps,
                              "solve_s": min(t), "updates_per_s": upd / min(t),
                              "dominant_launch_ms": 1e3 * k["seconds"] / max(1, k["launches"]),
                              "dominant_launches": k["launches"],
                              "dominant_alg_GBs": k["alg_bytes"] / max(k["seconds"], 1e-12) / 1e9,
                              "yb_launch_ms": 1e3 * kinds["yb"]["seconds"] / max(1, kinds["yb"]["launches"]),
                              "xb_launch_ms": 1e3 * kinds["xb"]["seconds"] / max(1, kinds["xb"]["launches"]),
                              "bitwise_equal_to_first": same}), flush=True)


if __name__ == "__main__":
    main()
