#!/usr/bin/env python3
"""Block-size sweep (BASELINE configs[2] / SURVEY.md §8d C3): heat 4128^2
(4096 is not divisible by 12 or 24) at b = 8, 12, 16, 24, 32 on one B200,
swept vs standard, with the dominant swept kernel's roofline fraction against
the minimum swept traffic of SURVEY §8d.  Also Euler 960^2 at b = 8, 12, 16, 24.
Prints one JSON line per configuration.

    python bench_sweep.py [--steps-heat 5000] [--reps 3]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps-heat", type=int, default=5000)
    ap.add_argument("--steps-euler", type=int, default=500)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nx", type=int, default=4128)
    ap.add_argument("--paper-sizes", action="store_true",
                    help="the paper's array sizes 320..1120 (PAPER.md:138), b16, 500 steps")
    args = ap.parse_args()
    import paper_2105_10332_b200 as sg
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6650.0}

    fp64 = sg.measure_fp64_peak()

    def timed(cfg, profile=False):
        s = sg.Solver(cfg)  # timed runs replay the solve's CUDA graph
        for _ in range(2):
            s.reset()
            s.solve()
        t = []
        for _ in range(args.reps):
            s.reset()
            t.append(s.solve())
        r = s.fetch()
        s.close()
        k = {"launches": 0}
        if profile:  # separate pass with per-launch events for the dominant kernel
            s = sg.Solver(cfg, profile=True)
            s.reset()
            s.solve()
            k = s.kernel_stats()
            s.close()
        return min(t), r, k

    cases = [("heat", args.nx, b, args.steps_heat) for b in (8, 12, 16, 24, 32)] + \
        [("euler", 960, b, args.steps_euler) for b in (8, 12, 16, 24)]
    if args.paper_sizes:
        cases = [(p, nx, 16, 500) for p in ("heat", "euler") for nx in (320, 480, 640, 800, 960, 1120)]
    for problem, nx, b, steps in cases:
        if True:
            line = {"problem": problem, "nx": nx, "block": b, "requested_steps": steps}
            try:
                ts, rs, ks = timed(sg.SolverConfig(problem=problem, nx=nx, block=b, steps=steps), profile=True)
                tt, rt, _ = timed(sg.SolverConfig(problem=problem, nx=nx, block=b, steps=rs.record.actual_steps,
                                                  engine="standard"))
                import numpy as np
                line.update(
                    actual_steps=rs.record.actual_steps,
                    swept_updates_per_s=rs.record.cell_updates / ts,
                    standard_updates_per_s=rt.record.cell_updates / tt,
                    swept_over_standard=(rs.record.cell_updates / ts) / (rt.record.cell_updates / tt),
                    bitwise_equal=bool(np.array_equal(rs.final_field.data, rt.final_field.data)))
                if problem == "heat" and ks["launches"]:
                    gbs = ks["alg_bytes"] / ks["seconds"] / 1e9
                    line.update(oct_alg_GBps=round(gbs, 1), oct_roofline_frac=round(gbs / peaks["hbm_gbs"], 4),
                                oct_share=round(ks["seconds"] / ts, 3))
                    # SURVEY.md §8d whole-solve roofline: min(HBM / B_alg, FP64 / 9 flops)
                    bpu = {8: 15.50, 12: 10.44, 16: 7.875, 24: 5.28, 32: 3.97}.get(b)
                    if bpu and fp64 > 0:
                        ceil = min(peaks["hbm_gbs"] * 1e9 / bpu, fp64 / 9.0)
                        line.update(solve_roofline_frac=round(rs.record.cell_updates / ts / ceil, 4))
            except Exception as e:  # noqa: BLE001
                line["error"] = str(e)
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
