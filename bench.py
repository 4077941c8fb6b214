#!/usr/bin/env python3
"""Benchmark: 2D swept-rule heat, weak scaling, 8192^2 cells per GPU, b=16,
10k requested steps (BASELINE.json configs[4]) -- swept and standard engines.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one full solve of the workload (10003 sub-step levels of the
8192^2-per-GPU grid) from the resident initial condition.  Prints ONE JSON
line on rank 0 (contract in the task statement):
  value     swept cell-updates/s over all GPUs, inputs resident in HBM, device
            time (CUDA events on the launching stream), max over ranks
  e2e       the same through the C-ABI with host buffers: pinned H2D of the
            initial field + solve + D2H of the final field, every step
  roofline  dominant kernel (Octahedron phase): algorithmic bytes per launch /
            mean launch time (CUDA events around each launch), vs measured HBM
  cpu_baseline  the reference (oracle/_ref, built from its own sources) timed
            on this host on a bounded sample of the same workload
Synthetic data = the reference's own deterministic initial condition
(sin*sin, engine.cpp:31-42).  Inputs (537 MB/plane) exceed L2 (126 MB).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PER_GPU = 8192
BLOCK = 16
REQ_STEPS = 10000
METRIC = "cell-updates/sec (fp64) + swept/standard speedup at 1/2/4/8 B200 vs CPU ref"
GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:  # noqa: BLE001
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows, self.proc = [], None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                      "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for i, nm in enumerate(names):
                    if r[5 + i].lower() == "active":
                        reasons.add(nm)
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(tag: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture summary (profiles/*.json with a matching `workload`)."""
    best = None
    for p in sorted((ROOT / "profiles").glob("*.json")):
        try:
            j = json.loads(p.read_text())
        except Exception:  # noqa: BLE001
            continue
        if isinstance(j, dict) and j.get("workload") == tag and j.get("dram_bytes_per_launch"):
            best = (j["dram_bytes_per_launch"], p.name)
    return best


def cpu_reference_sample(nx, ny, steps, engine, threads):
    """Time the reference (oracle/_ref/ref_run, built from the reference's own
    sources) on a bounded sample; returns (cell-updates/s, record)."""
    exe = ROOT / "oracle" / "_ref" / "ref_run"
    if not exe.exists():
        return None, None
    if ny != nx:  # the reference is square-only (config.hpp:50): sample the square per-GPU grid
        nx = ny = min(nx, ny)
    cols = nx // BLOCK
    if engine == "swept":
        ranks = max(r for r in range(1, threads + 1) if cols % r == 0)
        cfg = {"problem": "heat", "nx": nx, "block": BLOCK, "steps": steps, "ranks": ranks, "engine": "swept"}
    else:
        cfg = {"problem": "heat", "nx": nx, "block": BLOCK, "steps": steps, "ranks": 1, "engine": "standard",
               "pool_a": {"workers": threads, "cost": 1.0}}
    out = subprocess.run([str(exe), json.dumps(cfg), "1"], capture_output=True, text=True, timeout=900)
    try:
        rec = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:  # noqa: BLE001
        return None, None
    if "error" in rec:
        return None, rec
    return rec["cell_updates_per_s"], dict(rec, cfg=cfg)


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    px, py = GRIDS.get(args.gpus, (args.gpus, 1))
    nx, ny = PER_GPU * px, PER_GPU * py
    threads = os.cpu_count() or 1
    exe = ROOT / "oracle" / "_ref" / "ref_run"
    if not exe.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_run was not built on this host"}))
        return 0
    sample_steps = args.ref_sample_steps
    rates = []
    rec = None
    for i in range(args.warmup + args.steps):
        r, rec = cpu_reference_sample(nx, ny, sample_steps, "swept", threads)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": f"reference run failed: {rec}"}))
            return 0
        if i >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)
    sample = (f"reference swept engine, heat {rec['cfg']['nx']}^2 b{BLOCK}, {sample_steps} requested steps "
              f"({rec['actual_steps']} actual), {rec['cfg']['ranks']} ranks x 1 thread, median of {len(rates)}")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "cell-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["median_wall_seconds"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.gpus, nx, ny),
                       timed_sample={"nx": rec["cfg"]["nx"], "requested_steps": sample_steps,
                                     "actual_steps": rec["actual_steps"],
                                     "note": "each step times this bounded sample of the workload (the rate, "
                                             "cell-updates/s, is the compared quantity); the full 10k-step "
                                             "solve would take ~1 h of CPU per step"}),
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": rec["cfg"]["ranks"],
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(n, nx, ny):
    px, py = GRIDS.get(n, (n, 1))
    return {"workload": f"heat2d-swept-weak-{PER_GPU}sq-per-gpu-b{BLOCK}-{REQ_STEPS}steps", "problem": "heat",
            "nx": nx, "ny": ny, "block": BLOCK, "requested_steps": REQ_STEPS, "partition": f"{px}x{py}",
            "engine": "swept (standard timed alongside)", "l2": "inputs larger than L2 (537 MB per plane per GPU)"}


def main():
    global PER_GPU, REQ_STEPS, BLOCK
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--req-steps", type=int, default=REQ_STEPS)
    ap.add_argument("--per-gpu", type=int, default=PER_GPU)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-extra", action="store_true", help="skip the standard / Euler side measurements")
    ap.add_argument("--ref-sample-steps", type=int, default=21)
    ap.add_argument("--hash", action="store_true",
                    help="add the FNV-1a-64 of the assembled global final field (small grids: gathers to rank 0)")
    ap.add_argument("--block", type=int, default=BLOCK,
                    help="swept block size (default 16, the reference weak-scaling block; 32 is the fastest here)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    BLOCK = args.block

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import numpy as np
    import torch

    import paper_2105_10332_b200 as sg

    PER_GPU, REQ_STEPS = args.per_gpu, args.req_steps
    dist = None
    if world > 1:
        # one process per GPU: rank r owns partition r of the px x py grid;
        # torch.distributed (NCCL) is plumbing only (IPC handle exchange,
        # barriers, the max-over-ranks timing reduction)
        import torch.distributed as dist
        # SG_BENCH_SAME_DEVICE=1 + SG_BENCH_BACKEND=gloo: exercise the N-rank
        # path on a single GPU (all ranks share device 0; NCCL refuses that)
        same = os.environ.get("SG_BENCH_SAME_DEVICE") == "1"
        torch.cuda.set_device(0 if same else env_int("LOCAL_RANK", 0))
        dist.init_process_group(os.environ.get("SG_BENCH_BACKEND", "nccl"), init_method="env://")
    n = world if world > 1 else args.gpus
    px, py = GRIDS.get(n, (n, 1))
    nx, ny = PER_GPU * px, PER_GPU * py
    pw, ph = nx // px, ny // py
    pi, pj = rank % px, rank // px
    base = dict(problem="heat", nx=nx, ny=ny, block=BLOCK, steps=REQ_STEPS, ranks=px * py, px=px, py=py)

    def make(engine, profile=False, **over):
        cfg = sg.SolverConfig(engine=engine, **dict(base, **over))
        if dist is not None:
            return sg.DistSolver(cfg, rank=rank, world=world, profile=profile)
        return sg.Solver(cfg, profile=profile)

    def sync():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(engine, profile, **over):
        s = make(engine, profile, **over)
        for _ in range(args.warmup):
            s.reset()
            s.solve()
        sync()
        dev, kst = [], []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.reset()
            dev.append(s.solve())
            kst.append(s.kernel_stats())
        sync()
        wall = time.perf_counter() - t0
        return s, max_over_ranks(sum(dev)), kst, max_over_ranks(wall)

    clocks = Clocks()
    if rank == 0:
        clocks.start()
    # headline: the production path (CUDA-graph replay, XBridge side stream),
    # no per-launch events
    sw, sw_dev, _, sw_wall = timed("swept", False)
    ck = clocks.stop() if rank == 0 else None
    rec = sw.fetch().record
    updates = rec.cell_updates
    value = updates * args.steps / sw_dev
    # dominant-kernel timing in a separate pass: CUDA events around every
    # Octahedron launch (serialised launches, no graph)
    sp = make("swept", True)
    for _ in range(args.warmup):
        sp.reset()
        sp.solve()
    sync()
    sw_k = []
    prof_dev = 0.0
    for _ in range(max(1, min(args.steps, 2))):
        sp.reset()
        prof_dev += sp.solve()
        sw_k.append(sp.kernel_stats())
    prof_steps = len(sw_k)
    sync()  # no rank frees buffers a peer may still be pushing into
    sp.close()

    # ---- e2e: pinned host piece in -> solve -> host piece out, every step --
    nv = 1
    full = np.empty((nv, ny, nx))
    sw.initial(full)  # the reference initial condition (make_setup, engine.cpp:31-42)
    if dist is not None:
        piece = full[:, pj * ph:(pj + 1) * ph, pi * pw:(pi + 1) * pw]
    else:
        piece = full
    host_in = torch.from_numpy(np.ascontiguousarray(piece)).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    del full
    sw.upload(host_in)
    sw.reset()
    sw.solve()
    sw.download(host_out)
    ref_out = host_out.numpy().copy()
    sync()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sw.upload(host_in)
        sw.reset()
        sw.solve()
        sw.download(host_out)
    sync()
    e2e_wall = max_over_ranks(time.perf_counter() - t0)
    e2e_value = updates * args.steps / e2e_wall
    assert np.array_equal(host_out.numpy(), ref_out), "e2e output differs between repeats"
    launches = rec.kernel_launches * args.steps
    field_hash = None
    if args.hash:  # assemble the global field from the ranks' e2e outputs
        pieces = [None] * world if (dist is not None and rank == 0) else None
        if dist is not None:
            dist.gather_object((pi, pj, ref_out), pieces, dst=0)
        else:
            pieces = [(0, 0, ref_out)]
        if rank == 0:
            glob = np.empty((nv, ny, nx))
            for qi, qj, pc in pieces:
                glob[:, qj * ph:(qj + 1) * ph, qi * pw:(qi + 1) * pw] = pc
            field_hash = sg.fnv1a64(glob)

    # ---- roofline of the dominant kernel (Octahedron phase) ----------------
    peaks, peak_kind = measured_peaks()
    k = sw_k[-1]
    per_launch_bytes = k["alg_bytes"] / max(1, k["launches"])
    per_launch_s = k["seconds"] / max(1, k["launches"])
    achieved = per_launch_bytes / per_launch_s / 1e9
    tag = workload_config(n, nx, ny)["workload"]
    nt = ncu_traffic(tag)
    roof = {"kernel": f"swept_heat_col_kernel<{BLOCK}, Octahedron> (register-tile Octahedron launches)", "bound": "hbm",
            "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": nt[0] if nt else None,
            "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else
            "fallback 6650 GB/s (B200_PROFILING.md)",
            "alg_bytes_per_launch": per_launch_bytes, "mean_launch_ms": per_launch_s * 1e3,
            "launches_per_step": k["launches"], "share_of_step": round(k["seconds"] * prof_steps / prof_dev, 4),
            "timing": "separate profiling pass (events around each Octahedron launch, no graph); the headline "
                      "value is timed on the graph path without events",
            "traffic_source": nt[1] if nt else None}
    sw.close()
    # whole-solve roofline of SURVEY.md §8d: updates/s over
    # min(HBM / algorithmic bytes per update, FP64 non-FMA peak / flops per update)
    fp64 = sg.measure_fp64_peak() if rank == 0 else -1.0
    bpu = {8: 15.50, 12: 10.44, 16: 7.875, 24: 5.28, 32: 3.97}.get(BLOCK)
    solve_roof = None
    if bpu and fp64 > 0:
        ceil_hbm = peaks["hbm_gbs"] * 1e9 / bpu
        ceil_fp64 = fp64 / 9.0
        ceil = min(ceil_hbm, ceil_fp64)
        solve_roof = {"achieved": value / n, "unit": "cell-updates/s per GPU", "ceiling": ceil,
                      "frac": round(value / n / ceil, 4),
                      "bound": "hbm" if ceil_hbm <= ceil_fp64 else "fp64",
                      "alg_bytes_per_update": bpu, "flops_per_update": 9,
                      "fp64_nonfma_peak_flops": fp64, "fp64_peak_source": "measured (sg_measure_fp64_peak: DADD+DMUL "
                      "chains, 8 per thread, 8 CTAs x 256 threads per SM)"}

    extra = {}
    if not args.no_extra:
        # standard decomposition on the same workload (swept/standard speedup)
        st, st_dev, _, _ = timed("standard", False, steps=rec.actual_steps)
        st_rec = st.fetch().record
        st_value = st_rec.cell_updates * args.steps / st_dev
        st.close()
        extra["standard"] = {"value": st_value, "unit": "cell-updates/s", "ms_per_step": 1e3 * st_dev / args.steps}
        extra["swept_over_standard"] = value / st_value
        # the block-size axis (BASELINE configs[2]): b32 halves the swept bytes
        # per update on the same grid; the standard engine does not depend on b
        sb, sb_dev, sb_k, _ = timed("swept", False, block=32)
        sb_rec = sb.fetch().record
        sb.close()
        b32v = sb_rec.cell_updates * args.steps / sb_dev
        extra["swept_b32"] = {"value": b32v, "unit": "cell-updates/s",
                              "solve_roofline_frac": round(b32v / n / min(peaks["hbm_gbs"] * 1e9 / 3.97, fp64 / 9.0), 4)
                              if fp64 > 0 else None,
                              "actual_steps": sb_rec.actual_steps, "ms_per_step": 1e3 * sb_dev / args.steps,
                              "swept_over_standard": (sb_rec.cell_updates * args.steps / sb_dev) /
                              (st_rec.cell_updates / st_rec.actual_steps * sb_rec.actual_steps * args.steps / st_dev)}
        if n == 1:
            # configs[1]: Euler 960^2 b16 swept vs standard (one GPU)
            eu = {}
            for eng in ("swept", "standard"):
                cfg = sg.SolverConfig(problem="euler", nx=960, block=16, engine=eng,
                                      steps=500 if eng == "swept" else eu["swept"]["actual_steps"])
                s = sg.Solver(cfg)
                for _ in range(3):
                    s.reset()
                    s.solve()
                ts = []
                for _ in range(args.steps):
                    s.reset()
                    ts.append(s.solve())
                r = s.fetch()
                eu[eng] = {"value": r.record.cell_updates * args.steps / sum(ts),
                           "actual_steps": r.record.actual_steps, "ms_per_step": 1e3 * sum(ts) / args.steps}
                if eng == "standard":
                    eu["bitwise_equal"] = bool(np.array_equal(r.final_field.data, eu.pop("_field")))
                else:
                    eu["_field"] = r.final_field.data
                s.close()
            eu["swept_over_standard"] = eu["swept"]["value"] / eu["standard"]["value"]
            extra["euler_960_b16"] = eu
            # the same grid at b32 (the largest Euler block whose phase fits on chip)
            s = sg.Solver(sg.SolverConfig(problem="euler", nx=960, block=32, engine="swept", steps=500))
            for _ in range(3):
                s.reset()
                s.solve()
            ts = []
            for _ in range(args.steps):
                s.reset()
                ts.append(s.solve())
            r32 = s.fetch().record
            s.close()
            extra["euler_960_b32_swept"] = {"value": r32.cell_updates * args.steps / sum(ts),
                                            "actual_steps": r32.actual_steps,
                                            "ms_per_step": 1e3 * sum(ts) / args.steps}
            # the paper's own array sizes, b16, 500 requested steps:
            # the launch/latency-bound regime the swept rule targets
            ps = {}
            for prob in ("heat", "euler"):
                for nxp in (320, 640, 960):
                    rates = {}
                    steps_p = 500
                    for eng in ("swept", "standard"):
                        s = sg.Solver(sg.SolverConfig(problem=prob, nx=nxp, block=16, engine=eng, steps=steps_p))
                        for _ in range(3):
                            s.reset()
                            s.solve()
                        ts = []
                        for _ in range(args.steps):
                            s.reset()
                            ts.append(s.solve())
                        r = s.fetch().record
                        s.close()
                        rates[eng] = r.cell_updates / min(ts)
                        steps_p = r.actual_steps
                    ps[f"{prob}_{nxp}"] = {"swept": rates["swept"], "standard": rates["standard"],
                                           "swept_over_standard": rates["swept"] / rates["standard"]}
            extra["paper_sizes_b16"] = ps

    # ---- CPU baseline: the reference on this host, bounded sample ----------
    cpu = None
    if not args.no_cpu and n == 1 and rank == 0:
        threads = os.cpu_count() or 1
        v, crec = cpu_reference_sample(nx, ny, args.ref_sample_steps, "swept", threads)
        if v is not None:
            cpu = {"value": v, "unit": "cell-updates/s", "cores": crec["cfg"]["ranks"], "kind": "reference",
                   "sample": f"reference swept engine (oracle/_ref), heat {crec['cfg']['nx']}^2 b{BLOCK}, "
                             f"{args.ref_sample_steps} requested steps ({crec['actual_steps']} actual), "
                             f"{crec['cfg']['ranks']} ranks x 1 thread, wall {crec['median_wall_seconds']:.2f} s"}
            vs, _ = cpu_reference_sample(nx, ny, args.ref_sample_steps, "standard", threads)
            if vs is not None:
                cpu["standard_value"] = vs
                cpu["standard_sample"] = f"reference standard engine, 1 rank x {threads} OpenMP threads"
            # parity at the bench grid: the GPU swept solve of the very sample
            # the reference just ran must reproduce its final field byte for byte
            with sg.Solver(sg.SolverConfig(problem="heat", nx=crec["cfg"]["nx"], block=BLOCK,
                                           steps=args.ref_sample_steps)) as ps:
                ps.reset()
                ps.solve()
                got = sg.fnv1a64(ps.fetch().final_field.data)
            cpu["reference_parity"] = {"sample": f"heat {crec['cfg']['nx']}^2 b{BLOCK}, "
                                                 f"{args.ref_sample_steps} requested steps",
                                       "gpu_fnv1a64": got, "reference_fnv1a64": crec.get("fnv1a64"),
                                       "equal": got == crec.get("fnv1a64")}
            assert got == crec.get("fnv1a64"), f"GPU final field differs from the reference: {cpu['reference_parity']}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sw_dev / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(n, nx, ny),
            "e2e": {"value": e2e_value, "unit": "cell-updates/s", "h2d_bytes_per_step": nv * nx * ny * 8,
                    "d2h_bytes_per_step": nv * nx * ny * 8},
            "gpu_launches": launches,
            "roofline": roof, "solve_roofline": solve_roof, "cpu_baseline": cpu, "clocks": ck,
            "actual_steps": rec.actual_steps, "cell_updates_per_step": updates,
            "final_fnv1a64": field_hash,
            "wall_ms_per_step": 1e3 * sw_wall / args.steps,
            "multi_gpu": "one process per GPU; partition-edge records pushed by P2P stores from the phase "
                         "kernels, launches ordered by device-side epoch flags" if n > 1 else None,
        }
        line.update(extra)
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
