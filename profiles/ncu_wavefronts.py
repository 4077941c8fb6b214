"""L1 data-pipe (LSU) wavefront budget and opcode mix per launch of an ncu
report, per warp -- the limiter of the register-tile heat kernels:

    python profiles/ncu_wavefronts.py rep.ncu-rep [launches] > summary.json

For each launch: duration, warps, instructions per warp, LSU wavefronts per
warp split into shared-memory (LDS + LDGSTS shared side + SHFL: the shuffles
go through the same data pipe), global loads (table LDGs + LDGSTS global
side) and global stores, plus the dynamic opcode mix (per warp).
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def ncu_csv(rep, page, idx, extra=()):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv", "--launch-skip", str(idx), "--launch-count", "1", *extra]
    return list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def one(rep, idx):
    raw = ncu_csv(rep, "raw", idx)
    if len(raw) < 3:
        return None
    d = dict(zip(raw[0], raw[2]))
    units = dict(zip(raw[0], raw[1]))
    tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
        units.get("gpu__time_duration.sum", ""), 1.0)
    bscale = lambda k: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get(k, "byte"), 1.0)
    grid = num(d.get("launch__grid_size", "nan"))
    block = num(d.get("launch__block_size", "nan"))
    warps = grid * block / 32
    nsm = num(d.get("device__attribute_multiprocessor_count", "148"))
    pw = lambda k: round(num(d.get(k, "nan")) / warps, 1)
    out = {
        "kernel": d.get("Kernel Name", "?"),
        "duration_ms": round(num(d.get("gpu__time_duration.sum", "nan")) * tscale, 4),
        "warps": warps,
        "registers": num(d.get("launch__registers_per_thread", "nan")),
        "instructions_per_warp": pw("smsp__inst_executed.sum"),
        "lsu_wavefronts_pct": round(num(d.get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "nan")), 1),
        "lsu_wavefronts_per_warp": round(num(d.get("l1tex__data_pipe_lsu_wavefronts.avg", "nan")) * nsm / warps, 1),
        "shared_wavefronts_per_warp": pw("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "lds_wavefronts_per_warp": pw("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
        "global_ld_wavefronts_per_warp": pw("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum"),
        "global_st_wavefronts_per_warp": pw("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum"),
        "ldgsts_bank_conflicts_per_warp": pw("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum"),
        "fp64_pipe_pct": round(num(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "nan")), 1),
        "dram_bytes": num(d.get("dram__bytes_read.sum", "nan")) * bscale("dram__bytes_read.sum")
        + num(d.get("dram__bytes_write.sum", "nan")) * bscale("dram__bytes_write.sum"),
    }
    src = ncu_csv(rep, "source", idx, ("--print-source", "sass"))
    hdr, ops, seen = None, collections.Counter(), set()
    for r in src:
        if r and r[0] == "Address":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        e = dict(zip(hdr, r))
        if e["Address"] in seen:  # the source page lists some sections twice
            continue
        seen.add(e["Address"])
        s = re.sub(r"^@!?U?P\w+\s+", "", e["Source"].strip())
        ops[s.split()[0] if s else "?"] += num(e["Instructions Executed"] or 0)
    out["opcodes_per_warp"] = {k: round(v / warps, 1) for k, v in ops.most_common(16)}
    return out


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res = [r for r in (one(rep, i) for i in range(n)) if r]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
