"""Per-launch JSON summary of an ncu --set full report (what profiles/*.json
hold): duration, DRAM bytes, instructions, IPC, registers, occupancy, pipe
and L1 utilisation, warp-stall reasons per issued instruction.
    python profiles/ncu_json.py rep.ncu-rep > summary.json"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
names, units = rows[0], rows[1]
KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "issued_warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "ipc": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "l1tex_data_pipe_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "block_size": ("launch__block_size", 1.0),
}
# bytes -> bytes; times -> milliseconds
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0}
out = []
for r in rows[2:]:
    d = dict(zip(names, r))
    u = dict(zip(names, units))
    e = {"kernel": d.get("Kernel Name", "")[:160]}
    for k, (m, scale) in KEYS.items():
        if m not in d or d[m] in ("", "n/a"):
            continue
        v = float(d[m].replace(",", ""))
        if k == "duration_ms":
            v *= UNIT[u[m]]
        elif k.startswith("dram_") and k.endswith("bytes"):
            v *= UNIT.get(u[m], 1.0)
        e[k] = v
    e["stalls_per_issue"] = {
        m.split("stalled_")[1].replace("_per_issue_active.ratio", ""): round(float(d[m]), 3)
        for m in names
        if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio")
        and d[m] not in ("", "0", "0.000000") and float(d[m]) >= 0.05}
    if "dram_read_bytes" in e and "dram_write_bytes" in e:
        e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
    out.append(e)
print(json.dumps(out, indent=1))
