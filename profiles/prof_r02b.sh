#!/bin/bash
# Round-2b profile set (after the steady-state column-kernel rework), one B200,
# under gpurun, from the repo root:   bash profiles/prof_r02b.sh
# Writes JSON/text summaries into gpurun_out/ (the reports stay out of git).
#  1. launch list of a short bench run (cold-cache, serialised: shares only)
#  2. ncu --set full of one steady swept cycle (Oct, YB, XB) at b16 and b32:
#     ncu_json.py summary + ncu_wavefronts.py LSU budget / opcode mix
#  3. the bench's dominant-kernel traffic record (r02b_oct_col_b16.json)
set -u
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02b.csv \
    python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra > $O/launches_bench_r02b.log 2>&1
python profiles/launch_summary.py $O/launches_r02b.csv > $O/launches_r02b.txt 2>&1
for B in 16 32; do
  ncu --set full --clock-control none --import-source on -k regex:swept_heat_col -s 9 -c 4 \
      -o $O/cyc$B python bench.py --block $B --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
      > $O/cyc$B.log 2>&1
  python profiles/ncu_json.py $O/cyc$B.ncu-rep > $O/r02b_cycle_b$B.json
  python profiles/ncu_wavefronts.py $O/cyc$B.ncu-rep 4 > $O/r02b_cycle_b${B}_wavefronts.json
done
python - <<'PY'
import json
c = json.load(open("gpurun_out/r02b_cycle_b16.json"))[0]
alg = 262144 * (476 + 392) * 8
rec = {"workload": "heat2d-swept-weak-8192sq-per-gpu-b16-10000steps",
       "kernel": c["kernel"], "capture": "ncu --set full --clock-control none, launches 9..11 of bench.py --req-steps 140 (profiles/prof_r02b.sh)",
       "duration_ms": c["duration_ms"], "dram_bytes_per_launch": c["dram_read_bytes"] + c["dram_write_bytes"],
       "dram_read_bytes": c["dram_read_bytes"], "dram_write_bytes": c["dram_write_bytes"],
       "alg_bytes_per_launch": alg, "issued_warp_instructions": c["issued_warp_instructions"], "ipc": c["ipc"],
       "registers": c["registers"], "achieved_occupancy_pct": c["achieved_occupancy_pct"],
       "l1tex_data_pipe_wavefronts_pct": c["l1tex_data_pipe_wavefronts_pct"], "fp64_pipe_pct": c["fp64_pipe_pct"],
       "stalls_per_issue": c["stalls_per_issue"]}
json.dump(rec, open("gpurun_out/r02b_oct_col_b16.json", "w"), indent=1)
PY
rm -f $O/cyc16.ncu-rep $O/cyc32.ncu-rep
ls -la $O
