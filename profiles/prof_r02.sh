#!/bin/bash
# Round-2 profile set (one B200, under gpurun, from the repo root):
#   bash profiles/prof_r02.sh
# Writes small JSON/text summaries into gpurun_out/ (reports are deleted:
# they are tens of MB each).
#  1. launch list of a short bench run (per-launch device time; ncu
#     serialises launches cold-cache: compare shares, not absolutes)
#  2. ncu --set full: one steady swept cycle (Oct, YB, XB) at b16 and b32,
#     one standard heat step (8192^2), the Euler standard step and an Euler
#     Octahedron (960^2 b16 and b32)
set -u
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02.csv \
    python bench.py --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra > $O/launches_bench_r02.log 2>&1
python profiles/launch_summary.py $O/launches_r02.csv > $O/launches_r02.txt 2>&1
for B in 16 32; do
  ncu --set full --clock-control none --import-source on -k regex:swept_heat_col -s 9 -c 3 \
      -o $O/cyc$B python bench.py --block $B --req-steps 140 --steps 1 --warmup 3 --no-cpu --no-extra \
      > $O/cyc$B.log 2>&1
  python profiles/ncu_json.py $O/cyc$B.ncu-rep > $O/r02_cycle_b$B.json
  python profiles/ncu_opmix.py $O/cyc$B.ncu-rep 0 > $O/r02_cycle_b${B}_oct_opmix.txt 2>&1
  rm -f $O/cyc$B.ncu-rep
done
cat > /tmp/std.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2105_10332_b200 as sg
s = sg.Solver(sg.SolverConfig(problem="heat", nx=8192, block=16, steps=6, engine="standard"))
s.reset(); s.solve()
PY
SG_NO_GRAPH=1 ncu --set full --clock-control none -k regex:std_heat -s 3 -c 1 -o $O/stdheat python /tmp/std.py > $O/stdheat.log 2>&1
python profiles/ncu_json.py $O/stdheat.ncu-rep > $O/r02_std_heat_8192.json; rm -f $O/stdheat.ncu-rep
cat > /tmp/eu.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2105_10332_b200 as sg
for eng, b in (("standard", 16), ("swept", 16), ("swept", 32)):
    s = sg.Solver(sg.SolverConfig(problem="euler", nx=960, block=b, steps=20, engine=eng))
    s.reset(); s.solve()
PY
SG_NO_GRAPH=1 ncu --set full --clock-control none -k regex:std_euler -s 4 -c 1 -o $O/eustd python /tmp/eu.py > $O/eustd.log 2>&1
python profiles/ncu_json.py $O/eustd.ncu-rep > $O/r02_std_euler_960.json; rm -f $O/eustd.ncu-rep
SG_NO_GRAPH=1 ncu --set full --clock-control none -k regex:swept_euler -s 6 -c 1 -o $O/euoct python /tmp/eu.py > $O/euoct.log 2>&1
python profiles/ncu_json.py $O/euoct.ncu-rep > $O/r02_swept_euler_oct_960_b16.json; rm -f $O/euoct.ncu-rep
ls -la $O
