#!/bin/bash
# Euler ncu captures (round 2b): the standard column-marching step and the
# swept Octahedron at 960^2 b16 (configs[1]); JSON summaries in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
cat > /tmp/eu.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2105_10332_b200 as sg
for eng, b in (("standard", 16), ("swept", 16)):
    s = sg.Solver(sg.SolverConfig(problem="euler", nx=960, block=b, steps=20, engine=eng))
    s.reset(); s.solve()
PY
SG_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:std_euler -s 4 -c 1 -o $O/eustd python /tmp/eu.py > $O/eustd.log 2>&1
python profiles/ncu_json.py $O/eustd.ncu-rep > $O/r02b_std_euler_960.json
SG_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:swept_euler -s 6 -c 1 -o $O/euoct python /tmp/eu.py > $O/euoct.log 2>&1
python profiles/ncu_json.py $O/euoct.ncu-rep > $O/r02b_swept_euler_oct_960_b16.json
ls -la $O
