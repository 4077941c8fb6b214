#!/bin/bash
# ncu --set full of the Euler standard step and an Euler Octahedron launch (960^2 b16)
TAG=${1:-r01}
cat > /tmp/eu.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2105_10332_b200 as sg
for eng in ("standard", "swept"):
    s = sg.Solver(sg.SolverConfig(problem="euler", nx=960, block=16, steps=20, engine=eng))
    s.reset(); s.solve()
PY
ncu --set full --clock-control none --import-source on -k regex:std_euler -s 4 -c 1 -o gpurun_out/prof_eustd_$TAG python /tmp/eu.py > gpurun_out/prof_eustd_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:swept_euler -s 6 -c 1 -o gpurun_out/prof_euoct_$TAG python /tmp/eu.py > gpurun_out/prof_euoct_$TAG.log 2>&1
