"""Every code path of the register-tile heat kernels gives the same field.

The launcher picks, per launch, the steady-state kernel with the dense
slot-indexed gather (FLAGS 3), with the table gather (FLAGS 1), the dense
gather through registers (FLAGS 7), the Octahedron split into two launches
(b32, FLAGS bits 4-5; b24 measured no gain) or the general
kernel with the output / snapshot stash (FLAGS 0), and sizes the
shared-memory carveout (colkernel.cuh launch_heat_col_t).  The switches are
read once per process, so each variant runs in its own process; all must
reproduce the default solve bit for bit (the default itself is pinned to the
reference in test_gpu_fullsize.py / test_gpu_parity.py).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_2105_10332_b200 as sg
nx, b, steps = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
r = sg.run(sg.SolverConfig(problem="heat", nx=nx, block=b, steps=steps))
print("RESULT " + json.dumps({"fnv": sg.fnv1a64(r.final_field.data), "steps": r.record.actual_steps}))
"""

VARIANTS = {
    "default": {},
    "general": {"SG_FAST_KINDS": "0"},
    "table": {"SG_DENSE_KINDS": "0"},
    "regs": {"SG_REG_KINDS": "31"},
    "carve_default": {"SG_CARVE_OCT": "-1", "SG_CARVE_BR": "-1"},
    "one_octahedron_launch": {"SG_NO_OCT_SPLIT": "1"},
}


def _run(env_extra, nx, b, steps):
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(nx), str(b), str(steps)], env=env,
                       capture_output=True, text=True, timeout=600)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert line, p.stderr[-2000:]
    return json.loads(line[0][7:])


@pytest.mark.parametrize("nx,b,steps", [(512, 16, 300), (384, 12, 200), (512, 32, 200), (480, 24, 150)])
def test_kernel_variants_bitwise_equal(nx, b, steps):
    ref = _run({}, nx, b, steps)
    for name, env in VARIANTS.items():
        if name == "default":
            continue
        got = _run(env, nx, b, steps)
        assert got == ref, f"variant {name} ({env}) differs: {got} vs {ref}"
