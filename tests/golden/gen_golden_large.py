"""Generate tests/golden/golden_large.json: reference fingerprints at BASELINE's
full sizes (configs[1]-[4]), from the REFERENCE itself.

Runs oracle/_ref/ref_run -- the unmodified reference library built from
/root/reference/proj/src with its own flags (oracle/Makefile) -- through its
public run() (proj/src/engine.cpp:493-568) and records the RunRecord schedule
fields plus the FNV-1a-64 hash of the final field bytes.  The sizes are the
ones the GPU bench and block sweep run at; the step counts are the largest
the CPU finishes in about a minute per case.

Only runs where /root/reference is present (this container); the committed
JSON travels to the GPU box, where tests/test_gpu_fullsize.py checks the GPU
engines against it.
    python tests/golden/gen_golden_large.py
"""
import json
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
EXE = ROOT / "oracle" / "_ref" / "ref_run"

RUNS = [
    # configs[4] / the bench's own cpu_baseline sample: heat 8192^2, b16 and b32
    {"problem": "heat", "nx": 8192, "block": 16, "steps": 21, "ranks": 8},
    {"problem": "heat", "nx": 8192, "block": 32, "steps": 45, "ranks": 8},
    # configs[2]: the 4096^2-class block sweep (4128 = 96 * 43 divides every b)
    {"problem": "heat", "nx": 4128, "block": 8, "steps": 100, "ranks": 6},
    {"problem": "heat", "nx": 4128, "block": 12, "steps": 100, "ranks": 8},
    {"problem": "heat", "nx": 4128, "block": 16, "steps": 100, "ranks": 6},
    {"problem": "heat", "nx": 4128, "block": 24, "steps": 100, "ranks": 4},
    {"problem": "heat", "nx": 4128, "block": 32, "steps": 100, "ranks": 3},
    # configs[1]: Euler 960^2 b16 at the GPU timing length
    {"problem": "euler", "nx": 960, "block": 16, "steps": 100, "ranks": 6},
    {"problem": "euler", "nx": 960, "block": 32, "steps": 40, "ranks": 6},
    # configs[3]: Euler 8192^2 b16 (partitioned 2D on the GPU side)
    {"problem": "euler", "nx": 8192, "block": 16, "steps": 6, "ranks": 8},
]
KEYS = ("actual_steps", "total_levels", "octahedra", "communicates", "cell_updates", "final_level", "dt")


def main():
    if not EXE.exists():
        sys.exit(f"{EXE} missing: run `make -C oracle ref`")
    out = {"generator": "tests/golden/gen_golden_large.py", "tool": "oracle/_ref/ref_run (reference run())",
           "runs": []}
    for cfg in RUNS:
        c = dict(cfg, engine="swept")
        p = subprocess.run([str(EXE), json.dumps(c), "1"], capture_output=True, text=True,
                           env=dict(os.environ, OMP_NUM_THREADS="1"))
        if not p.stdout.strip():
            sys.exit(f"{cfg}: ref_run failed: {p.stderr[-500:]}")
        rec = json.loads(p.stdout.strip().splitlines()[-1])
        if "error" in rec:
            sys.exit(f"{cfg}: {rec['error']}")
        out["runs"].append({"cfg": cfg, "record": {k: rec[k] for k in KEYS}, "fnv1a64": rec["fnv1a64"],
                            "ref_wall_seconds": rec["wall_seconds"]})
        print(cfg, rec["fnv1a64"], f"{rec['wall_seconds']:.1f}s", flush=True)
    (HERE / "golden_large.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", HERE / "golden_large.json")


if __name__ == "__main__":
    main()
