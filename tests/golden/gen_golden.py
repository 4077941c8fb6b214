"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libsweptgrid_ref.so, built
by `make -C oracle ref` from /root/reference/proj/src with the reference's own
flags) through its public run() (engine.hpp:61) and records, per config, the
RunRecord fields that define the schedule and an FNV-1a-64 hash of the final
field bytes.  Also stores known answers of the physics primitives
(test_physics.cpp:86-119) and of the schedule arithmetic (test_geometry.cpp).

Only runs where /root/reference is present (this container); the committed
JSON travels to the GPU box.
    python tests/golden/gen_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_bind import Reference, Restated  # noqa: E402

fnv1a64 = Restated().fnv1a

RUNS = [
    # SURVEY.md §8c fingerprints + the acceptance / engine-test configs
    {"problem": "heat", "nx": 384, "block": 16, "steps": 500, "ranks": 8},
    {"problem": "heat", "nx": 96, "block": 16, "steps": 50, "ranks": 1},
    {"problem": "heat", "nx": 384, "block": 32, "steps": 500, "ranks": 6},
    {"problem": "heat", "nx": 384, "block": 8, "steps": 500, "ranks": 8},
    {"problem": "heat", "nx": 96, "block": 8, "steps": 50, "ranks": 4},
    {"problem": "heat", "nx": 192, "block": 16, "steps": 50, "ranks": 4},
    {"problem": "heat", "nx": 32, "block": 16, "steps": 10, "ranks": 1},
    {"problem": "heat", "nx": 64, "block": 8, "steps": 20, "ranks": 2},
    {"problem": "euler", "nx": 96, "block": 16, "steps": 50, "ranks": 1},
    {"problem": "euler", "nx": 192, "block": 8, "steps": 50, "ranks": 4},
    {"problem": "euler", "nx": 96, "block": 8, "steps": 50, "ranks": 2},
    {"problem": "euler", "nx": 32, "block": 16, "steps": 5, "ranks": 1},
    {"problem": "euler", "nx": 960, "block": 16, "steps": 10, "ranks": 6},
]
KEYS = ("actual_steps", "total_levels", "octahedra", "communicates", "cell_updates", "final_level", "dt")


def main():
    ref = Reference()
    out = {"generator": "tests/golden/gen_golden.py", "runs": [], "standard": [], "setup": []}
    for cfg in RUNS:
        field, rec = ref.run(cfg)
        out["runs"].append({"cfg": cfg, "record": {k: rec[k] for k in KEYS}, "fnv1a64": fnv1a64(field),
                            "max_abs": float(np.abs(field).max())})
        print(cfg, out["runs"][-1]["fnv1a64"], flush=True)
        if cfg["nx"] <= 192:
            sc = dict(cfg, engine="standard", steps=rec["actual_steps"])
            f2, r2 = ref.run(sc)
            out["standard"].append({"cfg": sc, "fnv1a64": fnv1a64(f2), "record": {k: r2[k] for k in KEYS}})
    for cfg in ({"problem": "heat", "nx": 64}, {"problem": "euler", "nx": 64}, {"problem": "euler", "nx": 960}):
        init, dt, dx, dy = ref.setup(cfg)
        out["setup"].append({"cfg": cfg, "dt": dt, "dx": dx, "dy": dy, "fnv1a64": fnv1a64(init)})
    sched = []
    for b, n, S in ((8, 1, 1), (12, 1, 1), (16, 1, 1), (24, 1, 1), (32, 1, 1), (8, 2, 2), (12, 2, 2), (16, 2, 2),
                    (24, 2, 2), (32, 2, 2)):
        for steps in (1, 5, 10, 50, 100, 500, 10000):
            try:
                rows, meta = ref.schedule(steps, b, n, S)
            except Exception as e:  # noqa: BLE001
                sched.append({"b": b, "n": n, "S": S, "steps": steps, "error": str(e)})
                continue
            sched.append({"b": b, "n": n, "S": S, "steps": steps, **meta, "entries": len(rows)})
    out["schedule"] = sched
    # SWPT2D snapshot streams written by the reference (snapshot.cpp:57-84)
    import hashlib
    import tempfile
    snaps = []
    for cfg in ({"problem": "heat", "nx": 32, "block": 8, "steps": 10},                 # test_engine.cpp:234-267
                {"problem": "heat", "nx": 32, "block": 8, "steps": 6, "engine": "standard", "ranks": 2},
                {"problem": "euler", "nx": 32, "block": 16, "steps": 5},                # odd flat level
                {"problem": "euler", "nx": 48, "block": 8, "steps": 4, "snapshot_every": 3},
                {"problem": "heat", "nx": 48, "block": 16, "steps": 30, "snapshot_every": 4}):
        with tempfile.TemporaryDirectory() as td:
            path = f"{td}/snap.bin"
            field, rec = ref.run(dict(cfg, snapshot=path))
            data = open(path, "rb").read()
        snaps.append({"cfg": cfg, "sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
                      "frames": rec["snapshot_frames"], "total_levels": rec["total_levels"]})
    out["snapshots"] = snaps
    (HERE / "golden.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
