"""Dynamic SASS opcode mix (warp-level instructions executed) of one launch:
    python profiles/ncu_opmix.py rep.ncu-rep [launch_index]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, ops, stall = None, collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    src = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip())
    op = src.split()[0] if src else "?"
    try:
        ops[op] += int(d["Instructions Executed"] or 0)
        stall[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    except (KeyError, ValueError):
        pass
tot = sum(ops.values()) or 1
ts = sum(stall.values()) or 1
print(f"warp instructions {tot}")
for op, n in ops.most_common(40):
    print(f"{op:28s} {n:12d} {100 * n / tot:5.1f}%  stall {100 * stall[op] / ts:5.1f}%")
