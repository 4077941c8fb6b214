"""Per-basic-block instruction / stall breakdown of an ncu source page (SASS).
    python profiles/sass_blocks.py rep.ncu-rep <instances per launch>"""
import csv
import io
import subprocess
import sys

rep, N = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
iW, iWI = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
tot = sum(float(r[iE] or 0) for r in data)
totS = sum(float(r[iS] or 0) for r in data)
print(f"per-unit instructions {tot / N:.0f}; smem wavefronts {sum(float(r[iW] or 0) for r in data) / N:.0f} "
      f"(ideal {sum(float(r[iWI] or 0) for r in data) / N:.0f})")
blocks, cur = [], None
for r in data:
    e = float(r[iE] or 0)
    if cur and cur[1] == e:
        cur[2] += 1
        cur[3] += float(r[iS] or 0)
    else:
        cur = [r[0][-5:], e, 1, float(r[iS] or 0), r[iSrc][:56]]
        blocks.append(cur)
for b in blocks:
    if b[1] * b[2] / N > 12 or b[3] / totS > 0.02:
        print(f"{b[0]} x{b[1] / N:6.1f} len {b[2]:3d} -> {b[1] * b[2] / N:7.1f}/unit stall {b[3] / totS * 100:5.1f}% {b[4]}")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
T = {c: sum(float(r[hdr.index(c)] or 0) for r in data) for c in cols}
tt = sum(T.values())
print(", ".join(f"{c[6:]}:{v / tt * 100:.0f}%" for c, v in sorted(T.items(), key=lambda x: -x[1])[:8]))
