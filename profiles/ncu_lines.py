"""Per-CUDA-source-line warp-stall samples and executed instructions of one
launch of an ncu report (needs -lineinfo and --import-source on):
    python profiles/ncu_lines.py rep.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
fname, hdr, out = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            ie = int(d.get("Instructions Executed", "0") or 0)
            ss = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if ie or ss:
            out.append((ss, ie, fname, r[0], r[1].strip()[:90]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {ts} instructions {ti}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{100 * o[0] / ts:5.1f}% stall {100 * o[1] / ti:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
