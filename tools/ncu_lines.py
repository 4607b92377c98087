"""Per-CUDA-source-line warp-stall samples from an ncu report:
   python tools/ncu_lines.py gpurun_out/x.ncu-rep [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"]
if len(sys.argv) > 3:
    cmd += ["-k", f"regex:{sys.argv[3]}"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
col, fname, out = None, "", []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        col = next((i for i, h in enumerate(r) if h.startswith("Warp Stall Sampling (All")), None)
        continue
    if col is None or len(r) <= col:
        continue
    try:
        s = int(r[col])
    except ValueError:
        continue
    if s:
        out.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
print("total samples", tot)
for s, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {loc:18s} {src}")
