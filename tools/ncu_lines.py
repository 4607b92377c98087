"""Per-CUDA-source-line warp-stall samples from an ncu report:
   python tools/ncu_lines.py gpurun_out/x.ncu-rep [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", f"regex:{sys.argv[3]}"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
fname, col, agg = "", None, {}
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        col = next((i for i, h in enumerate(r) if h.startswith("Warp Stall Sampling (All")), None)
        continue
    if col is None or len(r) <= col or not r[0].isdigit():
        continue
    try:
        s = int(r[col])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    if key not in agg:
        agg[key] = [0, r[1].strip()[:90]]
    agg[key][0] += s
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for (f, ln), (s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s:8d} {100.0 * s / max(tot, 1):5.1f}%  {f}:{ln}  {src}")
