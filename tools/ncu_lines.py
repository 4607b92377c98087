"""Per-CUDA-source-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
fname = ""
out = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0] not in ("", "Line No"):
        try:
            s = int(r[4])
        except ValueError:
            continue
        out.append((s, f"{fname}:{r[0]}", r[1][:100]))
tot = sum(o[0] for o in out) or 1
print("total samples", tot)
for s, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {loc:18s} {src}")
