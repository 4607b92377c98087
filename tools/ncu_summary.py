"""Key metrics of ncu raw-page CSVs -> markdown table + profiles/traffic.json
(dram bytes read + write per launch of each kernel, the bench's roofline
`traffic`).  usage: python tools/ncu_summary.py out.md raw1.csv [raw2.csv ...]"""
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("smsp__inst_executed.avg.per_cycle_active", "IPC/SMSP"), ("launch__registers_per_thread", "regs"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX %")]

out, traffic = [], {}
try:
    traffic = json.load(open(os.path.join("profiles", "traffic.json")))
except Exception:
    pass
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0].split("::")[-1].split("<")[0]
        vals = {}
        for k, label in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                vals[label] = (v, u.get(k, ""))
        rd = vals.get("DRAM read")
        wr = vals.get("DRAM write")
        if rd and wr:
            traffic[name] = int(rd[0] * UNITS.get(rd[1], 1) + wr[0] * UNITS.get(wr[1], 1))
        out.append((name, vals))
md = ["| kernel | " + " | ".join(l for _, l in KEYS) + " |", "|---|" + "---|" * len(KEYS)]
for name, vals in out:
    md.append(f"| {name} | " + " | ".join(f"{vals[l][0]:.4g} {vals[l][1]}" if l in vals else "-" for _, l in KEYS) + " |")
open(sys.argv[1], "w").write("\n".join(md) + "\n")
json.dump(traffic, open(os.path.join("profiles", "traffic.json"), "w"), indent=1)
print("\n".join(md))
