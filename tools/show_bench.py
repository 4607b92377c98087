"""Print the key fields of bench JSON lines in gpurun_out/."""
import json
import sys

for f in sys.argv[1:] or ["gpurun_out/bench_c2.log", "gpurun_out/bench_c3.log"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/step", round(d["ms_per_step"], 4), "p99", round(d["p99_decision_ms"], 4),
              {k: round(v, 4) for k, v in d["stage_ms"].items()}, {k: round(v, 4) for k, v in d.get("kernel_ms", {}).items()}, "phases", d["select_phases_us"]["us"],
              "e2e", round(d["e2e"]["ms_per_step"], 3), "victims", d["config"]["n_victims"],
              "roofline", d.get("roofline", {}).get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
