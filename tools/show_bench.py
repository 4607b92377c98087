"""Print the key fields of bench JSON lines in gpurun_out/."""
import json
import sys

for f in sys.argv[1:] or ["gpurun_out/bench_c2.log", "gpurun_out/bench_c3.log"]:
    try:
        lines = [x for x in open(f).read().strip().splitlines() if x.startswith("{")]
        d = json.loads(lines[-1])
        print(f, "ms/step", round(d["ms_per_step"], 4), "p99", round(d["p99_decision_ms"], 4),
              {k: round(v, 4) for k, v in d["stage_ms"].items()}, {k: round(v, 4) for k, v in d.get("kernel_ms", {}).items()})
        print("  phases", d["select_phases_us"]["us"])
        e = d.get("e2e") or {}
        print("  e2e", round(e.get("ms_per_step", 0), 3), "p99", round(e.get("p99_ms", 0), 3), e.get("host_wall_ms"))
        print("  victims", d["config"]["n_victims"], "roofline", d.get("roofline", {}).get("frac"),
              "sel", (d.get("roofline_select") or {}).get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
        for k, v in (d.get("need_sweep") or {}).items():
            print("  sweep", k, {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()})
        pf = d.get("prefetch")
        if pf:
            print("  prefetch", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in pf.items() if not isinstance(v, dict)})
            print("    e2e", pf.get("e2e"), "\n    roof", pf.get("roofline"), "\n    cpu", pf.get("cpu_baseline"))
        print("  launches", d.get("gpu_launches"), "lib", d.get("lib_calls"), "clocks", d.get("clocks"))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
