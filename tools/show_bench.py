import json, sys
for p in sys.argv[1:]:
    t = open(p).read().strip().splitlines()
    try:
        d = json.loads([x for x in t if x.startswith("{")][-1])
    except Exception:
        print(p, "\n".join(t[-12:])); continue
    r = d.get("roofline") or {}
    print(p, "value", d["value"], "ms", d["ms_per_step"], "e2e", (d.get("e2e") or {}).get("value"),
          "roof", r.get("kernel"), r.get("achieved"), r.get("frac"), "step_frac", r.get("step_frac"),
          "launches", d.get("gpu_launches"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    for k in ("kernels_ms", "codec", "parity", "method", "exchange", "phases"):
        if k in d:
            print("  ", k, d[k])
