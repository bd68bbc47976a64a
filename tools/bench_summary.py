import json, sys
for fn in sys.argv[1:]:
    try:
        d = json.load(open(fn))
    except Exception as e:
        print(fn, "unreadable", e); continue
    r = d["roofline"]
    print(d["config"]["workload"][:60], "| ms/step %.1f" % d["ms_per_step"], "| value %.3e" % d["value"],
          "| e2e %.3e" % d["e2e"]["value"], "| K4 %.2f TF frac %.3f share %.2f" % (r["achieved"] or 0, r["frac"] or 0, r["share_of_step"]))
    print("   ", {k: round(v, 2) for k, v in d["kernels_ms_per_step"].items() if v > 0.3})
