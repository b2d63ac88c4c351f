"""One line per bench JSON line: workload / op, value, ms, roofline frac + per-launch ms, clocks."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        if "value" not in d:
            print(f, d)
            continue
        r = d.get("roofline") or {}
        c = d.get("clocks") or {}
        print(f"{d['config'].get('workload')}/{d['config'].get('op', 'fwdbwd')} {d['value']:.4g} {d['unit']} "
              f"ms {d['ms_per_step']:.3f} frac {r.get('frac')} dom {r.get('kernel')} {r.get('launch_ms')} "
              f"clk {c.get('sm_mhz')} {c.get('reasons')}")
        for k in ("e2e", "w_bits", "cpu_baseline", "e2e_wbits"):
            v = d.get(k)
            if isinstance(v, dict):
                extra = v.get("roofline", {}).get("frac") if isinstance(v.get("roofline"), dict) else ""
                print(f"   {k}: {v.get('value'):.4g} {extra}")
