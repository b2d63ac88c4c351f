"""Aggregate ncu warp-stall samples and executed instructions per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python ncu_lines.py x.csv [N]
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
def f(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0
agg, text, cur, fname, hdr = {}, {}, None, "?", None
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0] and r[0].isdigit() and len(r) > 7:
        cur = (fname, int(r[0])); text[cur] = r[1].strip()
        a = agg.setdefault(cur, [0.0, 0.0, {}])
        a[0] += f(r[4]); a[1] += f(r[7])
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                a[2][h[6:]] = a[2].get(h[6:], 0.0) + f(r[i])
tot = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
print(f"samples {tot:.0f}  warp-insts {ti:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    st = sorted(v[2].items(), key=lambda x: -x[1])[:3]
    why = " ".join(f"{n}:{100*x/max(v[0],1):.0f}" for n, x in st)
    print(f"{k[0][:14]:14s}:{k[1]:<5d} {100*v[0]/tot:5.1f}% smp {100*v[1]/ti:5.1f}% ins [{why:28s}] {text.get(k,'')[:70]}")
