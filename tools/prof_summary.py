"""Summarise ncu --csv launch lists (gpu__time_duration, dram bytes) per libwhit kernel."""
import csv, json, sys
from collections import defaultdict


def summarise(path, last_n=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    launches = defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi or "whit" not in r[ki]:
            continue
        mult = {"ns": 1e-6, "usecond": 1e-3, "msecond": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
        launches[int(r[0])][r[mi]] = float(r[vi].replace(",", "")) * mult
        names[int(r[0])] = r[ki]
    per = defaultdict(list)
    for i in sorted(launches):
        per[names[i]].append(launches[i])
    out = {}
    for name, ls in per.items():
        ls = ls[-last_n:] if last_n else ls
        t = [l.get("gpu__time_duration.sum") for l in ls]
        rd = [l.get("dram__bytes_read.sum", 0) for l in ls]
        wr = [l.get("dram__bytes_write.sum", 0) for l in ls]
        out[name] = {"launches": len(ls), "avg_ms": sum(t) / len(t),
                     "dram_bytes_per_launch": (sum(rd) + sum(wr)) / len(ls) if rd[0] else None,
                     "dram_GBps": ((sum(rd) + sum(wr)) / len(ls)) / (sum(t) / len(t) / 1e3) / 1e9 if rd[0] else None}
    tot = sum(v["avg_ms"] * v["launches"] for v in out.values())
    for v in out.values():
        v["share_of_listed_time"] = v["avg_ms"] * v["launches"] / tot
    return out


if __name__ == "__main__":
    res = {}
    for p in sys.argv[1:]:
        res[p.split("/")[-1]] = summarise(p, last_n=2)
    print(json.dumps(res, indent=1))
