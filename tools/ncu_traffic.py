"""Rebuild profiles/ncu_traffic.json (the per-launch DRAM traffic bench.py reports as roofline.traffic).

usage: python tools/ncu_traffic.py <full.ncu-rep | raw.csv> <launch-list dir> <prefix> [out.json]

* headline (`whit_forward` / `whit_backward` keys): the two whit_kernel launches of one `ncu --set full`
  capture of tools/quick_time.py hetero (DRAM bytes, duration, fp64 pipe %, issue %, registers);
* workloads (`<workload>/<launch>` keys): mean over the launches of each `ncu --metrics gpu__time_duration.sum,
  dram__bytes_read.sum,dram__bytes_write.sum` launch list `<dir>/<prefix><tag>_whit.csv` of
  `bench.py <op> --steps 2 --warmup 3` (the launch list's kernels mapped to bench.py's launch names).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

# launch-list tag -> (workload key, {kernel-name prefix: bench launch name})
WORKLOADS = {
    "xopirregular": ("irregular", {"whit_irr_kernel<2, float, 1, 0>": "whit_forward_times",
                                    "whit_irr_kernel<2, float, 1, 1>": "whit_backward"}),
    "xoptable1": ("table1", {"whit_mb2_kernel<2, float, 1, 0, 1>": "whit_forward_times_bands",
                             "whit_mb2_kernel<2, float, 1, 1, 1>": "whit_backward_bands"}),
    "xoptrain": ("train", {"whit_kernel<2, float, 1, 0, 1, 0>": "whit_forward_mse",
                           "whit_kernel<2, float, 1, 1, 0, 0>": "whit_backward"}),
    "xopvariance": ("variance", {"whit_var_kernel<2, float, 1>": "whit_posterior_variance"}),
    "xconfigs2tile": ("s2tile", {"whit_mb2_kernel<2, float, 1, 0, 0>": "whit_forward_bands",
                                 "whit_mb2_kernel<2, float, 1, 1, 0>": "whit_backward_bands"}),
}


def raw_rows(src):
    if src.endswith(".ncu-rep"):
        out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
    else:
        rows = list(csv.reader(open(src)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def launch_list(path):
    per = defaultdict(lambda: defaultdict(list))  # kernel -> metric -> values (per launch)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        per[r["Kernel Name"]][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    return per


def main():
    src, ldir, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                             "ncu_traffic.json")
    res = {"source": "ncu --set full --clock-control none --import-source on -k regex:whit_kernel -s 6 -c 2, "
                     "tools/quick_time.py hetero (%s); dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                     "fp64 = sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" % os.path.basename(src)}
    for r, name in zip(raw_rows(src), ("whit_forward", "whit_backward")):
        rd, wr = float(r["dram__bytes_read.sum"]) * 1e9, float(r["dram__bytes_write.sum"]) * 1e9
        ms = float(r["gpu__time_duration.sum"])
        res[name] = {"kernel": r["Kernel Name"], "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                     "duration_ms": ms, "dram_TBps": round((rd + wr) / ms / 1e9, 3),
                     "fp64_pipe_pct": round(float(r["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]), 1),
                     "issue_active_pct": round(float(r["smsp__issue_active.avg.pct_of_peak_sustained_active"]), 1),
                     "registers": int(float(r["launch__registers_per_thread"]))}
    res["workloads_source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                               "-k regex:whit python bench.py <op> --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "
                               "(%s<tag>_whit.csv, mean over the launches); keys '<workload>/<launch>'" % prefix)
    for tag, (wl, names) in WORKLOADS.items():
        path = os.path.join(ldir, "%s%s_whit.csv" % (prefix, tag))
        if not os.path.exists(path):
            continue
        for kern, m in launch_list(path).items():
            launch = next((v for k, v in names.items() if kern.startswith("void " + k)), None)
            if launch is None:
                continue
            n = len(m["gpu__time_duration.sum"])
            byt = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / n
            ms = sum(m["gpu__time_duration.sum"]) / n / 1e6  # ns -> ms
            res["%s/%s" % (wl, launch)] = {"kernel": kern, "dram_bytes_per_launch": byt, "duration_ms": ms,
                                           "dram_TBps": round(byt / ms / 1e9, 3), "launches": n}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main()
