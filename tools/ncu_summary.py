#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a `--set full` report (.ncu-rep) and/or a
launch list (--metrics gpu__time_duration.sum CSV).

usage: python tools/ncu_summary.py [--rep X.ncu-rep] [--launches launches.csv] [--out profiles/foo.json]
"""
import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
    "smsp__cycles_active.avg",
]


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in h:
                v = r[h.index(m)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                d[m] = v
                if units[h.index(m)]:
                    d[m + ".unit"] = units[h.index(m)]
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = d["dram__bytes_read.sum"] * scale.get(d.get("dram__bytes_read.sum.unit", "byte"), 1)
            wr = d["dram__bytes_write.sum"] * scale.get(d.get("dram__bytes_write.sum.unit", "byte"), 1)
            d["dram_bytes_per_launch"] = rd + wr
        res.append(d)
    return res


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    unit = rows[hi + 1][h.index("Metric Unit")] if "Metric Unit" in h else "ns"
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:90]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "total_" + unit: sum(v), "avg_" + unit: sum(v) / len(v),
                    "share": sum(v) / tot})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out")
    a = ap.parse_args()
    res = {}
    if a.rep:
        res["full"] = rep_summary(a.rep)
    if a.launches:
        res["launch_list"] = launch_summary(a.launches)
    s = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(s)
    print(s)
