#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, on files gpurun brought back).

  python tools/ncu_summary.py full  gpurun_out/prof_c2.ncu-rep  profiles/r01_c2_full.json  [--traffic-key c2@1]
  python tools/ncu_summary.py launches gpurun_out/launches_c2.csv profiles/r01_c2_launches.json
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def full(rep, out, traffic_key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                rec[k] = {"value": _num(d[hdr.index(k)]), "unit": units[hdr.index(k)]}
        st = {h[len(STALLS):]: _num(d[i]) for i, h in enumerate(hdr) if h.startswith(STALLS) and h.endswith(".ratio")}
        rec["warp_stall_ratio_top"] = dict(sorted(((k, v) for k, v in st.items() if isinstance(v, float)),
                                                  key=lambda kv: -kv[1])[:6])
        res.append(rec)
    with open(out, "w") as f:
        json.dump({"source": os.path.basename(rep), "launches": res}, f, indent=1)
    if traffic_key:
        r = res[0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tb = sum(r[k]["value"] * scale.get(r[k]["unit"], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
        t = json.load(open(p)) if os.path.exists(p) else {}
        t[traffic_key] = int(tb)
        json.dump(t, open(p, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


def launches(csvf, out):
    txt = open(csvf).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    agg = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:120]
        v = _num(r[vi])
        a = agg.setdefault(name, {"launches": 0, "us_total": 0.0})
        if r[mi] == "gpu__time_duration.sum":
            v *= {"msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}.get(r[ui], 1.0)
            a["launches"] += 1
            a["us_total"] += v
        elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(r[ui], 1.0)
            a["dram_bytes_total"] = a.get("dram_bytes_total", 0.0) + v
    tot = sum(a["us_total"] for a in agg.values())
    for a in agg.values():
        a["share"] = round(a["us_total"] / tot, 4) if tot else None
        a["us_mean"] = round(a["us_total"] / a["launches"], 2) if a["launches"] else None
        if "dram_bytes_total" in a and a["launches"]:
            a["dram_bytes_per_launch"] = round(a.pop("dram_bytes_total") / a["launches"])
    res = dict(sorted(agg.items(), key=lambda kv: -kv[1]["us_total"]))
    json.dump({"source": os.path.basename(csvf), "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
               "(cold-cache, serialised: compare shares)", "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    mode, a, b = sys.argv[1:4]
    tk = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    full(a, b, tk) if mode == "full" else launches(a, b)
