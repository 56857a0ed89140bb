#!/usr/bin/env python
"""One line per bench JSON line in a file (mode, ms/step, roofline achieved / frac, kernel, parity)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "roofline" not in d:
            print(d)
            continue
        c = d.get("config", {})
        par = d.get("parity")
        par = [p.get("ok") for p in par] if isinstance(par, list) else (par or {}).get("ok")
        print(c.get("workload", "")[:4], c.get("mode"), c.get("layer_chunk"), d["ms_per_step"], d["roofline"]["achieved"],
              d["roofline"]["frac"], d["roofline"].get("kernel"), par, d.get("gpu_launches"),
              d.get("latency_ms", ""))
