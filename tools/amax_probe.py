#!/usr/bin/env python
"""kv_compute_scales (NEXT-1 dynamic fp8 scales) at c4 pair size on one GPU: one read pass
of the P rank's bf16 pool (10.7 GB) -> [L][2][H_d] scales.  For ncu captures of k_amax_rows.
    python tools/amax_probe.py [--iters 10]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import load_peaks  # noqa: E402
from tools._workload import Workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()["c4"]
    w = Workload(cfg, [0], [0], torch.device("cuda", 0))
    out = torch.empty(cfg.L * 2 * (cfg.H // cfg.tp_d), dtype=torch.float32, device="cuda")
    fn = lambda: kvx.compute_scales([w.src_lays[0]], [w.src_pools[0]], w.src_bt, w.dst_lays[0], out)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.iters)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    nb = w.src_bytes([0])
    print(json.dumps({"case": "c4 pair kv_compute_scales (amax pass)", "ms": round(ms, 4),
                      "GBs": round(nb / ms / 1e6, 1), "frac_measured": round(nb / ms / 1e6 / load_peaks()["hbm_gbs"], 3),
                      "note": "read-only pass: the copy peak (read + write) is the conservative denominator"}))


if __name__ == "__main__":
    main()
