#!/usr/bin/env python
"""Kernel-level sweep: the fused convert on one GPU for several BASELINE shapes (the
"1-GPU convert" rows of BASELINE.md), plus a torch copy_ calibration in the same process.
Prints one JSON line per case.  Not the driver's bench (see bench.py)."""
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
from tools._workload import Workload, sample_parity  # noqa: E402


def time_it(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in ev]
    return statistics.median(ts), min(ts)


def case(name, cfg, p_ranks, d_ranks, contiguous=False, parity=True, layer_chunk=0):
    import paper_2509_17542_b200 as kvx
    w = Workload(cfg, p_ranks, d_ranks, torch.device("cuda", 0), contiguous)
    S = [w.src_lays[p] for p in p_ranks]
    SP = [w.src_pools[p] for p in p_ranks]
    Dl = [w.dst_lays[q] for q in d_ranks]
    DP = [w.dst_pools[q] for q in d_ranks]
    lc = layer_chunk or cfg.L

    def fn():
        for l0 in range(0, cfg.L, lc):
            kvx.convert_reshard(S, SP, w.src_bt, Dl, DP, w.dst_bt, (l0, min(cfg.L, l0 + lc)))

    med, mn = time_it(fn)
    sb, db = w.src_bytes(p_ranks), w.dst_bytes(d_ranks)
    pk = load_peaks()["hbm_gbs"]
    out = {"case": name, "ms_med": round(med, 4), "ms_min": round(mn, 4), "src_GBs": round(sb / med / 1e6, 1),
           "hbm_GBs": round((sb + db) / med / 1e6, 1), "frac_measured": round((sb + db) / med / 1e6 / pk, 3),
           "bytes": sb + db, "layer_chunk": lc}
    if parity:
        ok, det = sample_parity(w, (0, 1), 0, p_ranks, d_ranks)
        out["parity_ok"] = ok
    print(json.dumps(out), flush=True)
    del w
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="copy,c2,c3,c4,c4c,c5")
    args = ap.parse_args()
    cf = synth.configs()
    sel = args.cases.split(",")
    if "copy" in sel:
        x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
        y = torch.empty_like(x)
        med, mn = time_it(lambda: y.copy_(x))
        print(json.dumps({"case": "torch copy_ 2 GiB r+w", "ms_med": round(med, 4),
                          "GBs": round(2 * x.numel() * 2 / med / 1e6, 1)}), flush=True)
        del x, y
        torch.cuda.empty_cache()
    if "copy1g" in sel:  # the same bytes as c2 (1 GiB read + 1 GiB written)
        x = torch.empty(1 << 29, dtype=torch.bfloat16, device="cuda")
        y = torch.empty_like(x)
        med, mn = time_it(lambda: y.copy_(x))
        print(json.dumps({"case": "torch copy_ 1 GiB r+w (c2's bytes)", "ms_med": round(med, 4),
                          "GBs": round(2 * x.numel() * 2 / med / 1e6, 1)}), flush=True)
        del x, y
        torch.cuda.empty_cache()
    if "c1" in sel:
        case("c1 tiny fp16->bf16 16->32", cf["c1"], [0], [0])
    if "c2" in sel:
        case("c2 TP2->1 fp16 (all ranks one GPU)", cf["c2"], [0, 1], [0])
    if "c2c" in sel:
        case("c2 TP2->1 fp16, contiguous tables", cf["c2"], [0, 1], [0], contiguous=True, parity=False)
    if "c3" in sel:
        case("c3 one D rank: P0,P1 -> D0 bf16 16->64", cf["c3"], [0, 1], [0])
    if "c4" in sel:
        case("c4 one pair: P0 -> D0 bf16->e4m3", cf["c4"], [0], [0])
    if "c4c" in sel:
        case("c4 one pair, contiguous tables", cf["c4"], [0], [0], contiguous=True, parity=False)
    if "c5" in sel:
        import dataclasses
        c5 = cf["c5"]
        inst_a = dataclasses.replace(c5, n_tokens=c5.n_tokens[0::2])  # P instance A's requests
        case(f"c5 instance A ({len(inst_a.n_tokens)} req, {inst_a.total_tokens} tok) rank0 -> D0,D1 split bf16",
             inst_a, [0], [0, 1], parity=True)


if __name__ == "__main__":
    main()
