#!/usr/bin/env python
"""NEXT-3: the paper's own host-staged transport (P:95 steps 3/5/6) as a measured
baseline for what NVLink buys (transfer.HostStaged): P packs each layer chunk and copies it
into a pinned host buffer, D copies it up and unpacks it -- event-chained per chunk, with the
host buffer shared (the stand-in "RDMA read" between the two CPU buffers is free, so this is
the fastest host-staged path the box allows: PCIe-bound).  Measured beside the same
machine's PCIe copy rates (1 GiB pinned D2H / H2D) and checked against the oracle.

    python tools/host_staged.py [--workload c4] [--layer-chunk 4] [--iters 3] [--one-gpu]
Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import d_tables, make_d_rank, make_p_rank, o1_compare, p_tables, sample_of  # noqa: E402


def pcie_rates(dev, nbytes=1 << 30):
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    out = {}
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
        ts = []
        for i in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(dev):
                e0.record()
                fn()
                e1.record()
            torch.cuda.synchronize(dev)
            if i:
                ts.append(e0.elapsed_time(e1))
        out[name] = round(nbytes / (min(ts) * 1e-3) / 1e9, 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--layer-chunk", type=int, default=4)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--one-gpu", action="store_true")
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import transfer as tr
    cfg = synth.configs()[args.workload]
    dp, dd = torch.device("cuda", 0), torch.device("cuda", 0 if args.one_gpu else 1)
    NB_p, NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_p), synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    torch.cuda.set_device(dp)
    pd, S, SP = make_p_rank(cfg, 0, NB_p, dp)
    pt = p_tables(cfg, NB_p)
    sbt = kvx.Batch(S, cfg.n_tokens, pt, dp)
    torch.cuda.set_device(dd)
    ddict, Dl, DP, sc = make_d_rank(cfg, 0, NB_d, dd)
    dt_ = d_tables(cfg, NB_d)
    dbt = kvx.Batch(Dl, cfg.n_tokens, dt_, dd)
    torch.cuda.set_device(dp)
    Dl_p = kvx.Layout.from_dict(ddict, None if sc is None else sc.to(dp))   # D's scales at the sender
    hs = tr.HostStaged(S, Dl_p, Dl, cfg.total_tokens, (0, cfg.L), args.layer_chunk, dp, dd)
    hs.step(SP, sbt, DP, dbt)       # warm-up
    torch.cuda.synchronize(dp)
    torch.cuda.synchronize(dd)
    ts = []
    for _ in range(args.iters):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        start = torch.cuda.Event()
        with torch.cuda.device(dp):
            start.record(hs.sp)
        with torch.cuda.device(dd):   # both timing events on D's device (P's start seen from D)
            hs.sd.wait_event(start)
            e0.record(hs.sd)
        hs.step(SP, sbt, DP, dbt)
        with torch.cuda.device(dd):
            e1.record(hs.sd)
        torch.cuda.synchronize(dp)
        torch.cuda.synchronize(dd)
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    wire = sum(hs.nbytes)
    rates = pcie_rates(dp)
    ss = [sample_of(SP, pd, pt, [0], (0, 2))]
    ds = [sample_of(DP, ddict, dt_, [0], (0, 2))]
    par = o1_compare(ss, ds, [cfg.n_tokens[0]], cfg.dst_dtype)
    print(json.dumps({"case": f"{args.workload} pair host-staged (pack, D2H, shared pinned buffer, H2D, unpack)"
                              + (" on one GPU" if args.one_gpu else " GPU0 -> GPU1"),
                      "ms_min": round(ms, 2), "ms_all": [round(t, 2) for t in ts],
                      "wire_GBs": round(wire / ms / 1e6, 2), "wire_bytes": wire, "layer_chunk": args.layer_chunk,
                      "pcie_copy_GBs": rates, "frac_of_pcie": round(wire / ms / 1e6 / min(rates.values()), 3),
                      "parity": par, "timing": "CUDA events, P stream start -> D stream end, best of iters"}),
          flush=True)


if __name__ == "__main__":
    main()
