#!/usr/bin/env python
"""NEXT-3 layout variants at c4 size on one GPU: one TP4 pair (L=80, 2 local heads, D=128,
32 x 4096 tokens, block 16) from an other-vendor-style P cache -- separate K and V pools,
the K pool x-packed ([LAYER], BLOCK, HEAD, D/8, SLOT, x=8), the V pool head_dim-major
([LAYER], BLOCK, HEAD, DIM, SLOT) -- into the NVIDIA-style D pool (BLOCK, LAYER, KV, HEAD, SLOT, DIM),
bf16 -> e4m3 (or --src fnuz).  Two convert calls (K, V) vs the combined-pool baseline.
    python tools/variants_bench.py [--src bf16|fnuz] [--iters 10]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import BLOCK, DIM, HEAD, KV, LAYER, SLOT  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="bf16", choices=["bf16", "fnuz", "e4m3"])
    ap.add_argument("--dst", default="e4m3", choices=["e4m3", "bf16", "fnuz", "f32"])
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    from bench import load_peaks
    L, H, D, tp, B = 80, 8, 128, 4, 16
    n_tokens = [4096] * 32
    names = {"bf16": synth.BF16, "fnuz": synth.FNUZ, "e4m3": synth.E4M3, "f32": synth.F32}
    sdt, ddt = names[args.src], names[args.dst]
    NB = synth.pool_capacity(n_tokens, B)
    st = synth.block_tables(11, n_tokens, B, NB)
    dt_ = synth.block_tables(12, n_tokens, B, NB)
    dev = torch.device("cuda", 0)
    ssc = torch.from_numpy(synth.pow2_scales(5, L, H // tp)).to(dev) if sdt in synth.FP8 else None
    dsc = torch.from_numpy(synth.pow2_scales(6, L, H // tp)).to(dev) if ddt in synth.FP8 else None
    vend = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)   # per-layer tensors; the KV axis has extent 1
    Kl = kvx.Layout(L, H, D, tp, 0, B, NB, sdt, vend, ssc, kv_part=1, dim_split=16 // synth.NBYTES[sdt])
    Vl = kvx.Layout(L, H, D, tp, 0, B, NB, sdt, vend, ssc, kv_part=2)
    Cl = kvx.Layout(L, H, D, tp, 0, B, NB, sdt, synth.P_ORDER, ssc)
    Dl = kvx.Layout(L, H, D, tp, 0, B, NB, ddt, synth.D_ORDER, dsc)
    pools = {}
    for name, lay in (("K", Kl), ("V", Vl), ("C", Cl)):
        t = lay.new_pool(dev)
        synth.fill_random_finite_(t.view(torch.uint8 if synth.NBYTES[sdt] == 1 else torch.int16), 40 + len(pools), sdt)
        pools[name] = t
    DP = Dl.new_pool(dev, fill=synth.CANARY)
    sbt = kvx.Batch(Cl, n_tokens, st, dev)
    dbt = kvx.Batch(Dl, n_tokens, dt_, dev)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.iters)]
        for a, b in ev:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ev)

    src_b = 2 * L * (H // tp) * D * sum(n_tokens) * synth.NBYTES[sdt]
    dst_b = 2 * L * (H // tp) * D * sum(n_tokens) * synth.NBYTES[ddt]
    pk = load_peaks()["hbm_gbs"]
    res = []
    for label, fn in [
        ("combined P pool (P_ORDER) -> D", lambda: kvx.convert_reshard([Cl], [pools["C"]], sbt, [Dl], [DP], dbt)),
        ("K pool (x-packed) + V pool -> D, two calls",
         lambda: (kvx.convert_reshard([Kl], [pools["K"]], sbt, [Dl], [DP], dbt),
                  kvx.convert_reshard([Vl], [pools["V"]], sbt, [Dl], [DP], dbt))),
        ("K pool (x-packed) only -> D", lambda: kvx.convert_reshard([Kl], [pools["K"]], sbt, [Dl], [DP], dbt)),
        ("V pool (head_dim-major) only -> D", lambda: kvx.convert_reshard([Vl], [pools["V"]], sbt, [Dl], [DP], dbt)),
    ]:
        ms = timed(fn)
        frac_b = (src_b + dst_b) / (2 if "only" in label else 1)
        res.append({"case": label, "src": args.src, "dst": args.dst, "ms": round(ms, 4), "hbm_GBs": round(frac_b / ms / 1e6, 1),
                    "frac_measured": round(frac_b / ms / 1e6 / pk, 3), "kernel": kvx.last_kernel()})
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
