#!/usr/bin/env python
"""Single-process NVLink push probe (2 GPUs): the P rank's pool on cuda:0, the D rank's
pool on cuda:1 with peer access enabled, the fused convert kernel on cuda:0 storing
straight into cuda:1's HBM.  Used for ncu captures of the push kernel (ncu must not wrap a
multi-rank command) and for a peer-copy ceiling in the same process.
    python tools/push_single.py [--workload c4] [--iters 10] [--copy]
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
from tools._workload import Workload, sample_parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--copy", action="store_true", help="also time a cudaMemcpyPeer-style torch copy 0 -> 1")
    ap.add_argument("--layer-chunk", type=int, default=0)
    ap.add_argument("--budgets", default="0", help="comma list of SM budgets to sweep (0 = all SMs)")
    ap.add_argument("--pull", action="store_true",
                    help="D-initiated read (the paper's direction): the kernel runs on cuda:1 and loads from cuda:0")
    ap.add_argument("--dst-dtype", default="", help="override the destination dtype (f16|bf16|e4m3|f32)")
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()[args.workload]
    if args.dst_dtype:
        import dataclasses
        cfg = dataclasses.replace(cfg, dst_dtype={"f16": synth.F16, "bf16": synth.BF16, "e4m3": synth.E4M3,
                                                  "f32": synth.F32}[args.dst_dtype])
    torch.cuda.set_device(0)
    kvx.peer_enable(1)
    src = Workload(cfg, [0], [], torch.device("cuda", 0))  # also holds D's tables on cuda:0
    torch.cuda.set_device(1)
    dst = Workload(cfg, [], [0], torch.device("cuda", 1))
    torch.cuda.set_device(0)
    S, SP = src.src_lays[0], src.src_pools[0]
    DP = dst.dst_pools[0]
    # P's view of the D layout: D's fp8 scales on P's GPU (the sender casts)
    sc = dst.dst_dicts[0].get("scales")
    Dl = kvx.Layout.from_dict(dst.dst_dicts[0], None if sc is None else torch.from_numpy(sc).to("cuda:0"))
    lc = args.layer_chunk or cfg.L

    dev = 0
    if args.pull:
        torch.cuda.set_device(1)
        kvx.peer_enable(0)
        torch.cuda.set_device(0)
        dev, Dl = 1, dst.dst_lays[0]

    def fn():
        with torch.cuda.device(dev):
            for l0 in range(0, cfg.L, lc):
                if args.pull:
                    kvx.convert_share(S, SP, dst.src_bt, [Dl], [DP], dst.dst_bt, (l0, min(cfg.L, l0 + lc)))
                else:
                    kvx.convert_share(S, SP, src.src_bt, [Dl], [DP], src.dst_bt, (l0, min(cfg.L, l0 + lc)))

    # P rank 0's share of D rank 0 (all of it when tp_p <= tp_d; half of c2's fan-in 2)
    nvl = src.src_bytes([0]) * synth.NBYTES[cfg.dst_dtype] // synth.NBYTES[cfg.src_dtype]
    whole = cfg.tp_p <= cfg.tp_d
    for budget in [int(x) for x in args.budgets.split(",")]:
        kvx.set_sm_budget(budget)
        for _ in range(3):
            fn()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        with torch.cuda.device(dev):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.iters)]
            for a, b in ev:
                a.record()
                fn()
                b.record()
        torch.cuda.synchronize(dev)
        ts = [a.elapsed_time(b) for a, b in ev]
        med = statistics.median(ts)
        out = {"case": f"{args.workload} pair {'pull (kernel on cuda:1)' if args.pull else 'push'} cuda:0 -> cuda:1", "sm_budget": budget or "all",
               "ms_med": round(med, 4), "ms_min": round(min(ts), 4),
               "nvlink_GBs": round(nvl / med / 1e6, 1), "frac_770": round(nvl / med / 1e6 / 770, 4),
               "src_GBs": round(src.src_bytes([0]) / med / 1e6, 1), "nvlink_bytes": nvl, "layer_chunk": lc}
        torch.cuda.synchronize(1)
        dst.src_pools[0], dst.src_dicts[0] = SP, src.src_dicts[0]
        out["kernel"] = kvx.last_kernel()
        out["tile_env"] = os.environ.get("KVX_TILE", "1")
        if whole:
            ok, det = sample_parity(dst, (0, 1), 0, [0], [0])
            out["parity_ok"] = ok
        print(json.dumps(out), flush=True)
    kvx.set_sm_budget(0)
    if args.copy:
        n = 1 << 30
        a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"case": "torch copy_ cuda:0 -> cuda:1 (1 GiB)", "ms": round(ms, 4),
                          "GBs": round(n / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
