#!/usr/bin/env python
"""NEXT-4: by-layer transmission overlapping prefill compute ("parallel transmission
and calculation ... through by-layer transmission").  One process, two GPUs: the P rank
(cuda:0) runs a synthetic prefill (one bf16 GEMM per layer, calibrated to roughly the
layer's transfer time) on a compute stream; the fused push of layer l (c4 pair, NVLink
into cuda:1) starts on a second stream as soon as layer l's compute event fires, with the
push limited to `budget` SMs (kv_set_sm_budget) so the GEMMs keep the rest.

Reports compute-only, push-only, sequential (compute then push) and overlapped times;
hidden = (sequential - overlapped) / min(compute, push).
    python tools/overlap.py [--budgets 0,64,32,16] [--gemm 4096]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import Workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--budgets", default="0,64,32,16")
    ap.add_argument("--gemm", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()[args.workload]
    torch.cuda.set_device(0)
    kvx.peer_enable(1)
    src = Workload(cfg, [0], [], torch.device("cuda", 0))
    torch.cuda.set_device(1)
    dst = Workload(cfg, [], [0], torch.device("cuda", 1))
    torch.cuda.set_device(0)
    S, SP = src.src_lays[0], src.src_pools[0]
    sc = dst.dst_dicts[0].get("scales")
    Dl = kvx.Layout.from_dict(dst.dst_dicts[0], None if sc is None else torch.from_numpy(sc).to("cuda:0"))
    DP = dst.dst_pools[0]
    n = args.gemm
    A = torch.randn(n, n, dtype=torch.bfloat16, device="cuda:0")
    B = torch.randn(n, n, dtype=torch.bfloat16, device="cuda:0")
    C = torch.empty(n, n, dtype=torch.bfloat16, device="cuda:0")
    cs, xs = torch.cuda.Stream(), torch.cuda.Stream()
    L = cfg.L

    def timed(fn):
        best = None
        for _ in range(args.iters + 1):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        return best

    def enqueue_compute(evs):
        with torch.cuda.stream(cs):
            for l in range(L):
                torch.matmul(A, B, out=C)
                evs[l].record(cs)

    def enqueue_push(evs):
        for l in range(L):
            if evs is not None:
                xs.wait_event(evs[l])
            kvx.convert_reshard([S], [SP], src.src_bt, [Dl], [DP], src.dst_bt, (l, l + 1), xs)

    def run(compute, push, overlap):
        cur = torch.cuda.current_stream()
        cs.wait_stream(cur)
        xs.wait_stream(cur)
        evs = [torch.cuda.Event() for _ in range(L)]
        if compute:
            enqueue_compute(evs)
        if push:
            if compute and not overlap:
                xs.wait_stream(cs)  # sequential: all prefill first
            enqueue_push(evs if (compute and overlap) else None)
        cur.wait_stream(cs)
        cur.wait_stream(xs)

    res = {"case": f"{args.workload} pair, {L} layers, GEMM {n}^3 bf16 per layer", "runs": []}
    t_c = timed(lambda: run(True, False, False))
    for budget in [int(x) for x in args.budgets.split(",")]:
        kvx.set_sm_budget(budget)
        t_x = timed(lambda: run(False, True, False))
        t_seq = timed(lambda: run(True, True, False))
        t_ovl = timed(lambda: run(True, True, True))
        res["runs"].append({"push_sm_budget": budget or 148, "compute_ms": round(t_c, 3), "push_ms": round(t_x, 3),
                            "sequential_ms": round(t_seq, 3), "overlapped_ms": round(t_ovl, 3),
                            "hidden_frac": round((t_seq - t_ovl) / min(t_c, t_x), 3),
                            "push_nvlink_GBs": round(dst.dst_bytes([0]) / t_x / 1e6, 1)})
    kvx.set_sm_budget(0)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
