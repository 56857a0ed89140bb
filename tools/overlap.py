#!/usr/bin/env python
"""NEXT-4: by-layer transmission overlapping prefill compute ("parallel transmission
and calculation ... through by-layer transmission").  One process, two GPUs: the P rank
(cuda:0) runs a synthetic prefill (one bf16 GEMM per layer, calibrated to roughly the
layer's transfer time) on a compute stream; the fused push of layer l (c4 pair, NVLink
into cuda:1) starts on a second stream as soon as layer l's compute event fires, with the
push limited to `budget` SMs (kv_set_sm_budget) so the GEMMs keep the rest.

Reports compute-only, push-only, sequential (compute then push) and overlapped times;
hidden = (sequential - overlapped) / min(compute, push).

--mode pull: the D-initiated read instead.  After layer l's GEMM the P rank packs + casts
layer l into a ring slot (kv_stage, one chunk) and releases it; the D rank (cuda:1) runs ONE
persistent kv_pull_staged over all layers that waits in-kernel for each layer.  P's SMs only
run the short HBM-bound packs, so the prefill loses little; the budget caps the pack.
    python tools/overlap.py [--mode push|pull] [--budgets 0,64,32,16] [--carveouts 16:16,24:24] [--gemm 4096]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from tools._workload import Workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--budgets", default="0,64,32,16")
    ap.add_argument("--gemm", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--mode", default="push", choices=["push", "pull"])
    ap.add_argument("--ring", type=int, default=4)
    ap.add_argument("--carveouts", default="",
                    help="budget:carveout pairs, e.g. 16:16,24:24 -- the transfer kernels capped at `budget` SMs "
                         "AND cuBLAS kept off `carveout` SMs (torch._C._set_sm_carveout_experimental), so the "
                         "prefill GEMMs and the pack / push run side by side instead of taking turns")
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
    pull = args.mode == "pull"
    if pull:
        torch.cuda.set_device(1)
        kvx.peer_enable(0)
        torch.cuda.set_device(0)
        ds = torch.cuda.Stream(device=1)
        Sd = kvx.Layout.from_dict(src.src_dicts[0])   # P's layout for D's calls (bf16: no device data)
        R = args.ring
        slot = max(kvx.wire_bytes(S, Dl, cfg.total_tokens, (l, l + 1)) for l in range(L))
        slot = (slot + 255) // 256 * 256
        ring = torch.empty(R * slot, dtype=torch.uint8, device="cuda:0")
        rp = [ring.data_ptr() + b * slot for b in range(R)]
        ready = torch.zeros(4, dtype=torch.int32, device="cuda:1")
        free = torch.zeros(4, dtype=torch.int32, device="cuda:0")
        err0 = torch.zeros(1, dtype=torch.int32, device="cuda:0")
        err1 = torch.zeros(1, dtype=torch.int32, device="cuda:1")
        counters = torch.zeros(2 * L + 1, dtype=torch.int32, device="cuda:1")
        seq = [0]

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

    def enqueue_pull(evs):
        for l in range(L):   # P: pack + cast layer l once its GEMM is done, release the slot
            if evs is not None:
                xs.wait_event(evs[l])
            kvx.stage(S, SP, src.src_bt, [Dl], rp, R, slot, [ready.data_ptr()], [free], seq[0] + l, err0,
                      (l, l + 1), 1, 20.0, xs)
        with torch.cuda.device(1):   # D: one persistent read of every layer as it is released
            kvx.pull_staged([Sd], rp, R, slot, dst.dst_lays[0], DP, dst.dst_bt, [ready], [free.data_ptr()], seq[0],
                            err1, (0, L), 1, 20.0, ds, counters=counters)
        seq[0] += L

    def run(compute, push, overlap):
        cur = torch.cuda.current_stream()
        cs.wait_stream(cur)
        xs.wait_stream(cur)
        if pull:
            st = torch.cuda.Event()
            st.record(cur)
            ds.wait_event(st)
        evs = [torch.cuda.Event() for _ in range(L)]
        if compute:
            enqueue_compute(evs)
        if push:
            if compute and not overlap:
                xs.wait_stream(cs)  # sequential: all prefill first
                if pull:
                    e = torch.cuda.Event()
                    e.record(cs)
                    ds.wait_event(e)
            if pull:
                enqueue_pull(evs if (compute and overlap) else None)
            else:
                enqueue_push(evs if (compute and overlap) else None)
        cur.wait_stream(cs)
        cur.wait_stream(xs)
        if pull:
            e = torch.cuda.Event()
            e.record(ds)
            cur.wait_event(e)

    res = {"case": f"{args.workload} pair, {L} layers, GEMM {n}^3 bf16 per layer, {args.mode}", "runs": []}
    pairs = [(int(x), 0) for x in args.budgets.split(",") if x]
    pairs += [tuple(int(v) for v in x.split(":")) for x in args.carveouts.split(",") if x]
    t_c0 = timed(lambda: run(True, False, False))
    for budget, carve in pairs:
        torch._C._set_sm_carveout_experimental(carve or None)
        t_c = timed(lambda: run(True, False, False)) if carve else t_c0
        kvx.set_sm_budget(budget)
        t_x = timed(lambda: run(False, True, False))
        t_seq = timed(lambda: run(True, True, False))
        t_ovl = timed(lambda: run(True, True, True))
        res["runs"].append({"transfer_sm_budget_on_P": budget or 148, "gemm_sm_carveout": carve,
                            "compute_ms": round(t_c, 3), "compute_ms_all_sms": round(t_c0, 3), "push_ms": round(t_x, 3),
                            "sequential_ms": round(t_seq, 3), "overlapped_ms": round(t_ovl, 3),
                            "hidden_frac": round((t_seq - t_ovl) / min(t_c, t_x), 3),
                            "vs_all_sm_prefill_ms": round(t_ovl - t_c0, 3),
                            "push_nvlink_GBs": round(dst.dst_bytes([0]) / t_x / 1e6, 1)})
    kvx.set_sm_budget(0)
    torch._C._set_sm_carveout_experimental(None)
    if pull:
        res["err"] = int(err0.item()) + int(err1.item())
        dst.src_pools[0], dst.src_dicts[0] = SP, src.src_dicts[0]
        from tools._workload import sample_parity
        res["parity_ok"] = sample_parity(dst, (0, 1), 0, [0], [0])[0]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
