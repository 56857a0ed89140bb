#!/usr/bin/env python
"""NEXT-3: the paper's own host-staged transport (P:95 steps 3/5/6) as a measured
baseline for what NVLink buys.  One process, two GPUs:

  P (cuda:0): kv_pack a layer chunk -> D2H into P's pinned "CPU buffer"
  host:       copy P's buffer -> D's pinned buffer (stand-in for the transfer engine's
              RDMA read between the two CPU buffers)
  D (cuda:1): H2D into a device wire -> kv_unpack into the D pool

double-buffered per layer chunk so the three copies overlap.  Compared with the fused
NVLink push of the same c4 pair (tools/push_single.py).  Prints one JSON line.
    python tools/host_staged.py [--workload c4] [--layer-chunk 4] [--iters 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import Workload, sample_parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--layer-chunk", type=int, default=4)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()[args.workload]
    torch.cuda.set_device(0)
    src = Workload(cfg, [0], [], torch.device("cuda", 0))
    torch.cuda.set_device(1)
    dst = Workload(cfg, [], [0], torch.device("cuda", 1))
    S, SP = src.src_lays[0], src.src_pools[0]
    Dl, DP = dst.dst_lays[0], dst.dst_pools[0]
    # P's view of the D layout: the fp8 scales must live on P's GPU (the sender casts)
    sc = dst.dst_dicts[0].get("scales")
    Dl_p = kvx.Layout.from_dict(dst.dst_dicts[0], None if sc is None else torch.from_numpy(sc).to("cuda:0"))
    lc = args.layer_chunk
    chunks = [(l0, min(cfg.L, l0 + lc)) for l0 in range(0, cfg.L, lc)]
    nb = max(kvx.wire_bytes(S, Dl, cfg.total_tokens, c) for c in chunks)
    w0 = [torch.empty(nb, dtype=torch.uint8, device="cuda:0") for _ in range(2)]
    w1 = [torch.empty(nb, dtype=torch.uint8, device="cuda:1") for _ in range(2)]
    hA = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]  # P's CPU buffer
    hB = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]  # D's CPU buffer
    s0 = torch.cuda.Stream(device=0)
    s1 = torch.cuda.Stream(device=1)

    def transfer():
        e0 = [None] * len(chunks)
        e1 = [None] * len(chunks)

        def enqueue_p(k):
            lr = chunks[k]
            n = kvx.wire_bytes(S, Dl, cfg.total_tokens, lr)
            with torch.cuda.device(0), torch.cuda.stream(s0):
                kvx.pack(S, SP, src.src_bt, Dl_p, w0[k % 2], lr, s0, wire_nbytes=n)
                hA[k % 2][:n].copy_(w0[k % 2][:n], non_blocking=True)
                e0[k] = torch.cuda.Event()
                e0[k].record(s0)

        enqueue_p(0)
        for k, lr in enumerate(chunks):
            n = kvx.wire_bytes(S, Dl, cfg.total_tokens, lr)
            if k + 1 < len(chunks):
                if k >= 1:
                    e0[k - 1].synchronize()  # slot (k+1)%2 of hA was consumed by the host copy of k-1
                enqueue_p(k + 1)
            e0[k].synchronize()
            if k >= 2:
                e1[k - 2].synchronize()  # D's buffer slot reused
            np.copyto(hB[k % 2][:n].numpy(), hA[k % 2][:n].numpy())  # the "RDMA read"
            with torch.cuda.device(1), torch.cuda.stream(s1):
                w1[k % 2][:n].copy_(hB[k % 2][:n], non_blocking=True)
                kvx.unpack(S, Dl, DP, dst.dst_bt, w1[k % 2], lr, s1, wire_nbytes=n)
                e1[k] = torch.cuda.Event()
                e1[k].record(s1)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)

    transfer()  # warm-up
    ts = []
    for _ in range(args.iters):
        t = time.perf_counter()
        transfer()
        ts.append(time.perf_counter() - t)
    ms = 1e3 * min(ts)
    nvl = dst.dst_bytes([0])
    dst.src_pools[0], dst.src_dicts[0] = SP, src.src_dicts[0]
    ok, _ = sample_parity(dst, (0, 1), 0, [0], [0])
    print(json.dumps({"case": f"{args.workload} pair host-staged (pack, D2H, host copy, H2D, unpack)",
                      "ms_min": round(ms, 2), "ms_all": [round(1e3 * t, 2) for t in ts],
                      "wire_GBs": round(nvl / ms / 1e6, 2), "src_GBs": round(src.src_bytes([0]) / ms / 1e6, 2),
                      "layer_chunk": lc, "wire_bytes": nvl, "parity_ok": ok,
                      "timing": "wall clock (host-orchestrated pipeline), best of iters"}), flush=True)


if __name__ == "__main__":
    main()
