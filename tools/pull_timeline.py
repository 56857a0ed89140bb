#!/usr/bin/env python
"""Timeline of one staged pull (2 GPUs, not part of the library): P = cuda:0 stages the
chunks one kv_stage call per chunk with %globaltimer stamps (kv_timestamp) after each
free-slot wait and after each pack + ready signal; D = cuda:1 runs the persistent
kv_pull_staged with stamps before and after.  Shows where a single request's transfer
waits: the pipeline fill (first pack), P waiting for free slots, D starving for chunks.
    python tools/pull_timeline.py [--workload c4] [--requests 1] [--layer-chunk 20] [--ring 3]
The two GPUs' globaltimers are compared directly (both follow the host clock; the skew is
printed as measured by a stamp pair taken back to back after a device synchronize).
"""
import argparse
import dataclasses
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
    ap.add_argument("--requests", type=int, default=1)
    ap.add_argument("--layer-chunk", type=int, default=20)
    ap.add_argument("--ring", type=int, default=3)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--sleep-ms", type=float, default=0.0,
                    help="P's stream sleeps this long first, so the host enqueues every chunk ahead of the GPU")
    ap.add_argument("--p-only", action="store_true", help="no D pull: ring slots for every chunk, packs alone")
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()[args.workload]
    if args.requests:
        cfg = dataclasses.replace(cfg, n_tokens=cfg.n_tokens[:args.requests])
    torch.cuda.set_device(0)
    kvx.peer_enable(1)
    src = Workload(cfg, [0], [], torch.device("cuda", 0))
    torch.cuda.set_device(1)
    kvx.peer_enable(0)
    dst = Workload(cfg, [], [0], torch.device("cuda", 1))
    torch.cuda.set_device(0)
    S, SP = src.src_lays[0], src.src_pools[0]
    sc = dst.dst_dicts[0].get("scales")
    Dv = kvx.Layout.from_dict(dst.dst_dicts[0], None if sc is None else torch.from_numpy(sc).to("cuda:0"))
    Dl, DP = dst.dst_lays[0], dst.dst_pools[0]
    Sd = kvx.Layout.from_dict(src.src_dicts[0])
    L, lc = cfg.L, args.layer_chunk
    chunks = [(l0, min(L, l0 + lc)) for l0 in range(0, L, lc)]
    nch = len(chunks)
    R = nch if args.p_only else args.ring
    assert kvx.chunk_count((0, L), lc) == nch
    slot = max(kvx.wire_bytes(S, Dv, cfg.total_tokens, c) for c in chunks)
    slot = (slot + 255) // 256 * 256
    ring = torch.empty(R * slot, dtype=torch.uint8, device="cuda:0")
    rp = [ring.data_ptr() + b * slot for b in range(R)]
    ready = torch.zeros(8, dtype=torch.int32, device="cuda:1")
    free = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    err0 = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    err1 = torch.zeros(1, dtype=torch.int32, device="cuda:1")
    counters = torch.zeros(2 * nch + 1, dtype=torch.int32, device="cuda:1")
    tp = torch.zeros(2 * nch + 2, dtype=torch.int64, device="cuda:0")
    td = torch.zeros(4, dtype=torch.int64, device="cuda:1")
    s0, s1 = torch.cuda.Stream(0), torch.cuda.Stream(1)
    seq = 0
    for it in range(args.iters):
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        # clock skew probe: stamps on both GPUs back to back
        with torch.cuda.device(1):
            kvx.timestamp(td[2:3], s1)
        with torch.cuda.device(0):
            kvx.timestamp(tp[2 * nch + 1:], s0)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        if not args.p_only:
            with torch.cuda.device(1):
                kvx.timestamp(td[0:1], s1)
                kvx.pull_staged([Sd], rp, R, slot, Dl, DP, dst.dst_bt, [ready], [free.data_ptr()], seq, err1, (0, L),
                                lc, 20.0, s1, counters=counters)
                kvx.timestamp(td[1:2], s1)
        with torch.cuda.device(0):
            if args.sleep_ms:
                with torch.cuda.stream(s0):
                    torch.cuda._sleep(int(args.sleep_ms * 1.9e6))
            kvx.timestamp(tp[0:1], s0)
            for k, (l0, l1) in enumerate(chunks):
                if k >= R:
                    kvx.wait(free, seq + k + 1 - R, err0, 20.0, s0)
                kvx.timestamp(tp[1 + 2 * k:2 + 2 * k], s0)
                kvx.stage(S, SP, src.src_bt, [Dv], rp, R, slot, [ready.data_ptr()], [free], seq + k, err0, (l0, l1),
                          lc, 20.0, s0)
                kvx.timestamp(tp[2 + 2 * k:3 + 2 * k], s0)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        seq += nch
        a, b = tp.cpu().tolist(), td.cpu().tolist()
        base = a[0]
        skew = b[2] - a[2 * nch + 1]
        if args.p_only:
            ready.zero_()
            free.fill_(seq)   # every slot "read": the next iteration's chunks may reuse them
        out = {"iter": it, "p_only": args.p_only, "sleep_ms": args.sleep_ms, "layer_chunk": lc, "chunks": nch, "ring": R, "err": int(err0.item()) + int(err1.item()),
               "skew_us_d_minus_p": round(skew / 1e3, 2),
               "d_start_us": round((b[0] - base) / 1e3, 1), "d_end_us": round((b[1] - base) / 1e3, 1),
               "p_slot_free_us": [round((a[1 + 2 * k] - base) / 1e3, 1) for k in range(nch)],
               "p_ready_us": [round((a[2 + 2 * k] - base) / 1e3, 1) for k in range(nch)],
               "wire_MB": round(kvx.wire_bytes(S, Dv, cfg.total_tokens, (0, L)) / 1e6, 1)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
