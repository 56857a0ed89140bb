#!/usr/bin/env python
"""Single-process probe of the staged pull (2 GPUs): P = cuda:0 packs (sender-side cast)
layer chunks into a ring, D = cuda:1 unpacks them straight from the peer-mapped ring.
  --mode d_only : P stages every chunk first (ring = all chunks), then D's pull alone is
                  timed (the kernel's own NVLink read rate, no pipeline effects);
  --mode overlap: P and D run concurrently with a ring of --ring slots (the real pipeline).
Each is run with the persistent one-launch D kernel (counters) and the per-chunk path.
    python tools/pull_probe.py [--workload c4] [--layer-chunk 8] [--ring 3] [--iters 5] [--requests 1]
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
    ap.add_argument("--layer-chunk", type=int, default=8)
    ap.add_argument("--ring", type=int, default=3)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--modes", default="d_only,overlap")
    ap.add_argument("--requests", type=int, default=0, help="first N requests only (1: batch-1 latency)")
    args = ap.parse_args()
    import paper_2509_17542_b200 as kvx
    cfg = synth.configs()[args.workload]
    if args.requests:
        import dataclasses
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
    Sd = kvx.Layout.from_dict(src.src_dicts[0])  # P layout handle for D's calls (no device data)
    L, lc = cfg.L, args.layer_chunk
    nch = kvx.chunk_count((0, L), lc)
    step = abs(lc) or L   # lc < 0: the ramped schedule (its chunks are never larger than |lc|)
    slot = max(kvx.wire_bytes(S, Dv, cfg.total_tokens, (l0, min(L, l0 + step))) for l0 in range(0, L, step))
    slot = (slot + 255) // 256 * 256
    ready = torch.zeros(8, dtype=torch.int32, device="cuda:1")
    free = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    err0 = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    err1 = torch.zeros(1, dtype=torch.int32, device="cuda:1")
    counters = torch.zeros(2 * nch + 1, dtype=torch.int32, device="cuda:1")
    s0, s1 = torch.cuda.Stream(0), torch.cuda.Stream(1)
    seq = [0]
    nvl = src.src_bytes([0]) * synth.NBYTES[cfg.dst_dtype] // synth.NBYTES[cfg.src_dtype]
    for mode in args.modes.split(","):
        R = nch if mode == "d_only" else args.ring
        ring = torch.empty(R * slot, dtype=torch.uint8, device="cuda:0")
        rp = [ring.data_ptr() + b * slot for b in range(R)]
        for persistent in (True, False):
            if persistent:
                os.environ.pop("KVX_PULL_CHUNKED", None)
            else:
                os.environ["KVX_PULL_CHUNKED"] = "1"

            def p_side():
                with torch.cuda.device(0):
                    kvx.stage(S, SP, src.src_bt, [Dv], rp, R, slot, [ready.data_ptr()], [free], seq[0], err0,
                              (0, L), lc, 20.0, s0)

            def d_side():
                with torch.cuda.device(1):
                    kvx.pull_staged([Sd], rp, R, slot, Dl, DP, dst.dst_bt, [ready], [free.data_ptr()], seq[0], err1,
                                    (0, L), lc, 20.0, s1, counters=counters if persistent else None)

            ts, p_ms = [], []
            for it in range(args.iters + 2):
                if mode == "d_only":
                    p_side()
                    torch.cuda.synchronize(0)
                    with torch.cuda.device(1):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(s1)
                        d_side()
                        b.record(s1)
                    torch.cuda.synchronize(1)
                else:
                    torch.cuda.synchronize(0)
                    torch.cuda.synchronize(1)
                    with torch.cuda.device(1):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(s1)
                    with torch.cuda.device(0):
                        a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a0.record(s0)
                    p_side()
                    with torch.cuda.device(0):
                        b0.record(s0)
                    d_side()
                    with torch.cuda.device(1):
                        b.record(s1)
                    torch.cuda.synchronize(0)
                    torch.cuda.synchronize(1)
                    if it >= 2:
                        p_ms.append(a0.elapsed_time(b0))
                seq[0] += nch
                if it >= 2:
                    ts.append(a.elapsed_time(b))
            med = statistics.median(ts)
            out = {"case": f"{args.workload} staged pull cuda:0 -> cuda:1", "mode": mode,
                   "d_kernel": "persistent k_pull_rows" if persistent else "per-chunk wait/unpack/signal",
                   "last_kernel": kvx.last_kernel(), "layer_chunk": lc, "chunks": nch, "ring": R,
                   "ms_med": round(med, 4), "ms_min": round(min(ts), 4), "nvlink_GBs": round(nvl / med / 1e6, 1),
                   "frac_770": round(nvl / med / 1e6 / 770, 4), "err": int(err0.item()) + int(err1.item()),
                   "p_stage_ms": round(statistics.median(p_ms), 4) if p_ms else None}
            dst.src_pools[0], dst.src_dicts[0] = SP, src.src_dicts[0]
            ok, det = sample_parity(dst, (0, 1), 0, [0], [0])
            out["parity_ok"] = ok
            print(json.dumps(out), flush=True)
        del ring


if __name__ == "__main__":
    main()
