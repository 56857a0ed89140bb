#!/usr/bin/env python
"""bench.py -- KV transfer GB/s and ms/request (P -> D, device-timed) vs the HBM/NVLink
roofline, for the heterogeneous-compatible KV transmission path (arXiv 2509.17542, III-B).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode push|nccl]

N = 1 (default): BASELINE configs[1] (c2: Llama-2-7B KV, one 2048-token prompt, P TP=2 -> D TP=1,
  fp16, block 16 -> 16, P layout NHD-per-layer -> D layout block-major HND) with all three
  ranks' pools on one GPU: one fused kv_convert_reshard launch per step, HBM-bound.
N >= 2 (torchrun, one process per GPU): BASELINE configs[3] (c4: Llama-3-70B GQA KV,
  32 x 4096 tokens, P TP=4 -> D TP=4, bf16 -> fp8-e4m3 per-head scale) as N/2 independent
  (P rank p -> D rank p) pairs on disjoint GPUs (P = ranks 0..N/2-1): N=8 is the full c4,
  N=2/4 its per-GPU-equivalent sub-configs; per-pair work fixed -> weak
  scaling.  `--workload c3|c2` runs the largest complete sub-transfer that fits (c3 at N=4:
  P0,P1 -> D0, fan-in 2; N=6 the full c3); `--workload c5` the mixed-length stream.
  Default mode "push": the fused gather+convert kernel stores into the D rank's
  IPC-mapped pool over NVLink, then a release flag (K4/K5); "nccl": pack -> ncclSend /
  ncclRecv -> unpack, per-layer pipelined.

One JSON line on rank 0 (contract in the task statement); `value` = logical source KV
GB (2*L*H*D*T*bytes_src summed over all requests and pairs) / max-over-ranks device time.
Inputs are larger than L2 (GBs per step), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "KV transfer GB/s and ms/request (P\u2192D, device-timed) vs HBM/NVLink roofline"  # BASELINE.json verbatim
NVLINK_MEASURED_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction
NVLINK_NOMINAL_GBS = 900.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="pull", choices=["push", "pull", "nccl"])
    ap.add_argument("--ring-slots", type=int, default=3, help="pull mode, narrowing cast: staging ring depth")
    ap.add_argument("--dynamic-scales", action="store_true",
                    help="pull mode, fp8 destination: P computes per-chunk amax scales and ships them (NEXT-1 i)")
    ap.add_argument("--layer-chunk", type=int, default=0, help="layers per chunk (0 = whole model)")
    ap.add_argument("--chunk-mib", type=int, default=64, help="c5: merge layers until a chunk moves this much")
    ap.add_argument("--c5-batch", action="store_true", help="c5: push each instance's requests as one batch")
    ap.add_argument("--requests", type=int, default=0,
                    help="use only the first N requests of the workload (e.g. 1: batch-1 latency of c3/c4)")
    ap.add_argument("--workload", default=None, help="override: c1..c5")
    ap.add_argument("--tokens", type=int, default=0, help="one request of this many tokens (paper points)")
    ap.add_argument("--tp-p", type=int, default=0, help="override the P TP degree")
    ap.add_argument("--tp-d", type=int, default=0, help="override the D TP degree")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-sample-layers", type=int, default=0)
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------------------------
# clocks during the timed region (pynvml polling thread)
# ------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, torch_dev):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                pr = torch.cuda.get_device_properties(torch_dev)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(int(torch_dev))
            self.h, self.nv = h, pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it, never fake numbers
            self.err = repr(e)

    def _poll(self):
        nv = self.nv
        getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(getr(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "nvml off")}
        self._stop.set()
        self.t.join()
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------------------
# workload construction (inputs from synth; device memory from torch)
# ------------------------------------------------------------------------------------
class Workload:
    """One instance pair's layouts, pools, tables for the P ranks / D ranks on this process."""

    def __init__(self, cfg, p_ranks, d_ranks, device, contiguous=False):
        import torch
        import paper_2509_17542_b200 as kvx
        self.cfg, self.device = cfg, device
        c = cfg
        self.NB_p = synth.pool_capacity(c.n_tokens, c.B_p)
        self.NB_d = synth.pool_capacity(c.n_tokens, c.B_d)
        self.src_tables = synth.block_tables(c.seed + 1, c.n_tokens, c.B_p, self.NB_p, contiguous)
        self.dst_tables = synth.block_tables(c.seed + 2, c.n_tokens, c.B_d, self.NB_d, contiguous)
        self.p_ranks, self.d_ranks = list(p_ranks), list(d_ranks)
        self.src_dicts, self.src_lays, self.src_pools = {}, {}, {}
        for p in self.p_ranks:
            d = synth.layout(c.L, c.H, c.D, c.tp_p, p, c.B_p, self.NB_p, c.src_dtype, c.p_order)
            lay = kvx.Layout.from_dict(d)
            pool = lay.new_pool(device)
            view = pool.view(torch.uint8 if synth.NBYTES[c.src_dtype] == 1 else torch.int16)
            synth.fill_random_finite_(view, c.seed + 100 + p, c.src_dtype)
            self.src_dicts[p], self.src_lays[p], self.src_pools[p] = d, lay, pool
        self.dst_dicts, self.dst_lays, self.dst_pools, self.scales = {}, {}, {}, {}
        for q in self.d_ranks:
            sc_np = None
            sc = None
            if c.dst_dtype == synth.E4M3:
                sc_np = synth.pow2_scales(c.seed + 200 + q, c.L, c.H // c.tp_d)
                sc = torch.from_numpy(sc_np).to(device)
            d = synth.layout(c.L, c.H, c.D, c.tp_d, q, c.B_d, self.NB_d, c.dst_dtype, c.d_order, sc_np)
            lay = kvx.Layout.from_dict(d, sc)
            self.dst_dicts[q], self.dst_lays[q], self.scales[q] = d, lay, sc
            self.dst_pools[q] = lay.new_pool(device, fill=synth.CANARY)
        any_src = self.src_lays[self.p_ranks[0]] if self.p_ranks else kvx.Layout.from_dict(
            synth.layout(c.L, c.H, c.D, c.tp_p, 0, c.B_p, self.NB_p, c.src_dtype, c.p_order))
        any_dst = self.dst_lays[self.d_ranks[0]] if self.d_ranks else kvx.Layout.from_dict(
            synth.layout(c.L, c.H, c.D, c.tp_d, 0, c.B_d, self.NB_d, c.dst_dtype, c.d_order,
                         np.ones((c.L, 2, c.H // c.tp_d), np.float32)),
            torch.ones(c.L * 2 * (c.H // c.tp_d), device=device))
        self._keep = (any_src, any_dst)
        self.src_bt = kvx.Batch(any_src, c.n_tokens, self.src_tables, device)
        self.dst_bt = kvx.Batch(any_dst, c.n_tokens, self.dst_tables, device)

    # algorithmic bytes: what the method must move
    def src_bytes(self, p_ranks=None):
        c = self.cfg
        n = len(p_ranks) if p_ranks is not None else c.tp_p
        return 2 * c.L * (c.H // c.tp_p) * n * c.D * c.total_tokens * synth.NBYTES[c.src_dtype]

    def dst_bytes(self, d_ranks=None):
        c = self.cfg
        n = len(d_ranks) if d_ranks is not None else c.tp_d
        padded = sum(synth.blocks_for(t, c.B_d) * c.B_d for t in c.n_tokens)
        return 2 * c.L * (c.H // c.tp_d) * n * c.D * padded * synth.NBYTES[c.dst_dtype]


def extract(pool_t, d, layers, block_ids):
    """Compact host copy of a pool restricted to layers [lb, le) and the given blocks
    (same axis order) -> (numpy codes, layout dict).  Bench/test infrastructure."""
    import torch
    nb = synth.NBYTES[d["dtype"]]
    tdt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[nb]
    ext = {synth.LAYER: d["L"], synth.KV: 2, synth.BLOCK: d["NB"], synth.SLOT: d["B"],
           synth.HEAD: d["H"] // d["tp"], synth.DIM: d["D"]}
    t = pool_t.view(tdt).view([ext[a] for a in d["order"]])
    t = t.index_select(d["order"].index(synth.LAYER), torch.arange(layers[0], layers[1], device=t.device))
    t = t.index_select(d["order"].index(synth.BLOCK), torch.as_tensor(block_ids, device=t.device, dtype=torch.long))
    a = t.contiguous().cpu().numpy().reshape(-1)
    a = a.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[nb])
    nd = dict(d)
    nd["L"], nd["NB"] = layers[1] - layers[0], len(block_ids)
    if d.get("scales") is not None:
        nd["scales"] = np.asarray(d["scales"])[layers[0]:layers[1]]
    return a, nd


def sample_parity(w: Workload, layers, req, p_ranks, d_ranks, dst_pool_of=None):
    """Oracle check of the measured buffers on a sample: request `req`, layers [lb, le),
    the given ranks.  Returns (ok, detail)."""
    from oracle import o1
    dst_pool_of = dst_pool_of or (lambda q: w.dst_pools[q])
    c = w.cfg
    st, dt = w.src_tables[req], w.dst_tables[req]
    src_lays, src_pools = [], []
    for p in p_ranks:
        a, nd = extract(w.src_pools[p], w.src_dicts[p], layers, st)
        src_lays.append(nd)
        src_pools.append(a)
    dst_lays, dst_pools, got = [], [], []
    for q in d_ranks:
        g, nd = extract(dst_pool_of(q), w.dst_dicts[q], layers, dt)
        dst_lays.append(nd)
        got.append(g)
        dst_pools.append(np.full_like(g, 0).view(np.uint8).copy().view(g.dtype))
        dst_pools[-1][:] = np.frombuffer(bytes([synth.CANARY]) * g.nbytes, dtype=g.dtype)
    o1.convert(src_lays, src_pools, dst_lays, dst_pools, [c.n_tokens[req]], [list(range(len(st)))],
               [list(range(len(dt)))])
    bad = 0
    maxulp = 0
    for g, want in zip(got, dst_pools):
        if c.dst_dtype == synth.E4M3:
            def ordv(x):
                x = x.astype(np.int32)
                return np.where(x & 0x80, -(x & 0x7F), x & 0x7F)
            dd = np.abs(ordv(g) - ordv(want))
            maxulp = max(maxulp, int(dd.max(initial=0)))
            bad += int((dd > 1).sum())
        else:
            bad += int((g != want).sum())
    n = sum(g.size for g in got)
    return bad == 0, {"elements": int(n), "mismatches": bad, "max_e4m3_ulp": maxulp if c.dst_dtype == synth.E4M3 else None,
                      "sample": f"request {req}, layers [{layers[0]},{layers[1]}), P ranks {list(p_ranks)} -> D ranks {list(d_ranks)}"}


def cpu_baseline(cfg, layers, p_ranks, d_ranks, req=0, threads=1):
    """Time the oracle O1 (as it stands) on a bounded sample of the workload.  threads > 1
    runs the same function on disjoint layer ranges in parallel (ctypes releases the GIL),
    the split SURVEY 8(d) names; threads = 1 is the plain single-thread oracle."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import o1
    from tests.kvcase import make_case
    case = make_case(layers, cfg.H, cfg.D, cfg.tp_p, cfg.tp_d, cfg.B_p, cfg.B_d, [cfg.n_tokens[req]], cfg.src_dtype,
                     cfg.dst_dtype, cfg.p_order, cfg.d_order, seed=cfg.seed, scales="pow2", tail_garbage=False)
    src_l = [case["src_lays"][p] for p in p_ranks]
    src_p = [case["src_pools"][p] for p in p_ranks]
    dst_l = [case["dst_lays"][q] for q in d_ranks]
    dst_p = [case["dst_pools"][q] for q in d_ranks]
    ranges = [(i * layers // threads, (i + 1) * layers // threads) for i in range(threads)]
    ranges = [r for r in ranges if r[1] > r[0]]
    o1.lib()
    t0 = time.perf_counter()
    if len(ranges) == 1:
        o1.convert(src_l, src_p, dst_l, dst_p, case["n_tokens"], case["src_tables"], case["dst_tables"])
    else:
        with ThreadPoolExecutor(len(ranges)) as ex:
            list(ex.map(lambda lr: o1.convert(src_l, src_p, dst_l, dst_p, case["n_tokens"], case["src_tables"],
                                              case["dst_tables"], lr), ranges))
    dt = time.perf_counter() - t0
    nbytes = 2 * layers * (cfg.H // cfg.tp_p) * len(p_ranks) * cfg.D * cfg.n_tokens[req] * synth.NBYTES[cfg.src_dtype]
    return nbytes, dt


# ------------------------------------------------------------------------------------
# N = 1: c2 on one GPU (HBM-bound fused convert)
# ------------------------------------------------------------------------------------
def run_single(args):
    import torch
    import paper_2509_17542_b200 as kvx
    torch.cuda.set_device(0)
    cfgs = synth.configs()
    wl_name = args.workload or "c2"
    cfg = _subset(cfgs[wl_name], args)
    dev = torch.device("cuda", 0)
    w = Workload(cfg, range(cfg.tp_p), range(cfg.tp_d), dev)
    S = [w.src_lays[p] for p in w.p_ranks]
    SP = [w.src_pools[p] for p in w.p_ranks]
    Dl = [w.dst_lays[q] for q in w.d_ranks]
    DP = [w.dst_pools[q] for q in w.d_ranks]
    stream = torch.cuda.current_stream()
    lc = args.layer_chunk or cfg.L

    def step(ev=None):
        for l0 in range(0, cfg.L, lc):
            if ev is not None:
                ev[0].record(stream)
            kvx.convert_reshard(S, SP, w.src_bt, Dl, DP, w.dst_bt, (l0, min(cfg.L, l0 + lc)), stream)
            if ev is not None:
                ev[1].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    K = args.steps
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(0)
    clocks.start()
    kvx.launch_count_reset()
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(K):
        step(kev[i] if lc == cfg.L else None)
    t1.record(stream)
    torch.cuda.synchronize()
    launches = kvx.launch_count()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    ms = total_ms / K
    src_b, dst_b = w.src_bytes(), w.dst_bytes()
    kts = [a.elapsed_time(b) for a, b in kev] if lc == cfg.L else [ms]
    kern_ms = statistics.mean(kts)
    peaks = load_peaks()
    alg = src_b + dst_b  # HBM read + write per launch
    achieved = alg / (kern_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(src_b / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
        "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 5),
        "ms_per_request": round(ms / len(cfg.n_tokens), 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype_name(cfg),
        "data": "synthetic (seeded random finite bit patterns, Fisher-Yates block tables)",
        "config": {"workload": f"{wl_name} one GPU: {cfg.note}; all P and D ranks' pools on cuda:0",
                   "requests": len(cfg.n_tokens), "tokens": cfg.total_tokens, "overrides": _overrides(args),
                   "layout": "P (L,KV,BLK,SLOT,H,D) -> D (BLK,L,KV,H,SLOT,D)",
                   "src_bytes_per_step": src_b, "dst_bytes_per_step": dst_b,
                   "l2": "inputs larger than L2 (no flush)", "parallelism": "none (1 GPU)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": _traffic(f"{wl_name}@1"),
                     "kernel": kvx.last_kernel(), "kernel_ms": round(kern_ms, 5),
                     "kernel_ms_median": round(statistics.median(kts), 5), "kernel_ms_min": round(min(kts), 5),
                     "algorithmic_bytes_per_launch": alg, "peak_source": peaks["source"],
                     "frac_vs_nominal_8TBs": round(achieved / 8000.0, 4)},
        "clocks": clk, "gpu_launches": int(launches),
    }
    if not args.no_parity:
        ok, det = sample_parity(w, (0, min(2, cfg.L)), 0, w.p_ranks, w.d_ranks)
        out["parity"] = {"ok": ok, **det}
    if not args.no_e2e:
        out["e2e"] = e2e_single(w, S, Dl, min(K, 10), stream, src_b)
    if not args.no_cpu_baseline:
        nl = args.cpu_sample_layers or min(cfg.L, 12)
        nb, dt = cpu_baseline(cfg, nl, w.p_ranks, w.d_ranks)
        out["cpu_baseline"] = {"value": round(nb / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                               "sample": f"O1 (plain C, 1 thread) on {wl_name} request 0, layers [0,{nl}) of {cfg.L}, "
                                         f"{nb} source bytes in {dt:.2f} s"}
        ncores = len(os.sched_getaffinity(0))
        nl_mt = min(cfg.L, max(nl, 2 * ncores))
        nb2, dt2 = cpu_baseline(cfg, nl_mt, w.p_ranks, w.d_ranks, threads=ncores)
        out["cpu_baseline_threads"] = {"value": round(nb2 / dt2 / 1e9, 4), "unit": "GB/s", "cores": ncores,
                                       "kind": "oracle",
                                       "sample": f"same O1 split by layer over {ncores} threads, layers [0,{nl_mt}), "
                                                 f"{nb2} source bytes in {dt2:.2f} s"}
    print(json.dumps(out), flush=True)


def e2e_single(w, S, Dl, K, stream, src_b):
    """Same metric through the public API with HOST buffers: every step uploads its source
    pools from pinned memory, runs the convert call and reads the destination pool back,
    all inside the timed region.  Steps are software-pipelined over two device buffer sets
    and three streams (upload, convert, read-back), so step k+1's upload and step k's
    read-back share the full-duplex PCIe link while step k converts."""
    import torch
    import paper_2509_17542_b200 as kvx
    hs = [_pinned_copy(w.src_pools[p]) for p in w.p_ranks]
    hd = [torch.empty(w.dst_pools[q].numel(), dtype=torch.uint8, pin_memory=True) for q in w.d_ranks]
    SP = [[w.src_pools[p] for p in w.p_ranks], [torch.empty_like(w.src_pools[p]) for p in w.p_ranks]]
    DP = [[w.dst_pools[q] for q in w.d_ranks], [w.dst_pools[q].clone() for q in w.d_ranks]]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    up.wait_stream(stream)
    down.wait_stream(stream)
    read_done = [None, None]
    for k in range(K):
        b = k & 1
        if read_done[b] is not None:          # the set's previous read-back must be done
            up.wait_event(read_done[b])
        with torch.cuda.stream(up):
            for d, h in zip(SP[b], hs):
                d.copy_(h, non_blocking=True)
        ev_up = torch.cuda.Event()
        ev_up.record(up)
        stream.wait_event(ev_up)
        kvx.convert_reshard(S, SP[b], w.src_bt, Dl, DP[b], w.dst_bt, None, stream)
        ev_cv = torch.cuda.Event()
        ev_cv.record(stream)
        down.wait_event(ev_cv)
        with torch.cuda.stream(down):
            for d, h in zip(DP[b], hd):
                h.copy_(d, non_blocking=True)
        read_done[b] = torch.cuda.Event()
        read_done[b].record(down)
    stream.wait_stream(down)
    stream.wait_stream(up)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / K
    return {"value": round(src_b / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int(sum(h.numel() for h in hs)), "d2h_bytes_per_step": int(sum(h.numel() for h in hd)),
            "steps": K, "pipelined": "2 buffer sets; upload / convert / read-back streams"}


def _pinned_copy(dev_tensor):
    """Pinned host copy of a device tensor without a pageable intermediate (GB-sized pools)."""
    import torch
    h = torch.empty(dev_tensor.numel(), dtype=dev_tensor.dtype, pin_memory=True)
    h.copy_(dev_tensor.view(-1))
    return h


def _subset(cfg, args):
    """--requests N: the first N requests of the configuration (batch-1 latency runs);
    --tokens T: one request of T tokens (the paper's input lengths: 256 / 512 /
    1024); --tp-p / --tp-d: other TP degrees on the same model (context points)."""
    import dataclasses
    if getattr(args, "requests", 0):
        cfg = dataclasses.replace(cfg, n_tokens=cfg.n_tokens[:args.requests])
    if getattr(args, "tokens", 0):
        cfg = dataclasses.replace(cfg, n_tokens=[args.tokens])
    if getattr(args, "tp_p", 0):
        cfg = dataclasses.replace(cfg, tp_p=args.tp_p)
    if getattr(args, "tp_d", 0):
        cfg = dataclasses.replace(cfg, tp_d=args.tp_d)
    return cfg


def _overrides(args):
    """The workload overrides of this run (empty for the BASELINE configurations as named)."""
    o = {k: getattr(args, k) for k in ("requests", "tokens", "tp_p", "tp_d") if getattr(args, k, 0)}
    return o or None


def _dtype_name(cfg):
    a, b = synth.DTYPE_NAMES[cfg.src_dtype], synth.DTYPE_NAMES[cfg.dst_dtype]
    return a if a == b else f"{a}->{b}"


def _traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture
    (profiles/traffic.json: "c2@1" single GPU, "<workload>:<mode>" for the NVLink modes)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(key)
    return None


# ------------------------------------------------------------------------------------
# N >= 2: c4 pairs across NVLink
# ------------------------------------------------------------------------------------
def run_multi(args):
    """N >= 2: a configuration's P -> D transfer across NVLink, P and D on disjoint GPUs.
    Ranks [0, n_p) are P TP ranks 0..n_p-1, [n_p, n_p + n_d) D TP ranks 0..n_d-1, the rest
    idle (transfer.present_ranks: the largest complete sub-transfer that fits; the full one
    when N >= tp_p + tp_d).  c4 (default): N/2 1:1 pairs; c3: P0,P1 -> D0 per 3 GPUs (fan-in
    2); c2: P0,P1 -> D0."""
    import torch
    import torch.distributed as dist
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import transfer as tr
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    wl_name = args.workload or "c4"
    cfg = _subset(synth.configs()[wl_name], args)
    n_p, n_d = tr.present_ranks(cfg.tp_p, cfg.tp_d, world)
    if n_p < 1 or n_d < 1:
        raise SystemExit(f"{wl_name} needs at least {1 + max(cfg.tp_p // cfg.tp_d, cfg.tp_d // cfg.tp_p, 1)} GPUs")
    roles = tr.roles(world, n_p, n_d, allow_idle=True)
    me = roles[rank]
    pairs = tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks=set(range(n_p)), d_ranks=set(range(n_d)))
    my_q = sorted({q for p, q, _, _ in pairs if me.kind == "P" and p == me.tp_rank})
    my_p = sorted({p for p, q, _, _ in pairs if me.kind == "D" and q == me.tp_rank})
    w = Workload(cfg, [me.tp_rank] if me.kind == "P" else [], [me.tp_rank] if me.kind == "D" else [], dev)
    stream = torch.cuda.current_stream()
    barrier_t = torch.zeros(1, device=dev)

    def barrier():
        dist.all_reduce(barrier_t)

    flags = torch.zeros(max(n_p, 1), dtype=torch.int32, device=dev)  # one word per P source
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    epoch = [0]
    lc = args.layer_chunk or cfg.L

    def d_view(q):  # P's view of D rank q's layout (D's fp8 scales on P's GPU: the sender casts)
        sc = None
        if cfg.dst_dtype == synth.E4M3:
            sc = torch.from_numpy(synth.pow2_scales(cfg.seed + 200 + q, cfg.L, cfg.H // cfg.tp_d)).to(dev)
        return kvx.Layout.from_dict(
            synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, w.NB_d, cfg.dst_dtype, cfg.d_order), sc)

    dyn = False
    if args.mode == "push":
        ch = tr.PushChannel(me, w.dst_pools.get(me.tp_rank), flags if me.kind == "D" else None)
        dst_lays = {q: d_view(q) for q in my_q}

        def step(ev=None):
            epoch[0] += 1
            if me.kind == "P":
                if ev is not None:
                    ev[0].record(stream)
                tr.push_step(w.src_lays[me.tp_rank], w.src_pools[me.tp_rank], w.src_bt, dst_lays, ch.peer_pool,
                             w.dst_bt, ch.peer_flag, epoch[0], lc, stream, flag_slot=me.tp_rank)
                if ev is not None:
                    ev[1].record(stream)
            elif me.kind == "D":
                for p in my_p:
                    kvx.wait(flags[p:p + 1], epoch[0], err, 30.0, stream)
    elif args.mode == "pull":
        # D-initiated read: D maps P's pool (or P's staging ring when the cast narrows)
        narrowing = synth.NBYTES[cfg.dst_dtype] < synth.NBYTES[cfg.src_dtype]
        p_lays = {p: kvx.Layout.from_dict(
            synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, w.NB_p, cfg.src_dtype, cfg.p_order))
            for p in my_p}
        R = max(1, args.ring_slots)
        if narrowing and not args.layer_chunk:
            # ~40 MiB of wire per chunk, at most 20 chunks (c4 full batch: 4 layers per chunk;
            # one request: 4 chunks of 20 layers), so the pipeline fill stays small and
            # per-chunk launch costs on P stay hidden behind D's reads.  Batch-1 c4 pair
            # (profiles/r01/batch1_chunks_c4_n2.jsonl): 2 / 4 / 8 / 16 chunks = 0.261 / 0.247 /
            # 0.286 / 0.359 ms
            pair_wire = 2 * cfg.L * min(cfg.H // cfg.tp_p, cfg.H // cfg.tp_d) * cfg.D * \
                synth.NBYTES[cfg.dst_dtype] * cfg.total_tokens
            n_ch = min(20, max(1, round(pair_wire / (40 << 20))))
            lc = -(-cfg.L // n_ch)
        ring, slot_bytes, dst_lays = None, 0, {}
        dyn = args.dynamic_scales and narrowing and synth.NBYTES[cfg.src_dtype] > 1
        own_scales = {}
        if me.kind == "P":
            if dyn:   # writable scale arrays on P: kv_stage fills them chunk by chunk
                own_scales = {q: torch.ones(cfg.L * 2 * (cfg.H // cfg.tp_d), device=dev) for q in my_q}
                dst_lays = {q: kvx.Layout.from_dict(
                    synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, w.NB_d, cfg.dst_dtype, cfg.d_order),
                    own_scales[q]) for q in my_q}
            else:
                dst_lays = {q: d_view(q) for q in my_q}
            S = w.src_lays[me.tp_rank]
            if narrowing:
                slot_bytes = max(kvx.wire_bytes(S, dst_lays[q], cfg.total_tokens, (l0, min(cfg.L, l0 + lc)))
                                 for q in my_q for l0 in range(0, cfg.L, lc))
                slot_bytes = (slot_bytes + 255) // 256 * 256
                ring = torch.empty(len(my_q) * R * slot_bytes, dtype=torch.uint8, device=dev)
                ring_ptrs = [ring.data_ptr() + (i * R + b) * slot_bytes for i in range(len(my_q)) for b in range(R)]
        pflags = torch.zeros(max(n_p, n_d, 1), dtype=torch.int32, device=dev)
        pch = tr.PullChannel(me, pflags, pool=w.src_pools[me.tp_rank] if me.kind == "P" and not narrowing else None,
                             ring=ring, ring_dst=my_q if ring is not None else (), ring_slots=R, slot_bytes=slot_bytes,
                             scales=w.scales.get(me.tp_rank) if dyn and me.kind == "D" else None)
        if me.kind == "D" and narrowing:
            slot_bytes = min(pch.slot_bytes[p] for p in my_p)
        nchunks = kvx.chunk_count((0, cfg.L), lc)
        counters = torch.zeros(2 * nchunks + 1, dtype=torch.int32, device=dev)
        seq = [0]

        def step(ev=None):
            epoch[0] += 1
            if ev is not None and me.kind == "D":
                ev[0].record(stream)
            if me.kind == "P":
                if narrowing:
                    kvx.stage(S, w.src_pools[me.tp_rank], w.src_bt, [dst_lays[q] for q in my_q],
                              ring_ptrs, R,
                              slot_bytes, [pch.peer_flag[q] for q in my_q], [pflags[q:q + 1] for q in my_q],
                              seq[0], err, (0, cfg.L), lc, 30.0, stream,
                              peer_scales=[pch.peer_scales[q] for q in my_q] if dyn else None)
                else:
                    for q in my_q:   # my KV is resident: D may read it; then wait until it has
                        kvx.signal(pch.peer_flag[q], epoch[0], stream)
                    for q in my_q:
                        kvx.wait(pflags[q:q + 1], epoch[0], err, 30.0, stream)
            elif me.kind == "D":
                q = me.tp_rank
                if narrowing:
                    kvx.pull_staged([p_lays[p] for p in my_p], [a for p in my_p for a in pch.src_ring[p]], R,
                                    slot_bytes, w.dst_lays[q], w.dst_pools[q], w.dst_bt,
                                    [pflags[p:p + 1] for p in my_p], [pch.peer_flag[p] for p in my_p], seq[0], err,
                                    (0, cfg.L), lc, 30.0, stream, counters=counters)
                else:
                    kvx.pull([p_lays[p] for p in my_p], [pch.src_pool[p] for p in my_p], w.src_bt, w.dst_lays[q],
                             w.dst_pools[q], w.dst_bt, [pflags[p:p + 1] for p in my_p],
                             [pch.peer_flag[p] for p in my_p], epoch[0], err, (0, cfg.L), lc, 30.0, stream)
            seq[0] += nchunks
            if ev is not None and me.kind == "D":
                ev[1].record(stream)
    else:
        # NCCL baseline: pack -> ncclSend / ncclRecv -> unpack, per-layer double-buffered
        uid = [kvx.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = kvx.Comm(world, rank, uid[0], local)
        lc = args.layer_chunk or 4
        s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
        events, wires = {}, {}
        if me.kind == "P":
            peers = {q: d_view(q) for q in my_q}
            S = w.src_lays[me.tp_rank]
        else:
            peers = {p: kvx.Layout.from_dict(
                synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, w.NB_p, cfg.src_dtype, cfg.p_order))
                for p in my_p}
        for k, other in peers.items():
            sl, dl = (S, other) if me.kind == "P" else (other, w.dst_lays[me.tp_rank])
            nb = max(kvx.wire_bytes(sl, dl, cfg.total_tokens, (l0, min(cfg.L, l0 + lc))) for l0 in range(0, cfg.L, lc))
            for b in range(2):
                wires[(k, b)] = torch.empty(nb, dtype=torch.uint8, device=dev)

        def step(ev=None):
            st = torch.cuda.Event()
            st.record(stream)
            s_a.wait_event(st)
            s_b.wait_event(st)
            if ev is not None:
                ev[0].record(stream)
            if me.kind == "P":
                tr.nccl_send_step(comm, w.src_lays[me.tp_rank], w.src_pools[me.tp_rank], w.src_bt, peers,
                                  {q: n_p + q for q in peers}, wires, lc, s_a, s_b, events)
            elif me.kind == "D":
                tr.nccl_recv_step(comm, peers, w.dst_lays[me.tp_rank], w.dst_pools[me.tp_rank], w.dst_bt,
                                  {p: p for p in peers}, wires, lc, s_a, s_b, events)
            for s_ in (s_a, s_b):
                e = torch.cuda.Event()
                e.record(s_)
                stream.wait_event(e)
            if ev is not None:
                ev[1].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    K = args.steps
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    kvx.launch_count_reset()
    barrier()
    t0.record(stream)
    for i in range(K):
        step(kev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = kvx.launch_count()
    clk = clocks.stop()
    barrier()
    my_ms = t0.elapsed_time(t1)
    mover = "D" if args.mode == "pull" else "P"   # the rank whose stream runs the data-path kernels
    kts = [a.elapsed_time(b) for a, b in kev] if me.kind == mover else [0.0]
    kern_ms = statistics.mean(kts)
    if int(err.item()):
        raise SystemExit(f"rank {rank}: flag wait timed out")
    # busiest link: P egress = bytes it sends, D ingress = bytes it receives (wire dtype = dst)
    nvl_in = w.dst_bytes([0]) if me.kind == "D" else 0
    nvl_out = sum(w.dst_bytes([0]) * (len([1 for p2, q2, _, _ in pairs if q2 == q and p2 == me.tp_rank])) //
                  max(1, len([1 for p2, q2, _, _ in pairs if q2 == q])) for q in my_q) if me.kind == "P" else 0
    stats = {"ms": my_ms, "kern_ms": kern_ms, "kern_med": statistics.median(kts), "kern_min": min(kts),
             "launches": launches, "kind": me.kind, "nvl": max(nvl_in, nvl_out),
             "kernel": kvx.last_kernel(),
             "clk": clk}
    parity = None
    if not args.no_parity and me.kind == "D":
        if dyn:   # decode the received codes with the scales P shipped
            w.dst_dicts[me.tp_rank]["scales"] = w.scales[me.tp_rank].cpu().numpy().reshape(cfg.L, 2, -1)
        parity = parity_multi(cfg, w, me, my_p, dev, dyn)
    e2e = None
    if not args.no_e2e and args.mode in ("push", "pull"):
        e2e = e2e_multi(w, me, step, stream, barrier, err, min(K, 3), rank)
    allx = tr.exchange({"stats": stats, "parity": parity, "e2e": e2e})
    if rank == 0:
        sts = [x["stats"] for x in allx]
        max_ms = max(x["ms"] for x in sts)
        ms = max_ms / K
        mover = "D" if args.mode == "pull" else "P"
        kms = max(x["kern_ms"] for x in sts if x["kind"] == mover)
        src_b = w.src_bytes(range(n_p))
        nvl_b = max(x["nvl"] for x in sts)
        achieved = nvl_b / (ms * 1e-3) / 1e9
        full = n_p == cfg.tp_p and n_d == cfg.tp_d
        out = {
            "metric": METRIC, "value": round(src_b / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "ms_per_request": round(ms / len(cfg.n_tokens), 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": _dtype_name(cfg),
            "data": "synthetic (seeded random finite bit patterns, Fisher-Yates block tables, pow2 fp8 scales)",
            "config": {"workload": f"{wl_name}: {cfg.note}; P ranks 0..{n_p - 1} on GPUs 0..{n_p - 1}, D ranks "
                                   f"0..{n_d - 1} on GPUs {n_p}..{n_p + n_d - 1}"
                                   + (" (full transfer)" if full else " (per-GPU-equivalent sub-config)")
                                   + (f", {world - n_p - n_d} idle GPU(s)" if world > n_p + n_d else ""),
                       "mode": args.mode + (" + dynamic fp8 scales (P amax per chunk, shipped)" if dyn else ""),
                       "layer_chunk": lc, "requests": len(cfg.n_tokens),
                       "tokens": cfg.total_tokens, "overrides": _overrides(args), "src_bytes_per_step": src_b,
                       "busiest_link_bytes_per_step": nvl_b, "pairs": [list(x[:2]) for x in pairs],
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"P TP{cfg.tp_p} x D TP{cfg.tp_d}, {n_p}+{n_d} ranks present"},
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_MEASURED_GBS,
                         "unit": "GB/s", "frac": round(achieved / NVLINK_MEASURED_GBS, 4),
                         "traffic": _traffic(f"{wl_name}:{args.mode}"),
                         "kernel": f"{[x['kernel'] for x in sts if x['kind'] == 'P'][0]} (peer-store push)"
                         if args.mode == "push"
                         else f"{[x['kernel'] for x in sts if x['kind'] == 'D'][0]} (peer-load pull on D)"
                         if args.mode == "pull"
                         else "pack + ncclSend/Recv + unpack (whole P step)",
                         "kernel_ms": round(kms, 4),
                         "kernel_ms_median": round(max(x["kern_med"] for x in sts if x["kind"] == mover), 4),
                         "kernel_ms_min": round(max(x["kern_min"] for x in sts if x["kind"] == mover), 4),
                         "algorithmic_bytes_per_step": nvl_b,
                         "note": "busiest GPU link (P egress or D ingress) bytes / step time",
                         "peak_source": "measured peer copy 770 GB/s/direction (B200_PROFILING.md)",
                         "frac_vs_nominal_900": round(achieved / NVLINK_NOMINAL_GBS, 4)},
            "clocks": sts[0]["clk"], "clocks_all_ranks": [x["clk"].get("reasons") for x in sts],
            "gpu_launches": int(sum(x["launches"] for x in sts)),
            "parity": [x["parity"] for x in allx if x["parity"] is not None],
        }
        es = [x["e2e"] for x in allx if x["e2e"] is not None]
        if es:
            ms_e = max(e["ms"] for e in es) / es[0]["steps"]
            out["e2e"] = {"value": round(src_b / (ms_e * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms_e, 3),
                          "h2d_bytes_per_step": int(sum(e["h2d"] for e in es)),
                          "d2h_bytes_per_step": int(sum(e["d2h"] for e in es)), "steps": es[0]["steps"]}
        print(json.dumps(out), flush=True)
    barrier()
    dist.destroy_process_group()


def e2e_multi(w, me, step, stream, barrier, err, ke, rank):
    """Same metric through the public API with host buffers: every step the P rank uploads
    its source pool from pinned memory before pushing, the D rank reads its pool back."""
    import torch
    host = None
    if me.kind == "P":
        host = _pinned_copy(w.src_pools[me.tp_rank])
    elif me.kind == "D":
        host = torch.empty(w.dst_pools[me.tp_rank].numel(), dtype=torch.uint8, pin_memory=True)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ke):
        if me.kind == "P":
            w.src_pools[me.tp_rank].copy_(host, non_blocking=True)
        step()
        if me.kind == "D":
            host.copy_(w.dst_pools[me.tp_rank], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    if int(err.item()):
        raise SystemExit(f"rank {rank}: flag wait timed out (e2e)")
    return {"ms": e0.elapsed_time(e1), "steps": ke, "h2d": host.numel() if me.kind == "P" else 0,
            "d2h": host.numel() if me.kind == "D" else 0}


def parity_multi(cfg, w, me, my_p, dev, dyn=False):
    """D rank: regenerate its P sources' pools from their seeds on this GPU and check a
    sample of the received pool against the oracle.  dyn: the fp8 scales were computed and
    shipped by P -- also check them against O1's amax scales over every request for the
    sampled layers."""
    import torch
    import paper_2509_17542_b200 as kvx
    q = me.tp_rank
    for p in my_p:
        d = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, w.NB_p, cfg.src_dtype, cfg.p_order)
        pool = kvx.Layout.from_dict(d).new_pool(dev)
        view = pool.view(torch.uint8 if synth.NBYTES[cfg.src_dtype] == 1 else torch.int16)
        synth.fill_random_finite_(view, cfg.seed + 100 + p, cfg.src_dtype)
        w.src_dicts[p], w.src_pools[p] = d, pool
    ok, det = sample_parity(w, (0, 2), 0, my_p, [q])
    det["rank"] = f"D{q}"
    if dyn:
        from oracle import o1
        ids = [b for t in w.src_tables for b in t]
        lays, pools = [], []
        for p in my_p:
            a, nd = extract(w.src_pools[p], w.src_dicts[p], (0, 2), ids)
            lays.append(nd)
            pools.append(a)
        k, tabs = 0, []
        for t in w.src_tables:
            tabs.append(list(range(k, k + len(t))))
            k += len(t)
        dd = dict(w.dst_dicts[q])
        dd["L"], dd["scales"] = 2, None
        want = o1.amax_scales(lays, pools, dd, cfg.n_tokens, tabs)
        got = np.asarray(w.dst_dicts[q]["scales"])[0:2]
        det["dynamic_scales_ok"] = bool(np.array_equal(got, want))
        det["dynamic_scales_sample"] = "O1 amax/448 over all requests, layers [0,2)"
        ok = ok and det["dynamic_scales_ok"]
    for p in my_p:
        del w.src_pools[p]
    return {"ok": ok, **det}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = synth.configs()[args.workload or ("c2" if world == 1 else "c4")]
    nl = args.cpu_sample_layers or 2
    p_ranks = list(range(cfg.tp_p)) if world == 1 else [0]
    d_ranks = list(range(cfg.tp_d)) if world == 1 else [0]
    for _ in range(max(args.warmup, 0)):
        cpu_baseline(cfg, 1, p_ranks, d_ranks)
    tot_b, tot_t = 0, 0.0
    for _ in range(args.steps):
        b, t = cpu_baseline(cfg, nl, p_ranks, d_ranks)
        tot_b += b
        tot_t += t
    v = tot_b / tot_t / 1e9
    sample = (f"O1 (plain C, 1 thread) per step: {cfg.name} request 0, layers [0,{nl}) of {cfg.L}, "
              f"P ranks {p_ranks} -> D ranks {d_ranks}")
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "GB/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype_name(cfg),
           "data": "synthetic", "config": {"workload": f"{cfg.name}: {cfg.note} (oracle on host, bounded sample)"},
           "cpu_baseline": {"value": round(v, 5), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(v, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_stream(args):
    """c5: mixed-length request stream (T ~ logU[512, 32k], 64 requests) from two P instances
    (TP2 each, requests alternate A/B) to one D instance (TP4), per-layer pipelined push.
    N GPUs: N/2 P ranks (instances A, B; ranks 0.. of each) and N/2 D ranks (0..N/2-1); N=8 is
    the full c5, N=4 its per-GPU-equivalent sub-config c5' (A0 + B0 -> D0, D1).  Every request
    is ready at t=0 and pushed in order, one fused convert launch per (request, layer chunk)
    covering all of the P rank's D peers; per-request completion is a release flag."""
    import dataclasses
    import torch
    import torch.distributed as dist
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import transfer as tr
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = synth.configs()["c5"]
    n_p = n_d = world // 2
    n_inst = 2 if n_p >= 2 else 1
    per_inst = n_p // n_inst
    inst_req = [list(range(i, len(cfg.n_tokens), 2)) for i in range(n_inst)]
    is_p = rank < n_p
    d_ranks = list(range(n_d))
    stream = torch.cuda.current_stream()
    K = args.steps
    # D side: one pool for all requests of both instances; flags[p_world] = requests landed
    d_cfg = cfg
    NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    dst_tables = synth.block_tables(cfg.seed + 2, cfg.n_tokens, cfg.B_d, NB_d)
    flags = torch.zeros(max(n_p, 1) * 8, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    mine = None
    pull = args.mode == "pull"

    def inst_setup(inst):
        """P rank tables / layout of instance `inst` (rebuilt from the seeds on D in pull mode)."""
        reqs = inst_req[inst]
        icfg = dataclasses.replace(cfg, n_tokens=[cfg.n_tokens[r] for r in reqs], seed=cfg.seed + 10 * inst)
        NB_p = synth.pool_capacity(icfg.n_tokens, cfg.B_p)
        return reqs, icfg, NB_p, synth.block_tables(icfg.seed + 1, icfg.n_tokens, cfg.B_p, NB_p)

    if pull:
        if is_p:
            inst, p = rank // per_inst, rank % per_inst
            reqs, icfg, NB_p, src_tables = inst_setup(inst)
            sd = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, NB_p, cfg.src_dtype, cfg.p_order)
            spool = kvx.Layout.from_dict(sd).new_pool(dev)
            synth.fill_random_finite_(spool.view(torch.int16), icfg.seed + 100 + p, cfg.src_dtype)
            mine = {"kind": "P", "r": rank, "pool": kvx.ipc_export(spool), "flags": kvx.ipc_export(flags)}
        else:
            q = rank - n_p
            dd = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, NB_d, cfg.dst_dtype, cfg.d_order)
            dl = kvx.Layout.from_dict(dd)
            pool = dl.new_pool(dev, fill=synth.CANARY)
            mine = {"kind": "D", "r": q, "flags": kvx.ipc_export(flags)}
    elif not is_p:
        q = rank - n_p
        dd = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, NB_d, cfg.dst_dtype, cfg.d_order)
        dl = kvx.Layout.from_dict(dd)
        pool = dl.new_pool(dev, fill=synth.CANARY)
        mine = {"q": q, "pool": kvx.ipc_export(pool), "flags": kvx.ipc_export(flags)}
    allx = tr.exchange(mine)
    peers = {e["q"]: e for e in allx if e is not None and "q" in e}
    src_bytes = 0
    lat = []
    if pull and is_p:
        # my KV is resident: release it to the D ranks, then wait until they have read it
        d_flag = {e["r"]: kvx.ipc_open(*e["flags"]) + 4 * rank for e in allx if e["kind"] == "D"}
        pairs = tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={p}, d_ranks=set(d_ranks))
        qs = [q for _, q, _, _ in pairs]
        src_bytes = sum(cfg.L * 2 * cfg.D * (cfg.H // cfg.tp_p) * synth.NBYTES[cfg.src_dtype] * t
                        for t in icfg.n_tokens)
        count = [0]

        def step(evs=None):
            count[0] += 1
            for q in qs:
                kvx.signal(d_flag[q], count[0], stream)
            for q in qs:
                kvx.wait(flags[q:q + 1], count[0], err, 60.0, stream)
        expected_per_step = 0
    elif pull:
        # D rank q: pull every request, in order, from the P rank of its instance holding q's heads
        srcs = [pr for pr in range(n_p) if any(qq == q for _, qq, _, _ in
                                               tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={pr % per_inst}))]
        p_ent = {e["r"]: e for e in allx if e["kind"] == "P"}
        src_pool = {pr: kvx.ipc_open(*p_ent[pr]["pool"]) for pr in srcs}
        p_flag = {pr: kvx.ipc_open(*p_ent[pr]["flags"]) + 4 * q for pr in srcs}
        order = []   # (source P world rank, its layout, src Batch, dst Batch) per request, stream order
        setups = {inst: inst_setup(inst) for inst in range(n_inst)}
        for r in range(len(cfg.n_tokens)):
            inst = r % n_inst if n_inst > 1 else 0
            reqs, icfg, NB_p, src_tables = setups[inst]
            i = reqs.index(r)
            pr = [x for x in srcs if x // per_inst == inst][0]
            sl = kvx.Layout.from_dict(synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, pr % per_inst, cfg.B_p, NB_p,
                                                   cfg.src_dtype, cfg.p_order))
            order.append((pr, sl, kvx.Batch(sl, [icfg.n_tokens[i]], [src_tables[i]], dev),
                          kvx.Batch(dl, [cfg.n_tokens[r]], [dst_tables[r]], dev)))
        count = [0]
        # one stream per source P rank, each on its share of the SMs: D pulls the two
        # instances' requests concurrently, so no P rank's egress carries two D ranks at once
        side = {pr: torch.cuda.Stream() for pr in srcs}
        if len(srcs) > 1:
            kvx.set_sm_budget(torch.cuda.get_device_properties(dev).multi_processor_count // len(srcs))

        def step(evs=None):
            count[0] += 1
            st = torch.cuda.Event()
            st.record(stream)
            for pr in srcs:
                side[pr].wait_event(st)
                kvx.wait(flags[pr:pr + 1], count[0], err, 60.0, side[pr])
            for j, (pr, sl, sbt, dbt) in enumerate(order):
                kvx.convert_reshard([sl], [src_pool[pr]], sbt, [dl], [pool], dbt, None, side[pr])
                if evs is not None:
                    evs[j].record(side[pr])
            for pr in srcs:
                kvx.signal(p_flag[pr], count[0], side[pr])
                e = torch.cuda.Event()
                e.record(side[pr])
                stream.wait_event(e)
    elif is_p:
        inst, p = rank // per_inst, rank % per_inst
        reqs = inst_req[inst]
        icfg = dataclasses.replace(cfg, n_tokens=[cfg.n_tokens[r] for r in reqs], seed=cfg.seed + 10 * inst)
        NB_p = synth.pool_capacity(icfg.n_tokens, cfg.B_p)
        src_tables = synth.block_tables(icfg.seed + 1, icfg.n_tokens, cfg.B_p, NB_p)
        sd = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, NB_p, cfg.src_dtype, cfg.p_order)
        sl = kvx.Layout.from_dict(sd)
        spool = sl.new_pool(dev)
        synth.fill_random_finite_(spool.view(torch.int16), icfg.seed + 100 + p, cfg.src_dtype)
        pairs = tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={p}, d_ranks=set(d_ranks))
        qs = [q for _, q, _, _ in pairs]
        dls = [kvx.Layout.from_dict(synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, NB_d, cfg.dst_dtype,
                                                 cfg.d_order)) for q in qs]
        ppools = [kvx.ipc_open(*peers[q]["pool"]) for q in qs]
        pflags = [kvx.ipc_open(*peers[q]["flags"]) + 4 * rank for q in qs]
        # per-request tables (one Batch per request on each side)
        sbt = [kvx.Batch(sl, [icfg.n_tokens[i]], [src_tables[i]], dev) for i in range(len(reqs))]
        dbt = [kvx.Batch(dls[0], [cfg.n_tokens[r]], [dst_tables[r]], dev) for r in reqs]
        per_tok_layer = 2 * cfg.D * (cfg.H // cfg.tp_p) * synth.NBYTES[cfg.src_dtype]
        chunk_bytes = args.chunk_mib << 20
        chunks = [max(1, -(-chunk_bytes // (per_tok_layer * t))) for t in icfg.n_tokens]
        src_bytes = sum(cfg.L * per_tok_layer * t for t in icfg.n_tokens)
        count = [0]

        if args.c5_batch:  # the whole instance batch in one launch per layer chunk (no per-request handoff)
            sbt_all = kvx.Batch(sl, icfg.n_tokens, src_tables, dev)
            dbt_all = kvx.Batch(dls[0], [cfg.n_tokens[r] for r in reqs], [dst_tables[r] for r in reqs], dev)

        def step(evs=None):
            if args.c5_batch:
                lc = args.layer_chunk or cfg.L
                for l0 in range(0, cfg.L, lc):
                    kvx.convert_share(sl, spool, sbt_all, dls, ppools, dbt_all, (l0, min(cfg.L, l0 + lc)), stream)
                count[0] += len(reqs)
                for f in pflags:
                    kvx.signal(f, count[0], stream)
                if evs is not None:
                    for e in evs:
                        e.record(stream)
                return
            for i in range(len(reqs)):
                lc = args.layer_chunk or chunks[i]
                for l0 in range(0, cfg.L, lc):
                    kvx.convert_share(sl, spool, sbt[i], dls, ppools, dbt[i], (l0, min(cfg.L, l0 + lc)), stream)
                count[0] += 1
                for f in pflags:
                    kvx.signal(f, count[0], stream)
                if evs is not None:
                    evs[i].record(stream)
        expected_per_step = 0
    else:
        q = rank - n_p
        srcs = [pr for pr in range(n_p) if any(qq == q for _, qq, _, _ in
                                               tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={pr % per_inst}))]
        n_req_of = {pr: len(inst_req[pr // per_inst]) for pr in srcs}
        count = [0]

        def step(evs=None):
            count[0] += 1
            for pr in srcs:
                kvx.wait(flags[pr:pr + 1], count[0] * n_req_of[pr], err, 60.0, stream)
    barrier_t = torch.zeros(1, device=dev)
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    dist.all_reduce(barrier_t)
    torch.cuda.synchronize()
    if pull:   # the D ranks run the data path: per-request completion events there
        nreq_mine = len(cfg.n_tokens) if not is_p else 0
    else:
        nreq_mine = len(inst_req[rank // per_inst]) if is_p else 0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nreq_mine)] for _ in range(K)]
    clocks = ClockSampler(local)
    clocks.start()
    kvx.launch_count_reset()
    dist.all_reduce(barrier_t)
    t0.record(stream)
    for k in range(K):
        step(evs[k] if nreq_mine else None)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = kvx.launch_count()
    if int(err.item()):
        raise SystemExit(f"rank {rank}: flag wait timed out")
    my_ms = t0.elapsed_time(t1)
    if nreq_mine:
        # latency of request i in step k = its completion - the step's start (previous step end)
        prev = t0
        for k in range(K):
            for i in range(nreq_mine):
                lat.append(prev.elapsed_time(evs[k][i]))
            prev = max(evs[k], key=lambda e: t0.elapsed_time(e))  # the step's last completion
    info = tr.exchange({"ms": my_ms, "src_bytes": src_bytes, "lat": lat, "launches": launches,
                        "nreq": nreq_mine})
    if rank == 0:
        max_ms = max(x["ms"] for x in info)
        ms = max_ms / K
        tot_b = sum(x["src_bytes"] for x in info)
        nreq = len(cfg.n_tokens) if pull else sum(x["nreq"] for x in info) // max(per_inst, 1)
        alll = sorted(l for x in info for l in x["lat"])
        # NVLink roofline: the busiest D rank's ingress (all its heads of every request moved)
        # NVLink bytes (wire dtype, valid tokens): each present D rank's ingress, and each P
        # rank's egress to the present D ranks -- with unequal instance loads the busier P
        # rank's egress, not a D rank's ingress, is the bound
        per_head = 2 * cfg.L * cfg.D * min(synth.NBYTES[cfg.src_dtype], synth.NBYTES[cfg.dst_dtype])
        d_in = per_head * (cfg.H // cfg.tp_d) * sum(cfg.n_tokens[r] for i in range(n_inst) for r in inst_req[i])
        heads_out = sum(he - hb for pp, qq, hb, he in tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={0},
                                                                  d_ranks=set(d_ranks)))
        p_out = max(per_head * heads_out * sum(cfg.n_tokens[r] for r in inst_req[i]) for i in range(n_inst))
        busiest = max(d_in, p_out)
        t_roof = busiest / (NVLINK_MEASURED_GBS * 1e9) * 1e3
        out = {"metric": METRIC, "value": round(tot_b / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": world,
               "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3),
               "ms_per_request": round(ms / max(nreq, 1), 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": _dtype_name(cfg), "data": "synthetic (seeded)",
               "config": {"workload": f"c5 stream: {cfg.note}; {n_inst} P instance(s) x {per_inst} rank(s) -> "
                                      f"D ranks {d_ranks}" + (" (full c5)" if world == 8 else " (c5' sub-config)"),
                          "requests": nreq, "src_bytes_per_step": tot_b,
                          "mode": "pull per request (D-initiated NVLink reads, one launch per request)" if pull
                          else "push, whole instance batch per launch" if args.c5_batch else
                          f"push per request, layer chunks >= {args.chunk_mib} MiB",
                          "l2": "inputs larger than L2 (no flush)"},
               "latency_ms": {"p50": round(alll[len(alll) // 2], 3) if alll else None,
                              "p99": round(alll[min(len(alll) - 1, int(0.99 * len(alll)))], 3) if alll else None,
                              "note": "per request, from the step start, requests issued in order"},
               "roofline": {"bound": "nvlink", "achieved": round(busiest / (ms * 1e-3) / 1e9, 1),
                            "peak": NVLINK_MEASURED_GBS, "unit": "GB/s", "frac": round(t_roof / ms, 4),
                            "traffic": None,
                            "kernel": "k_convert_rows (peer-load pull on D, per request)" if pull
                            else "k_convert_rows (peer-store push, per request)",
                            "algorithmic_bytes_per_step": busiest, "d_ingress_bytes": d_in, "p_egress_bytes": p_out,
                            "note": "busiest GPU link (max of D ingress, P egress) / step time"},
               "clocks": clk, "gpu_launches": int(sum(x["launches"] for x in info))}
        print(json.dumps(out), flush=True)
    dist.all_reduce(barrier_t)
    torch.cuda.synchronize()
    dist.destroy_process_group()


def _json_only_stdout():
    """The driver reads ONE JSON line from stdout, but native libraries write to fd 1 too (NCCL
    prints its version banner on rank 0 when the first communicator comes up).  Point fd 1 at
    stderr and give Python's sys.stdout the original descriptor, so only our prints reach it."""
    sys.stdout.flush()
    keep = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(keep, "w", buffering=1)


def main():
    _json_only_stdout()
    args = parse()
    if args.impl != "reference":   # a fresh checkout has no libkvx.so yet (no-op when up to date)
        import __graft_entry__
        __graft_entry__._lib_builder().build()
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if args.workload == "c5":
            return run_stream(args)
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    main()
