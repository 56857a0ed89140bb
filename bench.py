#!/usr/bin/env python
"""bench.py -- KV transfer GB/s and ms/request (P -> D, device-timed) vs the HBM/NVLink
roofline, for the heterogeneous-compatible KV transmission path (arXiv 2509.17542, III-B).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode pull|push|nccl]

N = 1 (default): BASELINE configs[3], the north-star workload (c4: Llama-3-70B GQA KV, 32 x
  4096 tokens, P TP=4 -> D TP=4, bf16 -> fp8-e4m3 with per-head scales, block 16 -> 16, P
  layout NHD-per-layer -> D layout block-major HND), which fits one B200: all four P ranks'
  and all four D ranks' pools (71 GB) on cuda:0, one fused kv_convert_reshard launch per step
  (42.9 GB read + 21.5 GB written), HBM-bound.  `--workload c1|c2|c3` for the others.
N >= 2 (torchrun, one process per GPU): c4 as (P rank p -> D rank p) pairs on disjoint GPUs
  (P = ranks 0..N/2-1): N = 8 is the full c4, N = 2 / 4 its per-GPU-equivalent sub-configs
  (SURVEY 8(d)); per-pair work is fixed -> weak scaling.  `--workload c3|c2` runs the largest
  complete sub-transfer that fits (transfer.present_ranks); `--workload c5` the mixed-length
  stream.  Default mode "pull" (the paper's D-initiated read): D reads P's pool, or P's
  staging ring when the cast narrows, across NVLink; "push": P's fused kernel stores into D's
  pool; "nccl": pack -> ncclSend / ncclRecv -> unpack, per-layer pipelined.
  Before the transfer the ranks exchange layouts, block tables and fp8 scales through the
  control plane (transfer.ControlPlane, A3): each instance chooses its own tables; nothing is
  regenerated from the other side's seeds.

Verification on the measured buffers: the oracle O1 on a sample (N = 1: all of c1 / c2 / c3',
requests {first, last} of c4), and K6 (kv_verify_fill / kv_verify_check) over every element
of every D pool after one more transfer of a hash-coded fill.

One JSON line on rank 0 (contract in the task statement); `value` = logical source KV GB
(2*L*H*D*T*bytes_src over all requests and present P ranks) / max-over-ranks device time.
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

METRIC = "KV transfer GB/s and ms/request (P→D, device-timed) vs HBM/NVLink roofline"  # BASELINE.json verbatim
NVLINK_NOMINAL_GBS = 900.0    # north_star: 900 GB/s per direction (the roofline denominator)
K6_SEED = 0x6B36


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="pull", choices=["push", "pull", "nccl"])
    ap.add_argument("--ring-slots", type=int, default=3, help="pull mode, narrowing cast: staging ring depth")
    ap.add_argument("--dynamic-scales", action="store_true",
                    help="pull mode, fp8 destination: P computes per-chunk amax scales and ships them (NEXT-1 i)")
    ap.add_argument("--layer-chunk", type=int, default=0, help="layers per chunk (0 = whole model / auto)")
    ap.add_argument("--chunk-ramp", action="store_true",
                    help="staged pull: ramp the first three layer chunks up (negative layer_chunk, kv_chunk_count); "
                         "measured slower on the c4 pair, so off by default")
    ap.add_argument("--chunk-mib", type=int, default=64, help="c5: merge layers until a chunk moves this much")
    ap.add_argument("--c5-batch", action="store_true", help="c5: each instance's requests as one batch (no per-request handoff)")
    ap.add_argument("--c5-no-sm-split", action="store_true", help="c5 pull: the two source streams share all SMs")
    ap.add_argument("--c5-per-request-launch", action="store_true",
                    help="c5 pull: one launch per request (default: one launch per source with in-kernel per-request "
                         "completion words)")
    ap.add_argument("--requests", type=int, default=0,
                    help="use only the first N requests of the workload (e.g. 1: batch-1 latency of c3/c4)")
    ap.add_argument("--workload", default=None, help="override: c1..c5")
    ap.add_argument("--tokens", type=int, default=0, help="one request of this many tokens (paper points)")
    ap.add_argument("--tp-p", type=int, default=0, help="override the P TP degree")
    ap.add_argument("--tp-d", type=int, default=0, help="override the D TP degree")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the K6 full-size check")
    ap.add_argument("--no-nvlink-probe", action="store_true")
    ap.add_argument("--cpu-sample-layers", type=int, default=0)
    ap.add_argument("--oversubscribe", action="store_true",
                    help="N >= 2 validation on fewer GPUs: ranks share GPUs, gloo control plane (not a bench number)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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
# inputs (synth: seeded, no method arithmetic; device memory from torch)
# ------------------------------------------------------------------------------------
def p_tables(cfg, NB_p, contiguous=False):
    """The P instance's block tables (P's allocator; D learns them through the control plane)."""
    return synth.block_tables(cfg.seed + 1, cfg.n_tokens, cfg.B_p, NB_p, contiguous)


def d_tables(cfg, NB_d, contiguous=False):
    """The D instance's block tables (D picks its blocks; P learns them through the control plane)."""
    return synth.block_tables(cfg.seed + 2, cfg.n_tokens, cfg.B_d, NB_d, contiguous)


def make_p_rank(cfg, p, NB_p, dev):
    import torch
    import paper_2509_17542_b200 as kvx
    d = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_p, p, cfg.B_p, NB_p, cfg.src_dtype, cfg.p_order)
    lay = kvx.Layout.from_dict(d)
    pool = lay.new_pool(dev)
    synth.fill_random_finite_(pool.view(torch.uint8 if synth.NBYTES[cfg.src_dtype] == 1 else torch.int16),
                              cfg.seed + 100 + p, cfg.src_dtype)
    return d, lay, pool


def make_d_rank(cfg, q, NB_d, dev):
    import torch
    import paper_2509_17542_b200 as kvx
    sc_np = sc = None
    if cfg.dst_dtype in synth.FP8:
        sc_np = synth.pow2_scales(cfg.seed + 200 + q, cfg.L, cfg.H // cfg.tp_d)
        sc = torch.from_numpy(sc_np.reshape(-1).copy()).to(dev)
    d = synth.layout(cfg.L, cfg.H, cfg.D, cfg.tp_d, q, cfg.B_d, NB_d, cfg.dst_dtype, cfg.d_order, sc_np)
    lay = kvx.Layout.from_dict(d, sc)
    return d, lay, lay.new_pool(dev, fill=synth.CANARY), sc


def src_bytes(cfg, n_p=None):
    n = cfg.tp_p if n_p is None else n_p
    return 2 * cfg.L * (cfg.H // cfg.tp_p) * n * cfg.D * cfg.total_tokens * synth.NBYTES[cfg.src_dtype]


def dst_bytes(cfg, n_d=None):
    n = cfg.tp_d if n_d is None else n_d
    padded = sum(synth.blocks_for(t, cfg.B_d) * cfg.B_d for t in cfg.n_tokens)
    return 2 * cfg.L * (cfg.H // cfg.tp_d) * n * cfg.D * padded * synth.NBYTES[cfg.dst_dtype]


def extract(pool_t, d, layers, block_ids):
    """Compact host copy of a pool restricted to layers [lb, le) and the given blocks (same
    axis order) -> (numpy codes, layout dict).  Bench infrastructure (oracle input)."""
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
        nd["scales"] = np.asarray(d["scales"]).reshape(d["L"], 2, -1)[layers[0]:layers[1]]
    return a, nd


def sample_of(pool_t, d, tables, reqs, layers):
    """extract() of the blocks of requests `reqs` (in order) -> (codes, layout dict, local tables)."""
    ids = [b for r in reqs for b in tables[r]]
    a, nd = extract(pool_t, d, layers, ids)
    loc, k = [], 0
    for r in reqs:
        loc.append(list(range(k, k + len(tables[r]))))
        k += len(tables[r])
    return a, nd, loc


def o1_compare(src_samples, dst_samples, n_tokens, dst_dtype, threads=1):
    """O1 over sampled sources -> expected sampled D pools; compare with the device's.
    src_samples / dst_samples: [(codes, layout dict, local tables)].  threads > 1 splits the
    layers over host threads (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import o1
    o1.lib()
    L = dst_samples[0][1]["L"]
    want = []
    for g, nd, _ in dst_samples:
        w = np.frombuffer(bytes([synth.CANARY]) * g.nbytes, dtype=g.dtype).copy()
        want.append(w)
    args = ([s[1] for s in src_samples], [s[0] for s in src_samples], [s[1] for s in dst_samples], want, n_tokens,
            src_samples[0][2], dst_samples[0][2])
    t0 = time.perf_counter()
    ranges = [(i * L // threads, (i + 1) * L // threads) for i in range(threads)]
    ranges = [r for r in ranges if r[1] > r[0]]
    if len(ranges) <= 1:
        o1.convert(*args)
    else:
        with ThreadPoolExecutor(len(ranges)) as ex:
            list(ex.map(lambda lr: o1.convert(*args, lr), ranges))
    t_o1 = time.perf_counter() - t0
    bad = exact = n = maxulp = 0
    for (g, _, _), w in zip(dst_samples, want):
        n += g.size
        if dst_dtype == synth.E4M3:
            def ordv(x):
                x = x.astype(np.int32)
                return np.where(x & 0x80, -(x & 0x7F), x & 0x7F)
            nan_w, nan_g = (w & 0x7F) == 0x7F, (g & 0x7F) == 0x7F
            dd = np.abs(ordv(g) - ordv(w))
            dd[nan_w & nan_g] = 0
            dd[nan_w != nan_g] = 99
            maxulp = max(maxulp, int(dd.max(initial=0)))
            bad += int((dd > 1).sum())
            exact += int((g == w).sum())
        else:
            bad += int((g != w).sum())
            exact += int((g == w).sum())
    return {"ok": bad == 0, "elements": int(n), "mismatches": int(bad), "bit_exact": int(exact),
            "max_e4m3_ulp": maxulp if dst_dtype == synth.E4M3 else None, "o1_seconds": round(t_o1, 2),
            "o1_threads": threads}


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
    o = {k: getattr(args, k) for k in ("requests", "tokens", "tp_p", "tp_d") if getattr(args, k, 0)}
    return o or None


def _dtype_name(cfg):
    a, b = synth.DTYPE_NAMES[cfg.src_dtype], synth.DTYPE_NAMES[cfg.dst_dtype]
    return a if a == b else f"{a}->{b}"


def _traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture
    (profiles/traffic.json: "<workload>@1" single GPU, "<workload>:<mode>" NVLink modes)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(key)
    return None


_REGISTERED = []


def _pinned_empty(nbytes):
    """Page-locked host buffer of exactly nbytes (a numpy allocation registered with
    cudaHostRegister): torch's pinned allocator rounds every block up to a power of two, which
    would pin ~100 GB for c4's 71 GB of pools."""
    import torch
    arr = np.empty(max(int(nbytes), 1), dtype=np.uint8)
    rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister of {nbytes} bytes failed ({rc})")
    _REGISTERED.append(arr)
    return torch.from_numpy(arr)[:nbytes]


def _unpin_all():
    import torch
    torch.cuda.synchronize()
    while _REGISTERED:
        torch.cuda.cudart().cudaHostUnregister(_REGISTERED.pop().ctypes.data)


def _pinned_copy(dev_tensor):
    """Pinned host copy of a device tensor without a pageable intermediate (GB-sized pools)."""
    h = _pinned_empty(dev_tensor.numel() * dev_tensor.element_size())
    h.copy_(dev_tensor.view(-1).view(__import__("torch").uint8))
    return h


# ------------------------------------------------------------------------------------
# N = 1: the whole transfer on one GPU (HBM-bound fused convert)
# ------------------------------------------------------------------------------------
def run_single(args):
    import torch
    import paper_2509_17542_b200 as kvx
    torch.cuda.set_device(0)
    wl_name = args.workload or "c4"
    cfg = _subset(synth.configs()[wl_name], args)
    dev = torch.device("cuda", 0)
    NB_p, NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_p), synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    P = [make_p_rank(cfg, p, NB_p, dev) for p in range(cfg.tp_p)]
    Dr = [make_d_rank(cfg, q, NB_d, dev) for q in range(cfg.tp_d)]
    pt, dt_ = p_tables(cfg, NB_p), d_tables(cfg, NB_d)
    S, SP = [x[1] for x in P], [x[2] for x in P]
    Dl, DP = [x[1] for x in Dr], [x[2] for x in Dr]
    src_bt = kvx.Batch(S[0], cfg.n_tokens, pt, dev)
    dst_bt = kvx.Batch(Dl[0], cfg.n_tokens, dt_, dev)
    stream = torch.cuda.current_stream()
    lc = args.layer_chunk or cfg.L

    def step(ev=None):
        for l0 in range(0, cfg.L, lc):
            if ev is not None:
                ev[0].record(stream)
            kvx.convert_reshard(S, SP, src_bt, Dl, DP, dst_bt, (l0, min(cfg.L, l0 + lc)), stream)
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
    kernel = kvx.last_kernel()
    ms = t0.elapsed_time(t1) / K
    sb, db = src_bytes(cfg), dst_bytes(cfg)
    kts = [a.elapsed_time(b) for a, b in kev] if lc == cfg.L else [ms]
    kern_ms = statistics.mean(kts)
    peaks = load_peaks()
    alg = sb + db  # HBM read + write per launch
    achieved = alg / (kern_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(sb / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
        "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 5),
        "ms_per_request": round(ms / len(cfg.n_tokens), 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": _dtype_name(cfg),
        "data": "synthetic (seeded random finite bit patterns, Fisher-Yates block tables, power-of-two fp8 scales)",
        "config": {"workload": f"{wl_name} on one GPU: {cfg.note}; all {cfg.tp_p} P and {cfg.tp_d} D ranks' pools on "
                               f"cuda:0, one fused convert per step",
                   "requests": len(cfg.n_tokens), "tokens": cfg.total_tokens, "overrides": _overrides(args),
                   "layout": "P (L,KV,BLK,SLOT,H,D) -> D (BLK,L,KV,H,SLOT,D)",
                   "src_bytes_per_step": sb, "dst_bytes_per_step": db,
                   "l2": "inputs larger than L2 (no flush)", "parallelism": "none (1 GPU)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": _traffic(f"{wl_name}@1"),
                     "kernel": kernel, "kernel_ms": round(kern_ms, 5),
                     "kernel_ms_median": round(statistics.median(kts), 5), "kernel_ms_min": round(min(kts), 5),
                     "algorithmic_bytes_per_launch": alg, "peak_source": peaks["source"],
                     "frac_vs_nominal_8TBs": round(achieved / 8000.0, 4)},
        "clocks": clk, "gpu_launches": int(launches),
    }
    def guarded(key, fn):
        # a failing check or side measurement must not cost the timed line: record the error
        try:
            out[key] = fn()
        except Exception as e:  # noqa: BLE001
            out[key] = {"ok": False, "error": repr(e)[:500]}

    if not args.no_parity:
        guarded("parity", lambda: single_parity(cfg, P, Dr, pt, dt_, SP, DP, sb))
    if not args.no_verify:
        guarded("fullsize", lambda: k6_single(cfg, S, SP, src_bt, Dl, DP, dst_bt, step))
    if not args.no_e2e:
        guarded("e2e", lambda: e2e_single(cfg, P, Dr, pt, dt_, S, SP, src_bt, Dl, DP, dst_bt, min(K, 5), stream, sb))
    if not args.no_cpu_baseline:
        guarded("cpu_baseline", lambda: single_cpu_baseline(cfg, args, wl_name, out))
    print(json.dumps(out), flush=True)


def single_parity(cfg, P, Dr, pt, dt_, SP, DP, sb):
    """O1 on the measured buffers: every request when the whole batch is small (c1, c2, c3),
    else the first and the last request -- all layers, all ranks."""
    ncores = len(os.sched_getaffinity(0))
    reqs = list(range(len(cfg.n_tokens))) if sb <= (3 << 30) else sorted({0, len(cfg.n_tokens) - 1})
    ss = [sample_of(SP[p], P[p][0], pt, reqs, (0, cfg.L)) for p in range(cfg.tp_p)]
    ds = [sample_of(DP[q], Dr[q][0], dt_, reqs, (0, cfg.L)) for q in range(cfg.tp_d)]
    res = o1_compare(ss, ds, [cfg.n_tokens[r] for r in reqs], cfg.dst_dtype, threads=min(ncores, cfg.L))
    res["sample"] = (f"requests {reqs} of {len(cfg.n_tokens)} (all layers, all ranks) vs O1" if len(reqs) <
                     len(cfg.n_tokens) else f"all {len(reqs)} request(s), all layers, all ranks vs O1")
    return res


def single_cpu_baseline(cfg, args, wl_name, out):
    """The oracle timed on the host cores: one thread (returned) and split over all cores
    (stored as cpu_baseline_threads)."""
    # about 10-30 s of single-thread O1: c4 (fp8 cast) ~31 MB/s -> 24 layers of request 0
    nl = args.cpu_sample_layers or min(cfg.L, 24 if cfg.H * cfg.D * cfg.n_tokens[0] > (1 << 21) else 12)
    nb, dt = cpu_baseline(cfg, nl, range(cfg.tp_p), range(cfg.tp_d))
    cb = {"value": round(nb / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
          "cpu": cpu_model(),
          "sample": f"O1 (plain C, 1 thread) on {wl_name} request 0, layers [0,{nl}) of {cfg.L}, "
                    f"all ranks, {nb} source bytes in {dt:.2f} s"}
    ncores = len(os.sched_getaffinity(0))
    nl_mt = min(cfg.L, max(nl, 2 * ncores))
    nb2, dt2 = cpu_baseline(cfg, nl_mt, range(cfg.tp_p), range(cfg.tp_d), threads=ncores)
    out["cpu_baseline_threads"] = {"value": round(nb2 / dt2 / 1e9, 4), "unit": "GB/s", "cores": ncores,
                                   "kind": "oracle", "cpu": cpu_model(),
                                   "sample": f"same O1 split by layer over {ncores} threads, layers [0,{nl_mt}), "
                                             f"{nb2} source bytes in {dt2:.2f} s"}
    return cb


def k6_single(cfg, S, SP, src_bt, Dl, DP, dst_bt, step):
    """K6: hash-coded fill of every P pool, one more transfer, every element of every D pool
    checked (SURVEY 8(d) full-size verification; SPEC S:272 conservation)."""
    import torch
    import paper_2509_17542_b200 as kvx
    if cfg.src_dtype in synth.FP8:
        return {"ok": None, "note": "K6 does not cover fp8 sources"}
    dev = SP[0].device
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    for lay, pool in zip(S, SP):
        kvx.verify_fill(lay, pool, src_bt, Dl, K6_SEED, err)
    step()
    tot = [0] * 4
    for lay, pool in zip(Dl, DP):
        res = torch.zeros(8, dtype=torch.int64, device=dev)
        scratch = torch.empty(lay.num_blocks, dtype=torch.uint8, device=dev)
        kvx.verify_check(S[0], lay, pool, dst_bt, K6_SEED, res, scratch)
        r = [int(x) for x in res.cpu()]
        tot = [a + b for a, b in zip(tot, r[:4])]
    ok = int(err.item()) == 0 and tot[0] == tot[1] == tot[2] == 0
    return {"ok": ok, "elements_checked": tot[3], "value_mismatches": tot[0], "tail_mismatches": tot[1],
            "canary_mismatches": tot[2], "fill_error": int(err.item()),
            "what": "K6: hash-coded fill of every valid P element, one more transfer, every element of every D pool "
                    "(valid = hash code, tail = 0, unused blocks = canary)"}


def _block_view(pool, d):
    """A pool as [outer, num_blocks, inner] int32 words (outer / inner: the axes before / after
    BLOCK in its order), for moving whole blocks."""
    import torch
    ext = {synth.LAYER: d["L"], synth.KV: 2, synth.BLOCK: d["NB"], synth.SLOT: d["B"], synth.HEAD: d["H"] // d["tp"],
           synth.DIM: d["D"]}
    order = d["order"]
    bi = order.index(synth.BLOCK)
    outer = int(np.prod([ext[a] for a in order[:bi]])) if bi else 1
    inner = int(np.prod([ext[a] for a in order[bi + 1:]])) * synth.NBYTES[d["dtype"]]
    assert inner % 4 == 0
    return pool.view(torch.uint8).view(torch.int32).view(outer, d["NB"], inner // 4)


def e2e_single(cfg, P, Dr, pt, dt_, S, SP, src_bt, Dl, DP, dst_bt, K, stream, sb):
    """Same metric through the public API with HOST buffers: every step moves the batch's
    blocks of the P pools up from pinned memory and its D blocks back, inside the timed
    region -- only the blocks the block tables name (the pools' ~10% free blocks stay put):
    H2D into a device staging copy, scattered into the pools by block id, the convert, then
    the D blocks gathered and read back.  Both directions are pipelined by layer chunk
    where the pools' orders allow it (P layer-major: the upload; D block-then-layer: the
    read-back): chunk k+1 crosses PCIe up while chunk k converts and chunk k-1 goes down,
    each staging chunk guarded by its own events (no step-wide barriers)."""
    import torch
    import paper_2509_17542_b200 as kvx
    dev = SP[0].device
    p_ids = torch.as_tensor(sorted({b for t in pt for b in t}), dtype=torch.long, device=dev)
    d_ids = torch.as_tensor(sorted({b for t in dt_ for b in t}), dtype=torch.long, device=dev)
    pv = [_block_view(pool, P[i][0]) for i, pool in enumerate(SP)]
    dv = [_block_view(pool, Dr[i][0]) for i, pool in enumerate(DP)]
    # pinned host copies of exactly the batch's blocks; device staging of the same shape
    hs, stage_p = [], []
    for v in pv:
        comp = v.index_select(1, p_ids)
        h = _pinned_empty(comp.numel() * 4).view(torch.int32).view(comp.shape)
        h.copy_(comp)
        hs.append(h)
        stage_p.append(comp)
    p_lay = cfg.p_order[0] == synth.LAYER and cfg.p_order[1] == synth.KV
    d_lay = cfg.d_order[0] == synth.BLOCK and cfg.d_order[1] == synth.LAYER
    n_ch = int(os.environ.get("KVX_E2E_CHUNKS", "8")) if (p_lay or d_lay) else 1
    bounds = [(i * cfg.L // n_ch, (i + 1) * cfg.L // n_ch) for i in range(n_ch)]
    # D read-back chunks: [1, blocks, layer-chunk words] slices of the block view (D_ORDER:
    # BLOCK then LAYER outermost), or one whole-step chunk
    d_words = [v.shape[2] for v in dv]
    d_cuts = [(l0 * w // cfg.L, l1 * w // cfg.L) for w in d_words for l0, l1 in bounds] if d_lay else None
    stage_d, hd = [], []
    for i, v in enumerate(dv):
        parts = [(a, b) for a, b in (d_cuts[i * n_ch:(i + 1) * n_ch] if d_lay else [(0, d_words[i])])]
        sd = [torch.empty((v.shape[0], len(d_ids), b - a), dtype=torch.int32, device=dev) for a, b in parts]
        stage_d.append((parts, sd))
        hd.append([_pinned_empty(x.numel() * 4).view(torch.int32).view(x.shape) for x in sd])
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    ev_up, ev_scat = [ev() for _ in bounds], [ev() for _ in bounds]
    nd = n_ch if d_lay else 1
    ev_gath, ev_down = [ev() for _ in range(nd)], [ev() for _ in range(nd)]
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    up.wait_stream(stream)
    down.wait_stream(stream)

    def read_back(j, step):
        if step:   # the previous step's D2H of staging chunk j has left it
            stream.wait_event(ev_down[j])
        for (parts, sd), v in zip(stage_d, dv):
            a, b = parts[j]
            torch.index_select(v[:, :, a:b], 1, d_ids, out=sd[j])
        ev_gath[j].record(stream)
        down.wait_event(ev_gath[j])
        with torch.cuda.stream(down):
            for (_, sd), h in zip(stage_d, hd):
                h[j].copy_(sd[j], non_blocking=True)
        ev_down[j].record(down)

    for step in range(K):
        for c, (l0, l1) in enumerate(bounds):
            r0, r1 = (2 * l0, 2 * l1) if p_lay else (0, pv[0].shape[0])
            if p_lay or c == 0:
                if step:   # the previous step's scatter of this staging chunk is done
                    up.wait_event(ev_scat[c])
                with torch.cuda.stream(up):
                    for st_, h in zip(stage_p, hs):
                        st_[r0:r1].copy_(h[r0:r1], non_blocking=True)
                ev_up[c].record(up)
                stream.wait_event(ev_up[c])
                for v, st_ in zip(pv, stage_p):
                    v[r0:r1].index_copy_(1, p_ids, st_[r0:r1])
                ev_scat[c].record(stream)
            kvx.convert_reshard(S, SP, src_bt, Dl, DP, dst_bt, (l0, l1), stream)
            if d_lay:
                read_back(c, step)
        if not d_lay:
            read_back(0, step)
    stream.wait_stream(down)
    stream.wait_stream(up)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / K
    h2d = int(sum(h.numel() * 4 for h in hs))
    d2h = int(sum(x.numel() * 4 for hl in hd for x in hl))
    del hs, hd, stage_p, stage_d
    _unpin_all()
    return {"value": round(sb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": K, "pipelined": f"{len(bounds)} layer chunks: upload, convert and read-back overlapped "
                                     "chunk by chunk; only the batch's blocks cross PCIe (device staging + "
                                     "block scatter / gather)"}


# ------------------------------------------------------------------------------------
# N >= 2: P -> D across NVLink
# ------------------------------------------------------------------------------------
def nvlink_probe(me, my_peer, dev, tr, kvx, barrier, nbytes=1 << 30):
    """In-run NVLink ceiling: 1 GiB copy-engine copies between each P rank and
    its first D peer, all pairs at once -- D reading P's buffer (the pull direction) and P
    writing D's buffer (the push direction).  Returns GB/s per direction (median of 3, this
    rank)."""
    import torch
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev) if me.kind in "PD" else None
    if buf is not None:
        buf.fill_(1)
    allx = tr.exchange({"kind": me.kind, "r": me.tp_rank, "h": kvx.ipc_export(buf) if buf is not None else None})
    peer = None
    if me.kind in "PD" and my_peer is not None:
        other = "D" if me.kind == "P" else "P"
        ent = [e for e in allx if e["kind"] == other and e["r"] == my_peer][0]
        peer = (kvx.ipc_open(*ent["h"]), ent["h"][1])
    s = torch.cuda.current_stream()
    out = {}
    for name, who, fn in (("ce_read", "D", lambda: kvx.memcpy_engine(buf, peer[0], nbytes, s)),
                          ("ce_write", "P", lambda: kvx.memcpy_engine(peer[0], buf, nbytes, s))):
        ts = []
        for i in range(4):
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if me.kind == who and peer is not None:
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1))
        if me.kind == who and peer is not None:
            out[name] = round(nbytes / (statistics.median(ts) * 1e-3) / 1e9, 1)
    torch.cuda.synchronize()
    barrier()
    if peer is not None:
        kvx.ipc_close(*peer)
    return out


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
    local, barrier_t = _init_dist(args, local)
    dev = torch.device("cuda", local)
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
    NB_p, NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_p), synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    stream = torch.cuda.current_stream()

    def barrier():
        dist.all_reduce(barrier_t)

    # ---- my side: only my instance's layout, pool, tables (and D's scales) ----
    mine = {}
    if me.kind == "P":
        d, lay, pool = make_p_rank(cfg, me.tp_rank, NB_p, dev)
        tabs = p_tables(cfg, NB_p)
        mine = dict(d=d, lay=lay, pool=pool, tables=tabs, bt=kvx.Batch(lay, cfg.n_tokens, tabs, dev))
        cp = tr.ControlPlane(me, lay, None, cfg.n_tokens, tabs, batch_id=1)
    elif me.kind == "D":
        d, lay, pool, sc = make_d_rank(cfg, me.tp_rank, NB_d, dev)
        tabs = d_tables(cfg, NB_d)
        mine = dict(d=d, lay=lay, pool=pool, tables=tabs, scales=sc, bt=kvx.Batch(lay, cfg.n_tokens, tabs, dev))
        cp = tr.ControlPlane(me, lay, None if sc is None else sc.cpu().numpy(), cfg.n_tokens, tabs, batch_id=1)
    else:
        cp = tr.ControlPlane(me)
    # ---- the peers, as the control plane delivered them ----
    peer_lays, peer_bt = {}, None
    if me.kind == "P":
        peer_lays = {q: cp.layout("D", q, dev) for q in my_q}   # D's scales on P's GPU: the sender casts
        peer_bt = cp.batch("D", peer_lays[my_q[0]], dev)
    elif me.kind == "D":
        peer_lays = {p: cp.layout("P", p, dev) for p in my_p}
        peer_bt = cp.batch("P", peer_lays[my_p[0]], dev)
    ctrl_info = {"bytes_received": cp.bytes_received, "messages": len(cp.msgs)}
    nvl = {}
    if not args.no_nvlink_probe:
        peer_of = my_q[0] if me.kind == "P" else my_p[0] if me.kind == "D" else None
        nvl = nvlink_probe(me, peer_of, dev, tr, kvx, barrier)

    flags = torch.zeros(max(n_p, 1), dtype=torch.int32, device=dev)  # one word per P source
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    epoch = [0]
    lc = args.layer_chunk or cfg.L
    dyn = False
    S = mine.get("lay")
    if args.mode == "push":
        ch = tr.PushChannel(me, mine.get("pool") if me.kind == "D" else None, flags if me.kind == "D" else None)

        def step(ev=None):
            epoch[0] += 1
            if me.kind == "P":
                if ev is not None:
                    ev[0].record(stream)
                tr.push_step(S, mine["pool"], mine["bt"], peer_lays, ch.peer_pool, peer_bt, ch.peer_flag, epoch[0],
                             lc, stream, flag_slot=me.tp_rank)
                if ev is not None:
                    ev[1].record(stream)
            elif me.kind == "D":
                for p in my_p:
                    kvx.wait(flags[p:p + 1], epoch[0], err, 30.0, stream)
    elif args.mode == "pull":
        # D-initiated read: D maps P's pool (or P's staging ring when the cast narrows)
        narrowing = synth.NBYTES[cfg.dst_dtype] < synth.NBYTES[cfg.src_dtype]
        R = max(1, args.ring_slots)
        if narrowing and not args.layer_chunk:
            # ~40 MiB of wire per chunk, at most 20 chunks (c4 full batch: 4 layers per chunk;
            # one request: 4 chunks of 20 layers), so the pipeline fill stays small and
            # per-chunk launch costs on P stay hidden behind D's reads
            # (profiles/r01/batch1_chunks_c4_n2.jsonl)
            pair_wire = 2 * cfg.L * min(cfg.H // cfg.tp_p, cfg.H // cfg.tp_d) * cfg.D * \
                synth.NBYTES[cfg.dst_dtype] * cfg.total_tokens
            n_ch = min(20, max(1, round(pair_wire / (40 << 20))))
            lc = -(-cfg.L // n_ch)
        ring, slot_bytes, ring_ptrs = None, 0, []
        dyn = args.dynamic_scales and narrowing and synth.NBYTES[cfg.src_dtype] > 1
        if me.kind == "P" and narrowing:
            slot_bytes = max(kvx.wire_bytes(S, peer_lays[q], cfg.total_tokens, (l0, min(cfg.L, l0 + lc)))
                             for q in my_q for l0 in range(0, cfg.L, lc))
            slot_bytes = (slot_bytes + 255) // 256 * 256
            ring = torch.empty(len(my_q) * R * slot_bytes, dtype=torch.uint8, device=dev)
            ring_ptrs = [ring.data_ptr() + (i * R + b) * slot_bytes for i in range(len(my_q)) for b in range(R)]
        pflags = torch.zeros(max(n_p, n_d, 1), dtype=torch.int32, device=dev)
        pch = tr.PullChannel(me, pflags, pool=mine["pool"] if me.kind == "P" and not narrowing else None,
                             ring=ring, ring_dst=my_q if ring is not None else (), ring_slots=R, slot_bytes=slot_bytes,
                             scales=mine.get("scales") if dyn and me.kind == "D" else None)
        if me.kind == "D" and narrowing:
            slot_bytes = min(pch.slot_bytes[p] for p in my_p)
        # --chunk-ramp: the timed step ramps its first chunks (negative layer_chunk,
        # kv_chunk_count); the e2e step stages whole uniform chunks range by range, so both
        # sides use uniform chunks there
        lc_ramp = -lc if args.chunk_ramp else lc
        counters = torch.zeros(max(kvx.pull_counter_words((0, cfg.L), x) for x in (lc, lc_ramp)), dtype=torch.int32,
                               device=dev)
        seq = [0]

        def step(ev=None, pre=None, uniform=False):
            """pre (e2e, narrowing pull, P side): (ranges, fn) -- stage the layer ranges one
            after the other (same chunk numbering as one call), fn(l0, l1) enqueued before each
            (its host upload), so the upload of range k+1 overlaps the transfer of range k.
            uniform (the e2e steps, both sides): uniform layer chunks instead of the ramp."""
            lcx = lc if uniform or pre else lc_ramp
            nchunks = kvx.chunk_count((0, cfg.L), lcx)
            epoch[0] += 1
            if ev is not None and me.kind == "D":
                ev[0].record(stream)
            if me.kind == "P":
                if narrowing:
                    s0 = seq[0]
                    for l0, l1 in (pre[0] if pre else [(0, cfg.L)]):
                        if pre:
                            pre[1](l0, l1)
                        kvx.stage(S, mine["pool"], mine["bt"], [peer_lays[q] for q in my_q], ring_ptrs, R,
                                  slot_bytes, [pch.peer_flag[q] for q in my_q], [pflags[q:q + 1] for q in my_q], s0,
                                  err, (l0, l1), lcx, 30.0, stream,
                                  peer_scales=[pch.peer_scales[q] for q in my_q] if dyn else None)
                        s0 += kvx.chunk_count((l0, l1), lcx)
                else:
                    for q in my_q:   # my KV is resident: D may read it; then wait until it has
                        kvx.signal(pch.peer_flag[q], epoch[0], stream)
                    for q in my_q:
                        kvx.wait(pflags[q:q + 1], epoch[0], err, 30.0, stream)
            elif me.kind == "D":
                if narrowing:
                    kvx.pull_staged([peer_lays[p] for p in my_p], [a for p in my_p for a in pch.src_ring[p]], R,
                                    slot_bytes, S, mine["pool"], mine["bt"], [pflags[p:p + 1] for p in my_p],
                                    [pch.peer_flag[p] for p in my_p], seq[0], err, (0, cfg.L), lcx, 30.0, stream,
                                    counters=counters)
                else:
                    kvx.pull([peer_lays[p] for p in my_p], [pch.src_pool[p] for p in my_p], peer_bt, S,
                             mine["pool"], mine["bt"], [pflags[p:p + 1] for p in my_p],
                             [pch.peer_flag[p] for p in my_p], epoch[0], err, (0, cfg.L), lc, 30.0, stream)
            seq[0] += nchunks
            if ev is not None and me.kind == "D":
                ev[1].record(stream)
        step.chunked_upload = (narrowing, lc)
    else:
        # NCCL baseline: pack -> ncclSend / ncclRecv -> unpack, per-layer double-buffered
        uid = [kvx.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = kvx.Comm(world, rank, uid[0], local)
        lc = args.layer_chunk or 4
        s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
        wires = {}
        for k, other in peer_lays.items():
            sl, dl = (S, other) if me.kind == "P" else (other, S)
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
                tr.nccl_send_step(comm, S, mine["pool"], mine["bt"], peer_lays, {q: n_p + q for q in peer_lays},
                                  wires, lc, s_a, s_b)
            elif me.kind == "D":
                tr.nccl_recv_step(comm, peer_lays, S, mine["pool"], mine["bt"], {p: p for p in peer_lays}, wires, lc,
                                  s_a, s_b)
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
    # busiest link: P egress = bytes it sends, D ingress = bytes it receives (wire dtype = the narrower)
    w_b = min(synth.NBYTES[cfg.src_dtype], synth.NBYTES[cfg.dst_dtype])
    per_head = 2 * cfg.L * cfg.D * cfg.total_tokens * w_b
    nvl_in = per_head * (cfg.H // cfg.tp_d) if me.kind == "D" else 0
    nvl_out = sum(per_head * (he - hb) for p, q, hb, he in pairs if me.kind == "P" and p == me.tp_rank)
    stats = {"ms": my_ms, "kern_ms": kern_ms, "kern_med": statistics.median(kts), "kern_min": min(kts),
             "launches": launches, "kind": me.kind, "nvl": max(nvl_in, nvl_out), "kernel": kvx.last_kernel(),
             "clk": clk, "nvlink_probe": nvl}
    # ---- oracle sample on the measured buffers: P ships request 0, layers [0, 2) of its pool ----
    parity = None
    if not args.no_parity:
        samp = None
        if me.kind == "P":
            samp = sample_of(mine["pool"], mine["d"], mine["tables"], [0], (0, min(2, cfg.L)))
            if dyn and cfg.tp_p <= cfg.tp_d:   # O1's amax scales of D heads (all held here), every request
                from oracle import o1
                allr = list(range(len(cfg.n_tokens)))
                a, nd, loc = sample_of(mine["pool"], mine["d"], mine["tables"], allr, (0, min(2, cfg.L)))
                want_sc = {}
                for q in my_q:
                    dd = dict(cp.message("D", q).desc)
                    dd["L"], dd["scales"] = min(2, cfg.L), None
                    want_sc[q] = o1.amax_scales([nd], [a], dd, cfg.n_tokens, loc)
                samp = samp + (want_sc,)
        allsamp = tr.exchange({"kind": me.kind, "r": me.tp_rank, "samp": samp})
        if me.kind == "D":
            srcs = {e["r"]: e["samp"] for e in allsamp if e["kind"] == "P" and e["r"] in my_p}
            dd = dict(mine["d"])
            if dyn:   # decode the received codes with the scales P shipped
                dd["scales"] = mine["scales"].cpu().numpy().reshape(cfg.L, 2, -1)
            ds = sample_of(mine["pool"], dd, mine["tables"], [0], (0, min(2, cfg.L)))
            parity = o1_compare([srcs[p][:3] for p in my_p], [ds], [cfg.n_tokens[0]], cfg.dst_dtype)
            parity["sample"] = f"request 0, layers [0,{min(2, cfg.L)}), P ranks {my_p} -> D{me.tp_rank} (P's sample " \
                               "shipped over the control plane)"
            if dyn and cfg.tp_p <= cfg.tp_d:
                got = dd["scales"][:min(2, cfg.L)]
                Hd = cfg.H // cfg.tp_d
                okd = True
                for p in my_p:   # each P rank computed the heads it holds
                    hb = max(p * (cfg.H // cfg.tp_p), me.tp_rank * Hd) - me.tp_rank * Hd
                    he = min((p + 1) * (cfg.H // cfg.tp_p), (me.tp_rank + 1) * Hd) - me.tp_rank * Hd
                    okd = okd and bool(np.array_equal(got[:, :, hb:he], srcs[p][3][me.tp_rank][:, :, hb:he]))
                parity["dynamic_scales_ok"] = okd
                parity["ok"] = parity["ok"] and okd
            parity["rank"] = f"D{me.tp_rank}"
    # ---- K6 over every element of every D pool (static scales) ----
    fullsize = None
    if not args.no_verify and not dyn:
        kerr = torch.zeros(1, dtype=torch.int32, device=dev)
        if me.kind == "P":
            kvx.verify_fill(S, mine["pool"], mine["bt"], [peer_lays[q] for q in my_q], K6_SEED, kerr)
        torch.cuda.synchronize()
        barrier()
        step()
        torch.cuda.synchronize()
        barrier()
        if me.kind == "D":
            res = torch.zeros(8, dtype=torch.int64, device=dev)
            scratch = torch.empty(S.num_blocks, dtype=torch.uint8, device=dev)
            kvx.verify_check(peer_lays[my_p[0]], S, mine["pool"], mine["bt"], K6_SEED, res, scratch)
            r = [int(x) for x in res.cpu()]
            fullsize = {"rank": f"D{me.tp_rank}", "elements_checked": r[3], "value_mismatches": r[0],
                        "tail_mismatches": r[1], "canary_mismatches": r[2]}
        elif me.kind == "P":
            fullsize = {"rank": f"P{me.tp_rank}", "fill_error": int(kerr.item())}
        if int(err.item()):
            raise SystemExit(f"rank {rank}: flag wait timed out (K6 step)")
    e2e = None
    if not args.no_e2e and args.mode in ("push", "pull"):
        e2e = e2e_multi(mine, me, step, stream, barrier, err, min(K, 5), rank, cfg.L)
    allx = tr.exchange({"stats": stats, "parity": parity, "e2e": e2e, "fullsize": fullsize, "ctrl": ctrl_info})
    if rank == 0:
        sts = [x["stats"] for x in allx]
        max_ms = max(x["ms"] for x in sts)
        ms = max_ms / K
        kms = max(x["kern_ms"] for x in sts if x["kind"] == mover)
        sb = src_bytes(cfg, n_p)
        nvl_b = max(x["nvl"] for x in sts)
        achieved = nvl_b / (ms * 1e-3) / 1e9
        full = n_p == cfg.tp_p and n_d == cfg.tp_d
        probes = [x["nvlink_probe"] for x in sts if x["nvlink_probe"]]
        meas = {k: round(statistics.mean([p[k] for p in probes if k in p]), 1)
                for k in ("ce_read", "ce_write") if any(k in p for p in probes)}
        ref_key = "ce_read" if args.mode == "pull" else "ce_write"
        fs = [x["fullsize"] for x in allx if x["fullsize"] is not None]
        fs_ok = None
        if fs:
            fs_ok = all(f.get("fill_error", 0) == 0 and f.get("value_mismatches", 0) == 0 and
                        f.get("tail_mismatches", 0) == 0 and f.get("canary_mismatches", 0) == 0 for f in fs)
        out = {
            "metric": METRIC, "value": round(sb / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "ms_per_request": round(ms / len(cfg.n_tokens), 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": _dtype_name(cfg),
            "data": "synthetic (seeded random finite bit patterns, Fisher-Yates block tables, pow2 fp8 scales)",
            "config": {"workload": f"{wl_name}: {cfg.note}; P ranks 0..{n_p - 1} on GPUs 0..{n_p - 1}, D ranks "
                                   f"0..{n_d - 1} on GPUs {n_p}..{n_p + n_d - 1}"
                                   + (" (full transfer)" if full else " (per-GPU-equivalent sub-config)")
                                   + (f", {world - n_p - n_d} idle GPU(s)" if world > n_p + n_d else ""),
                       "mode": args.mode + (" + dynamic fp8 scales (P amax per chunk, shipped)" if dyn else ""),
                       "layer_chunk": lc,
                       "chunks": (kvx.chunk_count((0, cfg.L), -lc if args.chunk_ramp else lc)
                                  if args.mode == "pull" and narrowing else None),
                       "requests": len(cfg.n_tokens),
                       "tokens": cfg.total_tokens, "overrides": _overrides(args), "src_bytes_per_step": sb,
                       "busiest_link_bytes_per_step": nvl_b, "pairs": [list(x[:2]) for x in pairs],
                       "control_plane": "layouts, block tables and fp8 scales exchanged as kv_ctrl messages "
                                        f"({allx[0]['ctrl']['bytes_received']} B)",
                       "l2": "inputs larger than L2 (no flush)",
                       "oversubscribed": (f"{world} ranks on {torch.cuda.device_count()} GPUs: validation of the "
                                          "N-rank path, not a bench number") if args.oversubscribe else None,
                       "parallelism": f"P TP{cfg.tp_p} x D TP{cfg.tp_d}, {n_p}+{n_d} ranks present"},
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_NOMINAL_GBS,
                         "unit": "GB/s", "frac": round(achieved / NVLINK_NOMINAL_GBS, 4),
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
                         "note": "busiest GPU link (P egress or D ingress) user bytes / step time",
                         "peak_source": "nominal NVLink 5, 900 GB/s per direction (north_star)",
                         "measured_in_run_gbs": meas or None,
                         "frac_vs_measured_copy_engine": round(achieved / meas[ref_key], 4) if ref_key in meas
                         else None},
            "clocks": sts[0]["clk"], "clocks_all_ranks": [x["clk"].get("reasons") for x in sts],
            "gpu_launches": int(sum(x["launches"] for x in sts)),
            "parity": [x["parity"] for x in allx if x["parity"] is not None],
            "fullsize": {"ok": fs_ok, "ranks": fs} if fs else None,
        }
        es = [x["e2e"] for x in allx if x["e2e"] is not None]
        if es:
            ms_e = max(e["ms"] for e in es) / es[0]["steps"]
            out["e2e"] = {"value": round(sb / (ms_e * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms_e, 3),
                          "h2d_bytes_per_step": int(sum(e["h2d"] for e in es)),
                          "d2h_bytes_per_step": int(sum(e["d2h"] for e in es)), "steps": es[0]["steps"]}
        print(json.dumps(out), flush=True)
    barrier()
    dist.destroy_process_group()


def e2e_multi(mine, me, step, stream, barrier, err, ke, rank, L=None):
    """Same metric through the public API with host buffers: every step the P rank uploads its
    batch's blocks from pinned memory (staging + scatter by block id) before the transfer, the
    D rank gathers its batch's blocks and reads them back -- only the blocks the tables name.
    Narrowing pull (the default c4 path): the P rank uploads layer range by layer range on a
    copy stream and stages each range as soon as it is resident (kv_stage per range, one
    chunk numbering), so PCIe and NVLink overlap; the D rank gathers on its transfer stream
    and reads back on a side stream, so its next pull does not wait for PCIe."""
    import torch
    host = stage = view = ids = None
    if me.kind in ("P", "D"):
        dev = mine["pool"].device
        ids = torch.as_tensor(sorted({b for t in mine["tables"] for b in t}), dtype=torch.long, device=dev)
        view = _block_view(mine["pool"], mine["d"])
        stage = view.index_select(1, ids)
        host = _pinned_empty(stage.numel() * 4).view(torch.int32).view(stage.shape)
        if me.kind == "P":
            host.copy_(stage)
    narrowing, lc = getattr(step, "chunked_upload", (False, 0))
    pre = None
    if me.kind == "P" and narrowing and L and tuple(mine["d"]["order"][:2]) == (synth.LAYER, synth.KV):
        nck = -(-L // lc)
        per = max(1, -(-nck // 8)) * lc          # ~8 upload ranges, each whole chunks
        ranges = [(l0, min(L, l0 + per)) for l0 in range(0, L, per)]
        up = torch.cuda.Stream()
        ev_up = [torch.cuda.Event() for _ in ranges]
        ev_sc = [torch.cuda.Event() for _ in ranges]
        first = [True]
        idx = {r: i for i, r in enumerate(ranges)}

        def upload(l0, l1):
            i = idx[(l0, l1)]
            if not first[0]:
                up.wait_event(ev_sc[i])       # the previous step's scatter of this range is done
            with torch.cuda.stream(up):
                stage[2 * l0:2 * l1].copy_(host[2 * l0:2 * l1], non_blocking=True)
            ev_up[i].record(up)
            stream.wait_event(ev_up[i])
            view[2 * l0:2 * l1].index_copy_(1, ids, stage[2 * l0:2 * l1])
            ev_sc[i].record(stream)
            if i == len(ranges) - 1:
                first[0] = False
        pre = (ranges, upload)
    down, ev_d = torch.cuda.Stream(), None
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    down.wait_stream(stream)
    for _ in range(ke):
        if me.kind == "P" and pre is None:
            stage.copy_(host, non_blocking=True)
            view.index_copy_(1, ids, stage)
        if pre is not None:
            step(pre=pre)
        elif getattr(step, "chunked_upload", None):
            step(uniform=True)   # the same uniform chunks P stages range by range
        else:
            step()
        if me.kind == "D":
            # gather on the transfer stream (the next step overwrites the pool), read back on a
            # side stream so the next step's pull does not wait for PCIe
            if ev_d is not None:
                stream.wait_event(ev_d)      # the previous read-back has left the staging buffer
            torch.index_select(view, 1, ids, out=stage)
            ev_g = torch.cuda.Event()
            ev_g.record(stream)
            down.wait_event(ev_g)
            with torch.cuda.stream(down):
                host.copy_(stage, non_blocking=True)
            ev_d = torch.cuda.Event()
            ev_d.record(down)
    if pre is not None:
        stream.wait_stream(up)
    if me.kind == "D":
        stream.wait_stream(down)
    e1.record(stream)
    torch.cuda.synchronize()
    if int(err.item()):
        raise SystemExit(f"rank {rank}: flag wait timed out (e2e)")
    n = host.numel() * 4 if host is not None else 0
    del host, stage
    _unpin_all()
    return {"ms": e0.elapsed_time(e1), "steps": ke, "h2d": n if me.kind == "P" else 0,
            "d2h": n if me.kind == "D" else 0, "pipelined": pre is not None}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = synth.configs()[args.workload or "c4"]
    nl = args.cpu_sample_layers or 2
    p_ranks = list(range(cfg.tp_p)) if world == 1 else [0]
    d_ranks = list(range(cfg.tp_d)) if world == 1 else [0]
    if world > 1 and cfg.tp_p != cfg.tp_d:
        p_ranks, d_ranks = list(range(cfg.tp_p)), list(range(cfg.tp_d))
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
           "cpu_baseline": {"value": round(v, 5), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                            "cpu": cpu_model()},
           "e2e": {"value": round(v, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_stream(args):
    """c5: mixed-length request stream (T ~ logU[512, 32k], 64 requests) from two P instances
    (TP2 each, requests alternate A/B) to one D instance (TP4), per-request transfers.  N GPUs:
    N/2 P ranks (instances A, B; ranks 0.. of each) and N/2 D ranks (0..N/2-1); N=8 is the full
    c5, N=4 its per-GPU-equivalent sub-config c5' (A0 + B0 -> D0, D1).  Every request is ready
    at t=0 and moved in order; per-request completion is a release flag (push) or a
    completion event on D (pull).  The transfer plan (who feeds whom, which flag word) is
    transfer.StreamPlan; tables and layouts travel through the control plane."""
    import dataclasses
    import torch
    import torch.distributed as dist
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import transfer as tr
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    local, barrier_t = _init_dist(args, local)
    dev = torch.device("cuda", local)
    cfg = synth.configs()["c5"]
    plan = tr.StreamPlan(world, cfg.tp_p, cfg.tp_d, cfg.H, len(cfg.n_tokens))
    me = plan.role(rank)
    stream = torch.cuda.current_stream()
    K = args.steps
    NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    flags = torch.zeros(plan.flag_words, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    pull = args.mode == "pull"
    # ---- my side ----
    if me.kind == "P":
        reqs = plan.requests_of(me.inst)
        icfg = dataclasses.replace(cfg, n_tokens=[cfg.n_tokens[r] for r in reqs], seed=cfg.seed + 10 * me.inst)
        NB_p = synth.pool_capacity(icfg.n_tokens, cfg.B_p)
        d, lay, pool = make_p_rank(icfg, me.tp_rank, NB_p, dev)
        tabs = p_tables(icfg, NB_p)
        cp = tr.ControlPlane(tr.Role("P", plan.p_index(me.inst, me.tp_rank), rank), lay, None, icfg.n_tokens, tabs)
    else:
        d, lay, pool, _ = make_d_rank(cfg, me.tp_rank, NB_d, dev)
        tabs = d_tables(cfg, NB_d)
        cp = tr.ControlPlane(tr.Role("D", me.tp_rank, rank), lay, None, cfg.n_tokens, tabs)
    # ---- data-plane maps (CUDA IPC) ----
    exp = {"kind": me.kind, "r": rank, "flags": kvx.ipc_export(flags)}
    if (me.kind == "P") == pull:
        exp["pool"] = kvx.ipc_export(pool)
    allx = tr.exchange(exp)
    ent = {e["r"]: e for e in allx}
    maps = []

    def opn(h):
        a = kvx.ipc_open(*h)
        maps.append((a, h[1]))
        return a
    lat = []
    src_b = 0
    if me.kind == "P":
        qs = plan.d_peers(rank)
        src_b = sum(cfg.L * 2 * cfg.D * (cfg.H // cfg.tp_p) * synth.NBYTES[cfg.src_dtype] * t for t in icfg.n_tokens)
        count = [0]
        d_flag = {q: opn(ent[plan.d_world(q)]["flags"]) + 4 * plan.flag_word(rank) for q in qs}
        if pull:
            def step(evs=None):
                # my KV is resident: release it to the D ranks, then wait until they have read it
                count[0] += 1
                for q in qs:
                    kvx.signal(d_flag[q], count[0], stream)
                for q in qs:
                    kvx.wait(flags[plan.flag_word(plan.d_world(q)):plan.flag_word(plan.d_world(q)) + 1], count[0],
                             err, 60.0, stream)
        else:
            dls = [cp.layout("D", q, dev) for q in qs]
            ppools = [opn(ent[plan.d_world(q)]["pool"]) for q in qs]
            n_d_tok, d_tabs = cp.tables("D")
            sbt = [kvx.Batch(lay, [icfg.n_tokens[i]], [tabs[i]], dev) for i in range(len(reqs))]
            dbt = [kvx.Batch(dls[0], [cfg.n_tokens[r]], [d_tabs[r]], dev) for r in reqs]
            per_tok_layer = 2 * cfg.D * (cfg.H // cfg.tp_p) * synth.NBYTES[cfg.src_dtype]
            chunk_bytes = args.chunk_mib << 20
            chunks = [max(1, -(-chunk_bytes // (per_tok_layer * t))) for t in icfg.n_tokens]
            if args.c5_batch:
                sbt_all = kvx.Batch(lay, icfg.n_tokens, tabs, dev)
                dbt_all = kvx.Batch(dls[0], [cfg.n_tokens[r] for r in reqs], [d_tabs[r] for r in reqs], dev)

            def step(evs=None):
                if args.c5_batch:
                    lc = args.layer_chunk or cfg.L
                    for l0 in range(0, cfg.L, lc):
                        kvx.convert_share(lay, pool, sbt_all, dls, ppools, dbt_all, (l0, min(cfg.L, l0 + lc)), stream)
                    count[0] += len(reqs)
                    for q in qs:
                        kvx.signal(d_flag[q], count[0], stream)
                    if evs is not None:
                        for e in evs:
                            e.record(stream)
                    return
                for i in range(len(reqs)):
                    lc = args.layer_chunk or chunks[i]
                    for l0 in range(0, cfg.L, lc):
                        kvx.convert_share(lay, pool, sbt[i], dls, ppools, dbt[i], (l0, min(cfg.L, l0 + lc)), stream)
                    count[0] += 1
                    for q in qs:
                        kvx.signal(d_flag[q], count[0], stream)
                    if evs is not None:
                        evs[i].record(stream)
    else:
        srcs = plan.p_sources(rank)                    # world ranks of the P ranks feeding me
        count = [0]
        if pull:
            src_pool = {pr: opn(ent[pr]["pool"]) for pr in srcs}
            p_flag = {pr: opn(ent[pr]["flags"]) + 4 * plan.flag_word(rank) for pr in srcs}
            order = []   # (source P world rank, its layout, src Batch, dst Batch) per request, stream order
            for r in range(len(cfg.n_tokens)):
                inst = plan.inst_of(r)
                pr = [x for x in srcs if plan.role(x).inst == inst][0]
                pidx = plan.p_index(inst, plan.role(pr).tp_rank)
                sl = cp.layout("P", pidx, dev)
                _, ptabs = cp.message("P", pidx).n_tokens, cp.message("P", pidx).tables
                i = plan.requests_of(inst).index(r)
                order.append((pr, sl, kvx.Batch(sl, [cfg.n_tokens[r]], [ptabs[i]], dev),
                              kvx.Batch(lay, [cfg.n_tokens[r]], [tabs[r]], dev)))
            notify = not args.c5_batch and not args.c5_per_request_launch
            if args.c5_batch or notify:   # one launch per source P rank over all of its instance's requests
                order = []
                for pr in srcs:
                    inst = plan.role(pr).inst
                    pidx = plan.p_index(inst, plan.role(pr).tp_rank)
                    sl = cp.layout("P", pidx, dev)
                    m = cp.message("P", pidx)
                    rq = plan.requests_of(inst)
                    order.append((pr, sl, kvx.Batch(sl, m.n_tokens, m.tables, dev),
                                  kvx.Batch(lay, [cfg.n_tokens[r] for r in rq], [tabs[r] for r in rq], dev)))
            # one stream per source P rank, each on its share of the SMs: D pulls the two
            # instances' requests concurrently, so no P rank's egress carries two D ranks at once
            side = {pr: torch.cuda.Stream() for pr in srcs}
            if len(srcs) > 1 and not args.c5_no_sm_split:
                kvx.set_sm_budget(torch.cuda.get_device_properties(dev).multi_processor_count // len(srcs))
            if notify:   # per-request completion words and times, one row per step
                n_steps = max(args.warmup, 1) + K + 2
                nrq = {pr: len(plan.requests_of(plan.role(pr).inst)) for pr in srcs}
                ncnt = {pr: torch.zeros(nrq[pr], dtype=torch.int32, device=dev) for pr in srcs}
                nflg = {pr: torch.zeros(nrq[pr], dtype=torch.int32, device=dev) for pr in srcs}
                nns = {pr: torch.zeros((n_steps, nrq[pr]), dtype=torch.int64, device=dev) for pr in srcs}
                tst = torch.zeros(n_steps, dtype=torch.int64, device=dev)

            def step(evs=None):
                count[0] += 1
                if notify:
                    kvx.timestamp(tst[count[0]:count[0] + 1], stream)
                st = torch.cuda.Event()
                st.record(stream)
                for pr in srcs:
                    side[pr].wait_event(st)
                    kvx.wait(flags[plan.flag_word(pr):plan.flag_word(pr) + 1], count[0], err, 60.0, side[pr])
                for j, (pr, sl, sbt, dbt) in enumerate(order):
                    if notify:   # requests handed off one by one as they land, inside one launch
                        kvx.convert_reshard_notify([sl], [src_pool[pr]], sbt, [lay], [pool], dbt, ncnt[pr], nflg[pr],
                                                   count[0], nns[pr][count[0]], None, side[pr])
                    else:
                        kvx.convert_reshard([sl], [src_pool[pr]], sbt, [lay], [pool], dbt, None, side[pr])
                    if evs is not None:
                        evs[j].record(side[pr])
                for pr in srcs:
                    kvx.signal(p_flag[pr], count[0], side[pr])
                    e = torch.cuda.Event()
                    e.record(side[pr])
                    stream.wait_event(e)
        else:
            n_req_of = {pr: len(plan.requests_of(plan.role(pr).inst)) for pr in srcs}

            def step(evs=None):
                count[0] += 1
                for pr in srcs:
                    kvx.wait(flags[plan.flag_word(pr):plan.flag_word(pr) + 1], count[0] * n_req_of[pr], err, 60.0,
                             stream)
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    dist.all_reduce(barrier_t)
    torch.cuda.synchronize()
    notify = pull and me.kind == "D" and not args.c5_batch and not args.c5_per_request_launch
    step0 = count[0]   # steps run so far (warm-up): the timed steps are step0 + 1 .. step0 + K
    if pull:   # the D ranks run the data path: per-request completion events there
        nreq_mine = 0 if notify else (len(order) if args.c5_batch else len(cfg.n_tokens)) if me.kind == "D" else 0
    else:
        nreq_mine = len(plan.requests_of(me.inst)) if me.kind == "P" else 0
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
    if notify:
        # in-kernel completion times (%globaltimer) of every request - the step's start stamp
        ts = tst.cpu().tolist()
        for pr in srcs:
            rows = nns[pr].cpu().tolist()
            for k in range(step0 + 1, step0 + K + 1):
                lat += [(v - ts[k]) * 1e-6 for v in rows[k]]
        nreq_mine = len(cfg.n_tokens)
    # ---- K6 over every element of every D pool ----
    fullsize = None
    if not args.no_verify:
        kerr = torch.zeros(1, dtype=torch.int32, device=dev)
        if me.kind == "P":
            rid = torch.tensor(plan.requests_of(me.inst), dtype=torch.int32, device=dev)
            bt_all = kvx.Batch(lay, icfg.n_tokens, tabs, dev)
            dl = [cp.layout("D", q, dev) for q in plan.d_peers(rank)]
            kvx.verify_fill(lay, pool, bt_all, dl, K6_SEED, kerr, req_ids=rid)
        torch.cuda.synchronize()
        dist.all_reduce(barrier_t)
        step()
        torch.cuda.synchronize()
        dist.all_reduce(barrier_t)
        if me.kind == "D":
            res = torch.zeros(8, dtype=torch.int64, device=dev)
            scratch = torch.empty(lay.num_blocks, dtype=torch.uint8, device=dev)
            sl = cp.layout("P", 0, dev)
            kvx.verify_check(sl, lay, pool, kvx.Batch(lay, cfg.n_tokens, tabs, dev), K6_SEED, res, scratch)
            r = [int(x) for x in res.cpu()]
            fullsize = {"rank": f"D{me.tp_rank}", "elements_checked": r[3], "value_mismatches": r[0],
                        "tail_mismatches": r[1], "canary_mismatches": r[2]}
        else:
            fullsize = {"rank": f"P{plan.p_index(me.inst, me.tp_rank)}", "fill_error": int(kerr.item())}
    info = tr.exchange({"ms": my_ms, "src_bytes": src_b, "lat": lat, "launches": launches, "nreq": nreq_mine,
                        "fullsize": fullsize})
    if rank == 0:
        max_ms = max(x["ms"] for x in info)
        ms = max_ms / K
        tot_b = sum(x["src_bytes"] for x in info)
        nreq = len(cfg.n_tokens) if pull else sum(x["nreq"] for x in info) // max(plan.per_inst, 1)
        alll = sorted(v for x in info for v in x["lat"])
        # NVLink bytes (wire dtype, valid tokens): each present D rank's ingress, and each P
        # rank's egress to the present D ranks -- with unequal instance loads the busier P
        # rank's egress, not a D rank's ingress, is the bound
        per_head = 2 * cfg.L * cfg.D * min(synth.NBYTES[cfg.src_dtype], synth.NBYTES[cfg.dst_dtype])
        d_in = per_head * (cfg.H // cfg.tp_d) * sum(cfg.n_tokens[r] for i in range(plan.n_inst)
                                                   for r in plan.requests_of(i))
        heads_out = sum(he - hb for pp, qq, hb, he in tr.pair_plan(cfg.tp_p, cfg.tp_d, cfg.H, p_ranks={0},
                                                                  d_ranks=set(range(plan.n_d))))
        p_out = max(per_head * heads_out * sum(cfg.n_tokens[r] for r in plan.requests_of(i))
                    for i in range(plan.n_inst))
        busiest = max(d_in, p_out)
        t_roof = busiest / (NVLINK_NOMINAL_GBS * 1e9) * 1e3
        fs = [x["fullsize"] for x in info if x["fullsize"] is not None]
        fs_ok = all(f.get("fill_error", 0) == 0 and f.get("value_mismatches", 0) == 0 and
                    f.get("tail_mismatches", 0) == 0 and f.get("canary_mismatches", 0) == 0 for f in fs) if fs else None
        out = {"metric": METRIC, "value": round(tot_b / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": world,
               "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3),
               "ms_per_request": round(ms / max(nreq, 1), 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": _dtype_name(cfg), "data": "synthetic (seeded)",
               "config": {"workload": f"c5 stream: {cfg.note}; {plan.n_inst} P instance(s) x {plan.per_inst} "
                                      f"rank(s) -> D ranks {list(range(plan.n_d))}"
                                      + (" (full c5)" if world == 8 else " (c5' sub-config)"),
                          "requests": nreq, "src_bytes_per_step": tot_b,
                          "mode": ("pull, one launch per source P rank, each request handed off by an in-kernel "
                                   "completion word as it lands (kv_convert_reshard_notify)" if pull and
                                   not args.c5_batch and not args.c5_per_request_launch else
                                   "pull, whole instance batch per launch" if pull and args.c5_batch else
                                   "pull per request (D-initiated NVLink reads, one launch per request)") if pull
                          else "push, whole instance batch per launch" if args.c5_batch else
                          f"push per request, layer chunks >= {args.chunk_mib} MiB",
                          "control_plane": "layouts and block tables exchanged as kv_ctrl messages",
                          "oversubscribed": (f"{world} ranks on {torch.cuda.device_count()} GPUs: validation of the "
                                             "N-rank path, not a bench number") if args.oversubscribe else None,
                          "l2": "inputs larger than L2 (no flush)"},
               "latency_ms": {"p50": round(alll[len(alll) // 2], 3) if alll else None,
                              "p99": round(alll[min(len(alll) - 1, int(0.99 * len(alll)))], 3) if alll else None,
                              "note": "per request, from the step start, requests issued in order"},
               "roofline": {"bound": "nvlink", "achieved": round(busiest / (ms * 1e-3) / 1e9, 1),
                            "peak": NVLINK_NOMINAL_GBS, "unit": "GB/s", "frac": round(t_roof / ms, 4),
                            "traffic": None,
                            "kernel": "k_convert_rows (peer-load pull on D)" if pull
                            else "k_convert_rows (peer-store push, per request)",
                            "algorithmic_bytes_per_step": busiest, "d_ingress_bytes": d_in, "p_egress_bytes": p_out,
                            "peak_source": "nominal NVLink 5, 900 GB/s per direction (north_star)",
                            "note": "busiest GPU link (max of D ingress, P egress) / step time"},
               "clocks": clk, "gpu_launches": int(sum(x["launches"] for x in info)),
               "fullsize": {"ok": fs_ok, "ranks": fs} if fs else None}
        print(json.dumps(out), flush=True)
    dist.all_reduce(barrier_t)
    torch.cuda.synchronize()
    for a, o in maps:
        kvx.ipc_close(a, o)
    dist.destroy_process_group()


def _init_dist(args, local):
    """One process per GPU over NCCL (the contract).  --oversubscribe (validation of the
    N-rank host logic on fewer GPUs, e.g. world 8 on a 4-GPU box): ranks share GPUs -- rank r
    on GPU r // ceil(world / n_gpus), so the two ranks of a GPU play the same role -- and the
    control plane runs over gloo (NCCL refuses two ranks on one GPU).  Timings taken that way
    are not bench numbers.  Returns (device index, barrier tensor)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ["WORLD_SIZE"])
    if getattr(args, "oversubscribe", False):
        if args.mode == "nccl":
            raise SystemExit("--oversubscribe: the NCCL transport cannot run two ranks on one GPU")
        ndev = torch.cuda.device_count()
        per = -(-world // ndev)
        idx = local // per
        torch.cuda.set_device(idx)
        dist.init_process_group("gloo")
        return idx, torch.zeros(1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    return local, torch.zeros(1, device=dev)


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
