"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(kv_convert_reshard over the whole batch, one GPU holding the ranks' pools).

The oracle cannot redo GBs, so: (1) sampled outputs -- requests first / middle / last, a
few layers, all their blocks, compared element by element with O1 run on the extracted
source blocks; (2) properties that hold at any size -- every destination block outside
the batch's tables keeps its canary bytes, and every request's tail slots are zero."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _tail_and_canary(w, q):
    """Blocks outside every request's table keep 0xA5; tail slots of the last block are 0."""
    d = w.dst_dicts[q]
    nb = synth.NBYTES[d["dtype"]]
    tdt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[nb]
    ext = {synth.LAYER: d["L"], synth.KV: 2, synth.BLOCK: d["NB"], synth.SLOT: d["B"], synth.HEAD: d["H"] // d["tp"],
           synth.DIM: d["D"]}
    pool = w.dst_pools[q].view(tdt).view([ext[a] for a in d["order"]])
    bax = d["order"].index(synth.BLOCK)
    used = sorted(b for t in w.dst_tables for b in t)
    free = sorted(set(range(d["NB"])) - set(used))
    if free:
        fb = pool.index_select(bax, torch.as_tensor(free, device=pool.device))
        assert bool((fb.view(torch.uint8) == synth.CANARY).all()), "a block outside the tables was written"
    sax = d["order"].index(synth.SLOT)
    for r, T in enumerate(w.cfg.n_tokens):
        tail = T % d["B"]
        if tail:
            blk = pool.index_select(bax, torch.as_tensor([w.dst_tables[r][-1]], device=pool.device))
            slots = blk.index_select(sax, torch.arange(tail, d["B"], device=pool.device))
            assert bool((slots == 0).all()), f"request {r}: tail slots not zero"


@pytest.mark.parametrize("name,p_ranks,d_ranks,reqs", [
    ("c2", [0, 1], [0], [0]),
    ("c3", [0, 1], [0], [0, 7, 15]),
    ("c4", [0], [0], [0, 16, 31]),
    ("c5", [0], [0, 1], [0, 15, 31]),
])
def test_fullsize_sampled(name, p_ranks, d_ranks, reqs):
    import dataclasses
    import paper_2509_17542_b200 as kvx
    from bench import Workload, sample_parity
    cfg = synth.configs()[name]
    if name == "c5":  # one P instance (A) of the stream: even requests
        cfg = dataclasses.replace(cfg, n_tokens=cfg.n_tokens[0::2])
    w = Workload(cfg, p_ranks, d_ranks, torch.device("cuda", 0))
    kvx.convert_reshard([w.src_lays[p] for p in p_ranks], [w.src_pools[p] for p in p_ranks], w.src_bt,
                        [w.dst_lays[q] for q in d_ranks], [w.dst_pools[q] for q in d_ranks], w.dst_bt)
    torch.cuda.synchronize()
    L = cfg.L
    for r in reqs:
        for layers in ((0, 1), (L // 2, L // 2 + 1), (L - 1, L)):
            ok, det = sample_parity(w, layers, r, p_ranks, d_ranks)
            assert ok, det
    for q in d_ranks:
        _tail_and_canary(w, q)


def test_fullsize_vendor_layouts(o1):
    """c4 pair at full size (80 layers, 2 local heads, 32 x 4096 tokens, block 16, TP4 -> 4
    rank 0 -> 0) from an other-vendor P cache -- x-packed K pool ([LAYER], BLOCK, HEAD,
    D/8, SLOT, 8) and head_dim-major V pool ([LAYER], BLOCK, HEAD, DIM, SLOT) -- into the
    NVIDIA-style D pool (BLOCK, LAYER, KV, HEAD, SLOT, DIM), bf16 -> e4m3, in the two
    calls tools/variants_bench.py times (k_convert_tr8).  Sampled: requests 0 / 17 / 31 x
    layers 0 / 40 / 79, all their blocks, vs O1 on the extracted blocks; canary outside."""
    import paper_2509_17542_b200 as kvx
    from synth import BLOCK, DIM, HEAD, KV, LAYER, SLOT
    L, H, D, tp, B = 80, 8, 128, 4, 16
    Hl = H // tp
    n_tokens = [4096] * 32
    dev = torch.device("cuda", 0)
    NB = synth.pool_capacity(n_tokens, B)
    st = synth.block_tables(11, n_tokens, B, NB)
    dt_ = synth.block_tables(12, n_tokens, B, NB)
    dsc_np = synth.pow2_scales(6, L, Hl)
    dsc = torch.from_numpy(dsc_np).to(dev)
    vend = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)
    Kl = kvx.Layout(L, H, D, tp, 0, B, NB, synth.BF16, vend, None, kv_part=1, dim_split=8)
    Vl = kvx.Layout(L, H, D, tp, 0, B, NB, synth.BF16, vend, None, kv_part=2)
    Dl = kvx.Layout(L, H, D, tp, 0, B, NB, synth.E4M3, synth.D_ORDER, dsc)
    Kp, Vp = Kl.new_pool(dev), Vl.new_pool(dev)
    synth.fill_random_finite_(Kp.view(torch.int16), 40, synth.BF16)
    synth.fill_random_finite_(Vp.view(torch.int16), 41, synth.BF16)
    DP = Dl.new_pool(dev, fill=synth.CANARY)
    sbt = kvx.Batch(Kl, n_tokens, st, dev)
    dbt = kvx.Batch(Dl, n_tokens, dt_, dev)
    kvx.convert_reshard([Kl], [Kp], sbt, [Dl], [DP], dbt)
    assert kvx.last_kernel() == "k_convert_tr8"
    kvx.convert_reshard([Vl], [Vp], sbt, [Dl], [DP], dbt)
    assert kvx.last_kernel() == "k_convert_tr8"
    torch.cuda.synchronize()
    K6 = Kp.view(torch.int16).view(L, 1, NB, Hl, D // 8, B, 8)
    V6 = Vp.view(torch.int16).view(L, 1, NB, Hl, D, B)
    D6 = DP.view(torch.uint8).view(NB, L, 2, Hl, B, D)
    for r in (0, 17, 31):
        sb = torch.as_tensor(st[r], device=dev)
        db = torch.as_tensor(dt_[r], device=dev)
        nb = len(st[r])
        for l in (0, 40, 79):
            ksub = K6[l:l + 1].index_select(2, sb).cpu().numpy().reshape(-1)
            vsub = V6[l:l + 1].index_select(2, sb).cpu().numpy().reshape(-1)
            got = D6.index_select(0, db)[:, l:l + 1].cpu().numpy().reshape(-1)
            want = np.full(got.size, synth.CANARY, np.uint8)
            sl = lambda part, x: synth.layout(1, H, D, tp, 0, B, nb, synth.BF16, vend, kv_part=part, dim_split=x)
            dl = synth.layout(1, H, D, tp, 0, B, nb, synth.E4M3, synth.D_ORDER, scales=dsc_np[l:l + 1])
            ids = [list(range(nb))]
            o1.convert([sl(1, 8)], [ksub], [dl], [want], [n_tokens[r]], ids, ids)
            o1.convert([sl(2, 0)], [vsub], [dl], [want], [n_tokens[r]], ids, ids)
            assert np.array_equal(got, want), f"request {r} layer {l}: {int((got != want).sum())} bytes differ"
    used = sorted(b for t in dt_ for b in t)
    free = sorted(set(range(NB)) - set(used))
    fb = D6.index_select(0, torch.as_tensor(free, device=dev))
    assert bool((fb == synth.CANARY).all()), "a block outside the tables was written"
