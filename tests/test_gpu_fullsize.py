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
