"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(kv_convert_reshard over the whole batch, one GPU holding the ranks' pools).

The oracle cannot redo GBs, so: (1) sampled outputs -- requests first / middle / last, a
few layers, all their blocks, compared element by element with O1 run on the extracted
source blocks; (2) K6 over the whole D pools after a second transfer of a hash-coded fill
(kv_verify_fill / kv_verify_check: every valid element, every tail slot, every unused
block's canary) -- itself pinned to O1 in tests/test_gpu_verify.py."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name,p_ranks,d_ranks,reqs", [
    ("c2", [0, 1], [0], [0]),
    ("c3", [0, 1], [0], [0, 7, 15]),
    ("c4", [0], [0], [0, 16, 31]),
    ("c5", [0], [0, 1], [0, 15, 31]),
])
def test_fullsize_sampled_and_k6(name, p_ranks, d_ranks, reqs):
    import dataclasses
    import paper_2509_17542_b200 as kvx
    from bench import K6_SEED, d_tables, make_d_rank, make_p_rank, o1_compare, p_tables, sample_of
    cfg = synth.configs()[name]
    if name == "c5":  # one P instance (A) of the stream: even requests
        cfg = dataclasses.replace(cfg, n_tokens=cfg.n_tokens[0::2])
    dev = torch.device("cuda", 0)
    NB_p, NB_d = synth.pool_capacity(cfg.n_tokens, cfg.B_p), synth.pool_capacity(cfg.n_tokens, cfg.B_d)
    P = {p: make_p_rank(cfg, p, NB_p, dev) for p in p_ranks}
    Dr = {q: make_d_rank(cfg, q, NB_d, dev) for q in d_ranks}
    pt, dt_ = p_tables(cfg, NB_p), d_tables(cfg, NB_d)
    S, SP = [P[p][1] for p in p_ranks], [P[p][2] for p in p_ranks]
    Dl, DP = [Dr[q][1] for q in d_ranks], [Dr[q][2] for q in d_ranks]
    sbt = kvx.Batch(S[0], cfg.n_tokens, pt, dev)
    dbt = kvx.Batch(Dl[0], cfg.n_tokens, dt_, dev)
    kvx.convert_reshard(S, SP, sbt, Dl, DP, dbt)
    torch.cuda.synchronize()
    L = cfg.L
    for r in reqs:
        for layers in ((0, 1), (L // 2, L // 2 + 1), (L - 1, L)):
            ss = [sample_of(P[p][2], P[p][0], pt, [r], layers) for p in p_ranks]
            ds = [sample_of(Dr[q][2], Dr[q][0], dt_, [r], layers) for q in d_ranks]
            res = o1_compare(ss, ds, [cfg.n_tokens[r]], cfg.dst_dtype)
            assert res["ok"] and res["mismatches"] == 0, (r, layers, res)
    # K6: a hash-coded fill, the same launch again, every element of every D pool
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    for lay, pool in zip(S, SP):
        kvx.verify_fill(lay, pool, sbt, Dl, K6_SEED, err)
    kvx.convert_reshard(S, SP, sbt, Dl, DP, dbt)
    for lay, pool in zip(Dl, DP):
        res = torch.zeros(8, dtype=torch.int64, device=dev)
        scratch = torch.empty(lay.num_blocks, dtype=torch.uint8, device=dev)
        kvx.verify_check(S[0], lay, pool, dbt, K6_SEED, res, scratch)
        r6 = [int(x) for x in res.cpu()]
        assert int(err.item()) == 0 and r6[:3] == [0, 0, 0], r6
        assert r6[3] == 2 * L * lay.h_local * cfg.D * cfg.total_tokens


def test_fullsize_vendor_layouts(o1):
    """c4 pair at full size (80 layers, 2 local heads, 32 x 4096 tokens, block 16, TP4 -> 4
    rank 0 -> 0) from an other-vendor P cache -- x-packed K pool ([LAYER], BLOCK, HEAD,
    D/8, SLOT, 8) and head_dim-major V pool ([LAYER], BLOCK, HEAD, DIM, SLOT) -- into the
    NVIDIA-style D pool (BLOCK, LAYER, KV, HEAD, SLOT, DIM), bf16 -> e4m3, in the two
    calls tools/variants_bench.py times (k_convert_tb for both).  Sampled: requests 0 / 17 / 31 x
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
    assert kvx.last_kernel() == "k_convert_tb"   # x-packed tiles through TMA
    kvx.convert_reshard([Vl], [Vp], sbt, [Dl], [DP], dbt)
    assert kvx.last_kernel() == "k_convert_tb"   # head_dim-major tiles through TMA
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
