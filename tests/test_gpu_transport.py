"""Transport parity on ONE GPU (A8 / A10 / A11): the pull, staged pull, push and flag
machinery of the multi-GPU data plane, with the P instance and the D instance as separate
pools on cuda:0 and one CUDA stream per TP rank, against the oracle O1 element by element.

The kernels are the ones the N >= 2 bench runs -- kv_stage (k_pack_rows into ring slots +
k_signal, k_wait on the free words), kv_pull_staged (the persistent k_pull_rows: dynamic
hand-out, in-kernel acquire of the ready words, in-order release of the ring slots), kv_pull
(k_wait, then the convert kernels reading the P pools), kv_push (convert_share + release
flag) and kv_signal / kv_wait -- only the pointers are local instead of IPC-mapped (the
paper's D-initiated read; by-layer transmission; step 5/6 handoff).

Same-GPU progress: every spinning kernel here is bounded (one warp for kv_wait, an SM budget
for the persistent pull), so the packs and converts they wait for always find free SMs, and
every wait has a timeout that sets the error word instead of hanging (the test then fails).
"""
import os

import numpy as np
import pytest
import torch

from synth import BF16, E4M3, F16
from tests.kvcase import expected, make_case

pytestmark = pytest.mark.gpu

R = 2          # ring slots: with 6 one-layer chunks every slot is reused three times
TIMEOUT = float(os.environ.get("KVX_TEST_TIMEOUT", "20"))
BUDGET = 16    # SMs per persistent pull kernel (the rest stay free for the P-side packs)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


def _case(shape, o1):
    if shape == "merge":      # c3-like: TP4 -> TP2, block 16 -> 64, bf16
        return make_case(6, 8, 128, 4, 2, 16, 64, [300, 77, 1], BF16, BF16, seed=31, o1=o1)
    if shape == "merge_fp8":  # c3-like merge TP4 -> TP2 with the narrowing cast (each P rank owns its heads' scales)
        return make_case(6, 8, 128, 4, 2, 16, 32, [100, 50, 2], BF16, E4M3, seed=34, o1=o1, scales="pow2")
    if shape == "split_fp8":  # c5-like split TP2 -> TP4 with a c4-like narrowing cast
        return make_case(6, 8, 128, 2, 4, 16, 16, [129, 40, 3], F16, E4M3, seed=32, o1=o1, scales="pow2")
    if shape == "identity_fp8":   # c4-like 1:1 pairs TP2 -> TP2, bf16 -> e4m3
        return make_case(6, 4, 128, 2, 2, 16, 16, [200, 17], BF16, E4M3, seed=33, o1=o1, scales="amax")
    if shape == "ragged_vendor":  # empty and 1-token requests; an x-packed K-only source pool
        from synth import LAYER, KV, BLOCK, SLOT, HEAD, DIM
        return make_case(6, 8, 64, 2, 2, 16, 32, [0, 45, 1, 0], BF16, BF16, (LAYER, KV, BLOCK, HEAD, DIM, SLOT),
                         seed=35, o1=o1, p_kv_part=1, p_split=8)
    raise ValueError(shape)


def _p_view_of_d(kvx, case, dyn):
    """P's own copies of D's layouts (what the control plane hands P): with dynamic scales
    P quantises with its own scale arrays and ships them into D's."""
    out = []
    for lay in case["dst_lays"]:
        sc = None
        if lay.get("scales") is not None:
            sc = torch.from_numpy(np.asarray(lay["scales"], np.float32)).cuda()
            if dyn:
                sc.fill_(-1.0)  # must be overwritten by kv_stage's amax pass
        out.append(kvx.Layout.from_dict(lay, sc))
    return out


def _run(o1, case, mode, serial_safe=False, lc=1):
    """serial_safe (the smoke): ring slots for every chunk and P's stages enqueued before D's
    persistent pulls, so the transfer also completes when every kernel runs alone in launch
    order (a profiler's replay, e.g. ncu over smoke()) -- P never waits for a free slot and
    each spin-wait is launched after the work it waits for."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    dc = DevCase(case, "cuda:0")
    S, D = dc.src_lays, dc.dst_lays
    dyn = mode == "pull_staged_dyn"
    DP = _p_view_of_d(kvx, case, dyn)          # P's view of D's layouts
    if dyn:
        for lay in D:
            lay.scales.fill_(-2.0)             # D's scale arrays: written by P (peer stores)
    pairs = kvx.plan_pairs(S[0].tp_degree, D[0].tp_degree, S[0].num_kv_heads)
    L = S[0].num_layers
    nch = kvx.chunk_count((0, L), lc)   # lc < 0: ramped chunk schedule (kv_chunk_count)
    ready = torch.zeros(128, dtype=torch.int32, device="cuda:0")   # D side: [q * 8 + p], P writes
    freew = torch.zeros(128, dtype=torch.int32, device="cuda:0")   # P side: [p * 8 + q], D writes
    err = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    w = lambda t, i: t.data_ptr() + 4 * i  # noqa: E731
    p_streams = [torch.cuda.Stream() for _ in S]
    d_streams = [torch.cuda.Stream() for _ in D]
    kvx.launch_count_reset()
    kernels = set()
    counters = {}
    torch.cuda.synchronize()
    if mode.startswith("pull_staged"):
        nb = max(kvx.wire_bytes(S[p], D[q], dc.src_bt.total_tokens, (l, min(L, l + abs(lc)))) for p, q, _, _ in pairs
                 for l in range(L))
        nb = max(16, (nb + 255) // 256 * 256)
        Rr = nch if serial_safe else R
        rings = {(p, q): torch.empty(Rr * nb, dtype=torch.uint8, device="cuda:0") for p, q, _, _ in pairs}
        persistent = mode != "pull_staged_chunked"

        def d_pulls():
            prev = kvx.set_sm_budget(BUDGET)
            try:
                for q in range(len(D)):
                    ps = [p for p, q2, _, _ in pairs if q2 == q]
                    if persistent:
                        counters[q] = torch.zeros(kvx.pull_counter_words((0, L), lc), dtype=torch.int32,
                                                  device="cuda:0")
                    with torch.cuda.stream(d_streams[q]):
                        kvx.pull_staged([S[p] for p in ps],
                                        [rings[(p, q)].data_ptr() + b * nb for p in ps for b in range(Rr)], Rr, nb,
                                        D[q], dc.dst_pools[q], dc.dst_bt, [w(ready, q * 8 + p) for p in ps],
                                        [w(freew, p * 8 + q) for p in ps], 0, err, (0, L), lc, TIMEOUT, d_streams[q],
                                        counters=counters.get(q))
                    kernels.add(kvx.last_kernel())
            finally:
                kvx.set_sm_budget(prev)

        # D first: the persistent kernels sit on their SM budget waiting for P's ready words
        if not serial_safe:
            d_pulls()
        for p in range(len(S)):
            qs = [q for p2, q, _, _ in pairs if p2 == p]
            with torch.cuda.stream(p_streams[p]):
                kvx.stage(S[p], dc.src_pools[p], dc.src_bt, [DP[q] for q in qs],
                          [rings[(p, q)].data_ptr() + b * nb for q in qs for b in range(Rr)], Rr, nb,
                          [w(ready, q * 8 + p) for q in qs], [w(freew, p * 8 + q) for q in qs], 0, err, (0, L), lc,
                          TIMEOUT, p_streams[p], peer_scales=[D[q].scales for q in qs] if dyn else None)
                kernels.add(kvx.last_kernel())
        if serial_safe:
            d_pulls()
        for p in range(len(S)):
            qs = [q for p2, q, _, _ in pairs if p2 == p]
            with torch.cuda.stream(p_streams[p]):
                for q in qs:   # every chunk consumed: P may reuse its ring
                    kvx.wait(w(freew, p * 8 + q), nch, err, TIMEOUT, p_streams[p])
    elif mode == "pull":
        prev = kvx.set_sm_budget(BUDGET)
        try:
            for q in range(len(D)):
                ps = [p for p, q2, _, _ in pairs if q2 == q]
                with torch.cuda.stream(d_streams[q]):
                    kvx.pull([S[p] for p in ps], [dc.src_pools[p] for p in ps], dc.src_bt, D[q], dc.dst_pools[q],
                             dc.dst_bt, [w(ready, q * 8 + p) for p in ps], [w(freew, p * 8 + q) for p in ps], 1, err,
                             (0, L), 2, TIMEOUT, d_streams[q])
                kernels.add(kvx.last_kernel())
        finally:
            kvx.set_sm_budget(prev)
        for p in range(len(S)):
            qs = [q for p2, q, _, _ in pairs if p2 == p]
            with torch.cuda.stream(p_streams[p]):
                for q in qs:
                    kvx.signal(w(ready, q * 8 + p), 1, p_streams[p])
                for q in qs:
                    kvx.wait(w(freew, p * 8 + q), 1, err, TIMEOUT, p_streams[p])
    elif mode == "push":
        for q in range(len(D)):   # D waits for every P rank feeding it
            ps = [p for p, q2, _, _ in pairs if q2 == q]
            with torch.cuda.stream(d_streams[q]):
                for p in ps:
                    kvx.wait(w(ready, q * 8 + p), 1, err, TIMEOUT, d_streams[q])
        for p in range(len(S)):
            qs = [q for p2, q, _, _ in pairs if p2 == p]
            with torch.cuda.stream(p_streams[p]):
                kvx.push(S[p], dc.src_pools[p], dc.src_bt, [DP[q] for q in qs], [dc.dst_pools[q] for q in qs],
                         dc.dst_bt, [w(ready, q * 8 + p) for q in qs], 1, (0, L), 2, p_streams[p])
                kernels.add(kvx.last_kernel())
    else:
        raise ValueError(mode)
    torch.cuda.synchronize()
    assert int(err.item()) == 0, "a flag wait timed out"
    if counters:   # every chunk handed out, completed and released in order
        for c in counters.values():
            assert int(c[2 * nch].item()) == nch, "ring slots not all released"
            assert bool((c[nch:2 * nch] > 0).all())
    return dc, kernels


def _scales_and_want(o1, case, dc):
    for q, lay in enumerate(case["dst_lays"]):
        want_sc = o1.amax_scales(case["src_lays"], case["src_pools"], lay, case["n_tokens"], case["src_tables"])
        got_sc = dc.dst_lays[q].scales.cpu().numpy().reshape(want_sc.shape)
        assert np.array_equal(got_sc, want_sc), f"D{q}: shipped dynamic scales differ from O1's amax scales"
        lay["scales"] = want_sc
    return expected(case, o1)


@pytest.mark.parametrize("mode", ["pull_staged", "pull_staged_chunked", "pull_staged_dyn", "pull", "push"])
@pytest.mark.parametrize("shape", ["merge", "merge_fp8", "split_fp8", "identity_fp8", "ragged_vendor"])
def test_transport_one_gpu(o1, mode, shape):
    from tests.test_gpu_parity import assert_pools_match
    if mode == "pull_staged_dyn" and shape in ("merge", "ragged_vendor"):
        pytest.skip("dynamic scales need an fp8 destination")
    case = _case(shape, o1)
    dc, kernels = _run(o1, case, mode)
    if mode == "pull_staged" or mode == "pull_staged_dyn":
        assert "k_pull_rows" in kernels, kernels
    if mode.startswith("pull_staged"):
        assert "k_pack_rows" in kernels or "k_pack" in kernels, kernels
    want = _scales_and_want(o1, case, dc) if mode == "pull_staged_dyn" else expected(case, o1)
    assert_pools_match(dc.dst_numpy(), want, case["dst_lays"][0]["dtype"])


@pytest.mark.parametrize("persistent_p", [False, True])
@pytest.mark.parametrize("lc", [-4, 4, -8])
def test_staged_pull_chunk_ramp(o1, lc, persistent_p, monkeypatch):
    """The ramped chunk schedule (negative layer_chunk: 1, 1, 2 layers, then |lc|) through the
    persistent pull with a 2-slot ring, against O1 -- both sides and the kernels enumerate
    the same chunks (A10); P as per-chunk packs or as the opt-in persistent
    k_stage_rows (KVX_STAGE_PERSISTENT=1, in-kernel free-slot waits and ready release)."""
    from tests.test_gpu_parity import assert_pools_match
    if persistent_p:
        monkeypatch.setenv("KVX_STAGE_PERSISTENT", "1")
    case = make_case(16, 4, 128, 2, 2, 16, 16, [200, 17, 1], BF16, E4M3, seed=37, o1=o1, scales="pow2")
    dc, kernels = _run(o1, case, "pull_staged", lc=lc)
    assert "k_pull_rows" in kernels, kernels
    assert ("k_stage_rows" if persistent_p else "k_pack_rows") in kernels, kernels
    assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])


@pytest.mark.parametrize("shape", ["merge_fp8", "identity_fp8", "merge"])
def test_staged_pull_persistent_stage(o1, shape, monkeypatch):
    """kv_stage as one persistent k_stage_rows launch (opt-in) on the one-destination shapes,
    2-slot ring reused three times, against O1."""
    from tests.test_gpu_parity import assert_pools_match
    monkeypatch.setenv("KVX_STAGE_PERSISTENT", "1")
    case = _case(shape, o1)
    dc, kernels = _run(o1, case, "pull_staged")
    assert {"k_pull_rows", "k_stage_rows"} <= kernels, kernels
    assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])


def test_smoke_with_serialized_launches():
    """smoke() (one-GPU staged pull included) with every launch synchronous, as when a
    profiler (ncu over smoke()) runs each kernel alone in launch order: no spin-wait may be
    launched ahead of the work that releases it."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1", KVX_TEST_TIMEOUT="10")
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "smoke ok" in r.stdout and "k_pull_rows" in r.stdout, r.stdout[-2000:]


def test_staged_pull_two_calls_seq0(o1):
    """Two kv_stage / kv_pull_staged rounds over the same rings and flags: the second call
    starts at seq0 = chunk_count of the first (slots keep rotating, free words keep rising)."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    from tests.test_gpu_parity import assert_pools_match
    case = make_case(5, 2, 128, 1, 1, 16, 16, [100, 33], BF16, E4M3, seed=36, o1=o1, scales="pow2")
    dc = DevCase(case, "cuda:0")
    S, D = dc.src_lays[0], dc.dst_lays[0]
    DP = _p_view_of_d(kvx, case, False)[0]
    L, lc = 5, 2
    nch = kvx.chunk_count((0, L), lc)
    nb = max(kvx.wire_bytes(S, D, dc.src_bt.total_tokens, (l, min(L, l + lc))) for l in range(0, L, lc))
    rings = torch.empty(R * nb, dtype=torch.uint8, device="cuda:0")
    ready = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    freew = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    err = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    ps, ds = torch.cuda.Stream(), torch.cuda.Stream()
    ctr = torch.zeros(kvx.pull_counter_words((0, L), lc), dtype=torch.int32, device="cuda:0")
    for rnd in range(2):
        seq0 = rnd * nch
        dc.dst_pools[0].fill_(0xA5)
        torch.cuda.synchronize()   # the fill (default stream) before the side streams' work
        prev = kvx.set_sm_budget(BUDGET)
        try:
            kvx.pull_staged([S], [rings.data_ptr() + b * nb for b in range(R)], R, nb, D, dc.dst_pools[0], dc.dst_bt,
                            [ready], [freew], seq0, err, (0, L), lc, TIMEOUT, ds, counters=ctr)
        finally:
            kvx.set_sm_budget(prev)
        kvx.stage(S, dc.src_pools[0], dc.src_bt, [DP], [rings.data_ptr() + b * nb for b in range(R)], R, nb, [ready],
                  [freew], seq0, err, (0, L), lc, TIMEOUT, ps)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        assert int(ready.item()) == seq0 + nch and int(freew.item()) == seq0 + nch
        assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)


def test_signal_wait_one_gpu():
    """kv_signal on one stream releases a kv_wait on another stream of the same GPU; work
    queued behind the wait runs only after the release; a wait that is never satisfied
    times out into the error word instead of hanging."""
    import paper_2509_17542_b200 as kvx
    flag = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    err = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    out = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    # every kernel that runs while the wait spins must have been loaded already (CUDA lazy
    # loading, include/kvx.h kv_preload): the library preloads its own; warm torch's
    torch.cuda._sleep(1000)
    out.copy_(flag[:1])
    torch.cuda.synchronize()
    kvx.wait(flag, 3, err, TIMEOUT, b)
    with torch.cuda.stream(b):
        out.copy_(flag[:1])                     # runs after the wait: sees the released value
    with torch.cuda.stream(a):
        torch.cuda._sleep(20_000_000)           # ~10 ms: the wait on stream b spins meanwhile
    kvx.signal(flag, 3, a)
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and int(out.item()) == 3
    # wrap-around order: a value "ahead" modulo 2^32 satisfies the wait
    flag[1] = 5
    kvx.signal(flag[1:2], 0x80000000 + 4, a)
    kvx.wait(flag[1:2], 0x80000000 + 2, err, TIMEOUT, b)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    # timeout: nobody signals word 2
    kvx.wait(flag[2:3], 1, err, 0.05, b)
    torch.cuda.synchronize()
    assert int(err.item()) == 1


@pytest.mark.parametrize("budget", [1, 7, 74])
@pytest.mark.parametrize("share", [False, True])
def test_sm_budget_parity(o1, budget, share):
    """NEXT-4: kv_set_sm_budget only shrinks the grid -- convert_reshard / convert_share with
    1, 7 or 74 SMs give O1's pools (P:289 overlap of transmission with prefill compute)."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    from tests.test_gpu_parity import assert_pools_match
    case = make_case(3, 8, 128, 4, 2, 16, 32, [150, 33, 1], BF16, E4M3, seed=40 + budget, o1=o1, scales="pow2")
    dc = DevCase(case, "cuda:0")
    prev = kvx.set_sm_budget(budget)
    try:
        if share:   # each P rank's share in turn (the distributed push's per-rank call)
            for p, lay in enumerate(dc.src_lays):
                qs = sorted({q for pp, q, _, _ in kvx.plan_pairs(4, 2, 8) if pp == p})
                kvx.convert_share(lay, dc.src_pools[p], dc.src_bt, [dc.dst_lays[q] for q in qs],
                                  [dc.dst_pools[q] for q in qs], dc.dst_bt)
        else:
            kvx.convert_reshard(dc.src_lays, dc.src_pools, dc.src_bt, dc.dst_lays, dc.dst_pools, dc.dst_bt)
        torch.cuda.synchronize()
    finally:
        assert kvx.set_sm_budget(prev) == budget
    assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)


@pytest.mark.parametrize("shape", ["identity_fp8", "merge"])
def test_host_staged_one_gpu(o1, shape):
    """NEXT-3: the paper's host-staged transport (pack -> D2H into a pinned CPU buffer -> H2D ->
    unpack, event-chained per layer chunk, 2 host slots reused) with P and D on cuda:0: the D
    pools equal O1's."""
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import transfer as tr
    from tests.gpu_util import DevCase
    from tests.test_gpu_parity import assert_pools_match
    case = _case(shape, o1)
    dc = DevCase(case, "cuda:0")
    S, D = dc.src_lays, dc.dst_lays
    DP = _p_view_of_d(kvx, case, False)
    L = S[0].num_layers
    torch.cuda.synchronize()
    for p, q, _, _ in kvx.plan_pairs(S[0].tp_degree, D[0].tp_degree, S[0].num_kv_heads):
        hs = tr.HostStaged(S[p], DP[q], D[q], dc.src_bt.total_tokens, (0, L), 2, 0, 0, slots=2)
        hs.step(dc.src_pools[p], dc.src_bt, dc.dst_pools[q], dc.dst_bt)
        torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])


@pytest.mark.parametrize("kind", ["rows", "tile"])
def test_convert_notify_per_request(o1, monkeypatch, kind):
    """A11 per request inside one launch (kv_convert_reshard_notify, the c5 stream's handoff):
    every request's flag carries the epoch and a completion time, requests with no tokens
    complete at once, and the pools equal O1's -- on the row kernel (in-kernel completion
    counting) and on the TMA tile path (completion when the launch ends)."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    from tests.test_gpu_parity import assert_pools_match
    if kind == "rows":
        case = make_case(3, 8, 128, 2, 4, 16, 16, [300, 0, 17, 1, 64], BF16, E4M3, seed=51, o1=o1, scales="pow2")
    else:
        monkeypatch.setenv("KVX_TILE", "2")
        case = make_case(2, 8, 128, 2, 1, 16, 16, [70, 0, 16], F16, F16, seed=52, o1=o1)
    dc = DevCase(case, "cuda:0")
    n = len(case["n_tokens"])
    cnt = torch.zeros(n, dtype=torch.int32, device="cuda:0")
    flags = torch.zeros(n, dtype=torch.int32, device="cuda:0")
    ns = torch.zeros(n, dtype=torch.int64, device="cuda:0")
    t0 = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    kvx.timestamp(t0)
    kvx.convert_reshard_notify(dc.src_lays, dc.src_pools, dc.src_bt, dc.dst_lays, dc.dst_pools, dc.dst_bt, cnt, flags,
                               7, ns)
    assert kvx.last_kernel() == ("k_convert_rows" if kind == "rows" else "k_tile_copy")
    torch.cuda.synchronize()
    assert flags.tolist() == [7] * n
    start = int(t0.item())
    assert all(v >= start for v in ns.tolist())
    assert_pools_match(dc.dst_numpy(), expected(case, o1), case["dst_lays"][0]["dtype"])
