"""Multi-GPU parity (needs >= 2 GPUs): P instance on cuda:0, D instance on cuda:1, one
process each.  Both transports against the oracle:
  * push: the fused convert kernel stores into the D pools mapped through CUDA IPC, then
    a release flag; D acquires it and checks its pools;
  * nccl: kv_pack -> ncclSend / ncclRecv -> kv_unpack per (p, q) pair and layer chunk;
  * pull: D maps the P pools through CUDA IPC and kv_pull reads them after P's ready flag;
  * pull_staged: P kv_stage-s layer chunks into 2-slot rings, D kv_pull_staged-s them from
    the peer-mapped slots (4 chunks: every slot is reused behind a free flag) -- one
    persistent k_pull_rows launch with chunk counters, or (pull_staged_chunked) one
    wait / unpack / signal triple per chunk.
Control plane: a gloo process group (object exchange)."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, blob, mode, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    if mode == "pull_staged_pp":  # P side as the opt-in persistent k_stage_rows
        os.environ["KVX_STAGE_PERSISTENT"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_2509_17542_b200 as kvx
        from paper_2509_17542_b200 import transfer as tr
        from tests.gpu_util import DevCase
        case = pickle.loads(blob)
        dc = DevCase(case, device=f"cuda:{rank}")
        flag = torch.zeros(4, dtype=torch.int32, device=f"cuda:{rank}")
        err = torch.zeros(1, dtype=torch.int32, device=f"cuda:{rank}")
        if mode == "push":
            exp = None
            if rank == 1:
                exp = [kvx.ipc_export(p) for p in dc.dst_pools] + [kvx.ipc_export(flag)]
            allx = tr.exchange(exp)
            if rank == 0:
                mapped = [kvx.ipc_open(h, o) for h, o in allx[1]]
                # one launch: all P ranks -> all D ranks, stores over NVLink
                kvx.convert_reshard(dc.src_lays, dc.src_pools, dc.src_bt, dc.dst_lays, mapped[:-1], dc.dst_bt)
                kvx.signal(mapped[-1], 1)
                torch.cuda.synchronize()
                dist.barrier()
                for (h, o), m in zip(allx[1], mapped):
                    kvx.ipc_close(m, o)
                q.put((rank, None))
            else:
                kvx.wait(flag, 1, err, 20.0)
                torch.cuda.synchronize()
                assert int(err.item()) == 0, "flag wait timed out"
                q.put((rank, [a.copy() for a in dc.dst_numpy()]))
                dist.barrier()
        elif mode.startswith("pull"):
            _pull_worker(rank, dc, kvx, tr, dist, q, mode.startswith("pull_staged"),
                         mode in ("pull_staged", "pull_staged_dyn", "pull_staged_pp"), mode == "pull_staged_dyn")
        else:
            uid = kvx.Comm.unique_id() if rank == 0 else None
            lst = [uid]
            dist.broadcast_object_list(lst, src=0)
            comm = kvx.Comm(2, rank, lst[0], rank)
            pairs = kvx.plan_pairs(dc.src_lays[0].tp_degree, dc.dst_lays[0].tp_degree, dc.src_lays[0].num_kv_heads)
            L = dc.src_lays[0].num_layers
            for l0 in range(0, L, 2):  # layer chunks of 2
                lr = (l0, min(L, l0 + 2))
                for p, qq, _, _ in pairs:
                    S, D = dc.src_lays[p], dc.dst_lays[qq]
                    nb = kvx.wire_bytes(S, D, dc.src_bt.total_tokens, lr)
                    wire = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{rank}")
                    if rank == 0:
                        kvx.pack(S, dc.src_pools[p], dc.src_bt, D, wire, lr)
                        comm.send(1, wire, nb)
                    else:
                        comm.recv_unpack(0, wire, nb, S, D, dc.dst_pools[qq], dc.dst_bt, lr)
                    torch.cuda.synchronize()
            comm.close()
            q.put((rank, None if rank == 0 else [a.copy() for a in dc.dst_numpy()]))
    finally:
        dist.destroy_process_group()


def _pull_worker(rank, dc, kvx, tr, dist, q, staged, persistent, dyn=False):
    """P = rank 0 (all P ranks, one stream each), D = rank 1 (all D ranks, one stream each).
    Flag words: D's ready[q * 8 + p] (P writes), P's done / free[p * 8 + q] (D writes)."""
    dev = f"cuda:{rank}"
    flags = torch.zeros(64, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    S, D = dc.src_lays, dc.dst_lays
    pairs = kvx.plan_pairs(S[0].tp_degree, D[0].tp_degree, S[0].num_kv_heads)
    L = S[0].num_layers
    R, lc = 2, 1
    nb = 0
    for p, qq, _, _ in pairs:
        nb = max(nb, max(kvx.wire_bytes(S[p], D[qq], dc.src_bt.total_tokens, (l, l + 1)) for l in range(L)))
    rings = {}
    if rank == 0 and staged:
        for p, qq, _, _ in pairs:
            rings[(p, qq)] = torch.empty(R * nb, dtype=torch.uint8, device=dev)
    exp = {"flags": kvx.ipc_export(flags)}
    if rank == 1 and dyn:   # D's scale arrays: P computes the dynamic scales and writes them here
        exp["scales"] = [kvx.ipc_export(lay.scales) for lay in D]
    if rank == 0:
        exp["src"] = {k: kvx.ipc_export(v) for k, v in rings.items()} if staged else \
            [kvx.ipc_export(pl) for pl in dc.src_pools]
    allx = tr.exchange(exp)
    other = allx[1 - rank]
    fbase = kvx.ipc_open(*other["flags"])
    maps = [(fbase, other["flags"][1])]
    streams = {}
    peer_sc = []
    if rank == 0 and dyn:
        peer_sc = [kvx.ipc_open(h, o) for h, o in other["scales"]]
        maps += [(a, o) for a, (h, o) in zip(peer_sc, other["scales"])]
    # every P rank of the test shares GPU0: persistent P kernels (KVX_STAGE_PERSISTENT) each
    # get an SM budget so all of them stay resident (a spinning one must not starve another)
    prev_budget = kvx.set_sm_budget(16) if rank == 0 and os.environ.get("KVX_STAGE_PERSISTENT") else None
    if rank == 0:
        for p in range(len(S)):
            qs = [qq for pp, qq, _, _ in pairs if pp == p]
            st = streams[p] = torch.cuda.Stream()
            with torch.cuda.stream(st):
                if staged:
                    kvx.stage(S[p], dc.src_pools[p], dc.src_bt, [D[qq] for qq in qs],
                              [rings[(p, qq)].data_ptr() + b * nb for qq in qs for b in range(R)], R, nb,
                              [fbase + 4 * (qq * 8 + p) for qq in qs], [flags[p * 8 + qq:p * 8 + qq + 1] for qq in qs],
                              0, err, (0, L), lc, 20.0, st,
                              peer_scales=[peer_sc[qq] for qq in qs] if dyn else None)
                    for qq in qs:   # all chunks consumed: free >= number of chunks
                        kvx.wait(flags[p * 8 + qq:p * 8 + qq + 1], L, err, 20.0, st)
                else:
                    for qq in qs:
                        kvx.signal(fbase + 4 * (qq * 8 + p), 1, st)
                    for qq in qs:
                        kvx.wait(flags[p * 8 + qq:p * 8 + qq + 1], 1, err, 20.0, st)
        if prev_budget is not None:
            kvx.set_sm_budget(prev_budget)
        torch.cuda.synchronize()
        assert int(err.item()) == 0, "P-side wait timed out"
        dist.barrier()
        q.put((rank, None))
    else:
        if staged:
            src = {k: kvx.ipc_open(h, o) for k, (h, o) in other["src"].items()}
            maps += [(src[k], other["src"][k][1]) for k in src]
        else:
            src = [kvx.ipc_open(h, o) for h, o in other["src"]]
            maps += [(a, o) for a, (h, o) in zip(src, other["src"])]
        counters = {qq: torch.zeros(2 * L + 1, dtype=torch.int32, device=dev) for qq in range(len(D))}
        for qq in range(len(D)):
            ps = [pp for pp, q2, _, _ in pairs if q2 == qq]
            st = streams[qq] = torch.cuda.Stream()
            with torch.cuda.stream(st):
                if staged:
                    kvx.pull_staged([S[p] for p in ps], [src[(p, qq)] + b * nb for p in ps for b in range(R)], R, nb,
                                    D[qq], dc.dst_pools[qq], dc.dst_bt, [flags[qq * 8 + p:qq * 8 + p + 1] for p in ps],
                                    [fbase + 4 * (p * 8 + qq) for p in ps], 0, err, (0, L), lc, 20.0, st,
                                    counters=counters[qq] if persistent else None)
                else:
                    kvx.pull([S[p] for p in ps], [src[p] for p in ps], dc.src_bt, D[qq], dc.dst_pools[qq], dc.dst_bt,
                             [flags[qq * 8 + p:qq * 8 + p + 1] for p in ps], [fbase + 4 * (p * 8 + qq) for p in ps],
                             1, err, (0, L), lc, 20.0, st)
        torch.cuda.synchronize()
        assert int(err.item()) == 0, "D-side wait timed out"
        assert kvx.last_kernel() == ("k_pull_rows" if persistent else "k_unpack_rows" if staged else kvx.last_kernel())
        if persistent:   # every chunk handed out and completed in full
            for c in counters.values():
                nxt, done = c[:L].cpu(), c[L:2 * L].cpu()
                assert bool((done > 0).all()) and bool((nxt >= done).all())
                assert int(c[2 * L]) == L   # every chunk released, in order
        res = [a.copy() for a in dc.dst_numpy()]
        if dyn:
            res = (res, [lay.scales.cpu().numpy().reshape(L, 2, -1) for lay in D])
        q.put((rank, res))
        dist.barrier()
    for a, o in maps:
        kvx.ipc_close(a, o)


@pytest.mark.parametrize("mode", ["push", "nccl", "pull", "pull_staged", "pull_staged_chunked", "pull_staged_dyn",
                                  "pull_staged_pp"])
@pytest.mark.parametrize("shape", ["merge", "split_fp8", "ragged_vendor"])
def test_p_to_d_across_gpus(o1, mode, shape):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    from synth import BF16, E4M3, F16
    from tests.kvcase import expected, make_case
    from tests.test_gpu_parity import assert_pools_match
    if mode == "pull_staged_dyn" and shape == "merge":
        pytest.skip("dynamic scales need each P rank to hold all of its D ranks' heads (bf16 merge has no fp8)")
    if shape == "ragged_vendor" and mode in ("pull_staged_dyn",):
        pytest.skip("the vendor pools here carry no fp8 destination")
    if shape == "merge":   # c3-like: TP4 -> TP2, block 16 -> 64
        case = make_case(4, 8, 128, 4, 2, 16, 64, [300, 77, 1], BF16, BF16, seed=3, o1=o1)
    elif shape == "ragged_vendor":  # an empty request, a 1-token one; an x-packed K-only source pool
        from synth import LAYER, KV, BLOCK, SLOT, HEAD, DIM
        case = make_case(3, 8, 64, 2, 2, 16, 32, [0, 45, 1, 0], BF16, BF16, (LAYER, KV, BLOCK, HEAD, DIM, SLOT),
                         seed=5, o1=o1, p_kv_part=1, p_split=8)
    else:                  # c5-like split TP2 -> TP4 with a c4-like fp8 cast
        case = make_case(4, 8, 128, 2, 4, 16, 16, [129, 40], F16, E4M3, seed=4, o1=o1, scales="pow2")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    blob = pickle.dumps(case)
    ps = [ctx.Process(target=_worker, args=(r, port, blob, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    if mode == "pull_staged_dyn":
        # NEXT-1 (i): the shipped scales are O1's amax scales; the codes decode with them
        got, got_sc = res[1]
        for qq, lay in enumerate(case["dst_lays"]):
            want_sc = o1.amax_scales(case["src_lays"], case["src_pools"], lay, case["n_tokens"], case["src_tables"])
            assert np.array_equal(got_sc[qq], want_sc), f"D{qq} scales"
            lay["scales"] = want_sc
        assert_pools_match(got, expected(case, o1), case["dst_lays"][0]["dtype"])
        return
    assert_pools_match(res[1], expected(case, o1), case["dst_lays"][0]["dtype"])
