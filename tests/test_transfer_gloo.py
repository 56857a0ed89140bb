"""Host-side logic of the multi-GPU path, on CPU with world_size-2 gloo process groups:
roles, the pair plan each rank derives, and the IPC handle exchange of PushChannel (with
the CUDA IPC calls replaced by fakes -- the control plane is what is under test)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_17542_b200 import transfer as tr
        roles = tr.roles(world, world // 2, world // 2)
        me = roles[rank]
        # every rank derives the same plan independently
        plan = tr.pair_plan(4, 4, 8, p_ranks=set(range(world // 2)), d_ranks=set(range(world // 2)))
        plans = tr.exchange(plan)
        exported, opened = [], []

        def fake_export(t):
            exported.append(t)
            return (bytes([rank]) * 64, 4096 * rank + len(exported))

        def fake_open(handle, off):
            opened.append((handle[0], off))
            return 0x7000_0000 + handle[0] * 0x100000 + off

        pool = "pool" if me.kind == "D" else None
        flag = "flag" if me.kind == "D" else None
        ch = tr.PushChannel(me, pool, flag, ipc_export=fake_export, ipc_open=fake_open)
        q.put((rank, me.kind, me.tp_rank, plans, exported, opened, ch.peer_pool, ch.peer_flag))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 6, 8])
def test_roles_plan_and_handle_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    npair = world // 2
    for rank, kind, tpr, plans, exported, opened, peer_pool, peer_flag in res:
        assert kind == ("P" if rank < npair else "D") and tpr == rank % npair
        assert all(pl == plans[0] for pl in plans)
        assert sorted((p, q) for p, q, _, _ in plans[0]) == [(i, i) for i in range(npair)]
        if kind == "D":
            assert exported == ["pool", "flag"] and opened == []
            assert peer_pool == {}
        else:
            assert exported == []
            # one pool + one flag handle per D rank, mapped with the exporter's offsets
            assert sorted(peer_pool) == list(range(npair)) and sorted(peer_flag) == list(range(npair))
            for qd in range(npair):
                owner = npair + qd
                assert peer_pool[qd] == 0x7000_0000 + owner * 0x100000 + 4096 * owner + 1
                assert peer_flag[qd] == 0x7000_0000 + owner * 0x100000 + 4096 * owner + 2


def test_roles_validation():
    from paper_2509_17542_b200 import transfer as tr
    with pytest.raises(ValueError):
        tr.roles(4, 1, 2)
    r = tr.roles(8, 4, 4)
    assert [x.kind for x in r] == ["P"] * 4 + ["D"] * 4
    # c3: TP4 -> TP2 merge; c5 per P instance: TP2 -> TP4 split
    assert sorted((p, q) for p, q, _, _ in tr.pair_plan(4, 2, 8)) == [(0, 0), (1, 0), (2, 1), (3, 1)]
    assert sorted((p, q) for p, q, _, _ in tr.pair_plan(2, 4, 8)) == [(0, 0), (0, 1), (1, 2), (1, 3)]


def test_present_ranks_sub_transfers():
    """The largest complete sub-transfer per GPU count: every present D rank has all the P
    ranks holding its heads; N >= tp_p + tp_d is the full transfer."""
    from paper_2509_17542_b200 import transfer as tr
    assert tr.present_ranks(2, 1, 2) == (0, 0)   # c2 needs 3 GPUs
    assert tr.present_ranks(2, 1, 3) == (2, 1)   # c2 full
    assert tr.present_ranks(4, 2, 4) == (2, 1)   # c3' (fan-in 2) + 1 idle GPU
    assert tr.present_ranks(4, 2, 6) == (4, 2)   # c3 full
    assert tr.present_ranks(4, 4, 2) == (1, 1)   # c4 one pair
    assert tr.present_ranks(4, 4, 8) == (4, 4)   # c4 full
    assert tr.present_ranks(2, 4, 3) == (1, 2)   # split: one P rank feeds two D ranks
    for tp_p, tp_d in [(2, 1), (4, 2), (4, 4), (2, 4), (1, 8)]:
        for n in range(2, 10):
            n_p, n_d = tr.present_ranks(tp_p, tp_d, n)
            assert n_p + n_d <= n
            if n_d:
                heads_needed = {p for p, q, _, _ in tr.pair_plan(tp_p, tp_d, 8) if q < n_d}
                assert heads_needed <= set(range(n_p))
    r = tr.roles(4, 2, 1, allow_idle=True)
    assert [x.kind for x in r] == ["P", "P", "D", "X"]


def _pull_worker(rank, world, port, q, staged):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_17542_b200 import transfer as tr
        n_p = world - 1
        me = tr.roles(world, n_p, 1)[rank]   # fan-in: P0..P{n_p-1} -> D0 (c2 / c3' shape)
        exported = []

        def fake_export(t):
            exported.append(t)
            return (bytes([rank]) * 64, 100 * len(exported))

        def fake_open(handle, off):
            return 0x7000_0000 + handle[0] * 0x100000 + off

        kw = {}
        if me.kind == "P":
            kw = dict(ring="ring", ring_dst=[0], ring_slots=2, slot_bytes=1000) if staged else dict(pool="pool")
        ch = tr.PullChannel(me, "flags", ipc_export=fake_export, ipc_open=fake_open, **kw)
        q.put((rank, me.kind, me.tp_rank, exported, ch.src_pool, ch.src_ring, ch.peer_flag))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,staged", [(2, False), (3, False), (3, True), (5, True), (8, False)])
def test_pull_channel_exchange(world, staged):
    """PullChannel: D maps every P rank's pool (or its ring slots for this D rank) and the
    word it owns in P's flag array; P maps its word in D's ready array."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pull_worker, args=(r, world, port, q, staged)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n_p = world - 1
    d_rank = n_p
    for rank, kind, tpr, exported, src_pool, src_ring, peer_flag in res:
        if kind == "P":
            assert exported == ["flags", "ring" if staged else "pool"]
            # P rank tpr signals word tpr of D0's ready array (D exported flags at offset 100)
            assert peer_flag == {0: 0x7000_0000 + d_rank * 0x100000 + 100 + 4 * tpr}
            assert src_pool == {} and src_ring == {}
        else:
            assert exported == ["flags"]
            assert sorted(peer_flag) == list(range(n_p))
            for p in range(n_p):
                base = 0x7000_0000 + p * 0x100000
                assert peer_flag[p] == base + 100 + 4 * 0   # D0's word in P's done/free array
                if staged:
                    assert src_pool == {}
                    assert src_ring[p] == [base + 200 + b * 1000 for b in range(2)]
                else:
                    assert src_pool[p] == base + 200 and src_ring == {}


def test_stream_plan_wiring():
    """c5 (2 P instances x TP2 -> D TP4): at N = 8 the full stream -- every D rank is fed by
    one P rank of EACH instance holding its heads, every P rank feeds the two D ranks its heads
    go to; at N = 4 the c5' sub-config (A0 + B0 -> D0, D1); flag words are world ranks and
    distinct per peer."""
    from paper_2509_17542_b200 import transfer as tr
    pl = tr.StreamPlan(8, 2, 4, 8, 64)
    assert [(r.kind, r.inst, r.tp_rank) for r in map(pl.role, range(8))] == \
        [("P", 0, 0), ("P", 0, 1), ("P", 1, 0), ("P", 1, 1), ("D", -1, 0), ("D", -1, 1), ("D", -1, 2), ("D", -1, 3)]
    assert [pl.d_peers(r) for r in range(4)] == [[0, 1], [2, 3], [0, 1], [2, 3]]
    assert [pl.p_sources(pl.d_world(q)) for q in range(4)] == [[0, 2], [0, 2], [1, 3], [1, 3]]
    assert pl.requests_of(0) == list(range(0, 64, 2)) and pl.requests_of(1) == list(range(1, 64, 2))
    assert all(pl.inst_of(r) == r % 2 for r in range(64))
    assert sorted(pl.p_index(i, t) for i in range(2) for t in range(2)) == [0, 1, 2, 3]
    for d in range(4, 8):   # the words a D rank's sources signal in its array never collide
        words = [pl.flag_word(pr) for pr in pl.p_sources(d)]
        assert len(set(words)) == len(words) and all(0 <= w < pl.flag_words for w in words)
    for p in range(4):      # nor do the D peers' words in a P rank's array
        words = [pl.flag_word(pl.d_world(q)) for q in pl.d_peers(p)]
        assert len(set(words)) == len(words) and all(0 <= w < pl.flag_words for w in words)
    # every (request, D rank, head) is delivered by exactly one P rank
    for r in range(64):
        inst = pl.inst_of(r)
        for q in range(4):
            feeders = [pr for pr in pl.p_sources(pl.d_world(q)) if pl.role(pr).inst == inst]
            assert len(feeders) == 1
    small = tr.StreamPlan(4, 2, 4, 8, 64)
    assert (small.n_inst, small.per_inst, small.n_d) == (2, 1, 2)
    assert [small.d_peers(r) for r in range(2)] == [[0, 1], [0, 1]]
    assert [small.p_sources(small.d_world(q)) for q in range(2)] == [[0, 1], [0, 1]]
    with pytest.raises(ValueError):
        tr.StreamPlan(1, 2, 4, 8, 64)
