"""A3 control plane on CPU: the kv_ctrl message (layout descriptor + fp8 scales + block
tables, include/kvx.h) round-trips byte-exactly, rejects corrupted / inconsistent messages,
and transfer.ControlPlane delivers every rank's message to every other rank of a gloo job of
2, 4, 6 and 8 processes -- the full c3 (6 GPUs: TP4 -> TP2), c4 (8 GPUs: TP4 -> TP4) and c5
(8 GPUs: 2 x TP2 -> TP4) role layouts included -- so that a P rank's view of D's tables and
scales, and a D rank's view of P's, equal what the owner chose."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


@pytest.fixture(scope="module")
def kvx():
    import __graft_entry__ as g
    g.build()
    import paper_2509_17542_b200 as k
    return k


def _lay(kvx, dtype=None, scales=None, tp=2, rank=1, NB=50, B=16, L=3, H=8, D=64, order=synth.D_ORDER):
    import torch
    dtype = synth.BF16 if dtype is None else dtype
    sc = None
    if dtype in synth.FP8:
        sc = torch.from_numpy(np.asarray(scales, np.float32).reshape(-1).copy())
    return kvx.Layout(L, H, D, tp, rank, B, NB, dtype, order, sc)


def test_ctrl_roundtrip(kvx):
    rng = np.random.default_rng(0)
    sc = np.ldexp(1.0, rng.integers(-8, 9, size=(3, 2, 4))).astype(np.float32)
    sc[0, 1, 2] = 0.0123456   # any fp32 travels bit-exactly
    lay = _lay(kvx, synth.E4M3, sc)
    nt = [33, 0, 16, 1]
    tables = synth.block_tables(7, nt, 16, 50)
    msg = kvx.ctrl_encode(lay, sc, nt, tables, batch_id=77)
    assert len(msg) == 128 + 4 * sc.size + 4 * len(nt) + 4 * sum(len(t) for t in tables)
    assert msg[:4] == b"KVC1"
    m = kvx.ctrl_decode(msg)
    assert m.batch_id == 77 and m.n_tokens == nt
    assert [list(t) for t in m.tables] == tables
    assert m.scales.dtype == np.float32 and np.array_equal(m.scales.view(np.uint32), sc.view(np.uint32))
    d = m.desc
    assert (d["L"], d["H"], d["D"], d["tp"], d["rank"], d["B"], d["NB"], d["dtype"], d["order"]) == \
        (3, 8, 64, 2, 1, 16, 50, synth.E4M3, tuple(synth.D_ORDER))
    # the received layout describes the same pool
    lay2 = m.layout("cpu")
    assert lay2.pool_bytes == lay.pool_bytes and lay2.axis_order == lay.axis_order
    # layout only (no scales, no tables)
    m2 = kvx.ctrl_decode(kvx.ctrl_encode(_lay(kvx)))
    assert m2.scales is None and m2.tables is None and m2.n_tokens is None
    # empty batch
    m3 = kvx.ctrl_decode(kvx.ctrl_encode(_lay(kvx), None, [], []))
    assert m3.n_tokens == [] and m3.tables == []


def test_ctrl_rejects_bad_messages(kvx):
    lay = _lay(kvx)
    nt = [40, 8]
    tables = synth.block_tables(3, nt, 16, 50)
    msg = bytearray(kvx.ctrl_encode(lay, None, nt, tables))
    # any payload byte flipped: digest mismatch
    for pos in (128, len(msg) - 1):
        bad = bytearray(msg)
        bad[pos] ^= 1
        with pytest.raises(kvx.KvError, match="digest"):
            kvx.ctrl_decode(bytes(bad))
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        kvx.ctrl_decode(bytes(msg[:-4]))          # truncated
    bad = bytearray(msg)
    bad[0:4] = b"KVX1"
    with pytest.raises(kvx.KvError, match="magic"):
        kvx.ctrl_decode(bytes(bad))
    bad = bytearray(msg)
    bad[24 + 4 * 4:24 + 4 * 5] = (3).to_bytes(4, "little")   # tp_degree 3 does not divide 8 heads
    with pytest.raises(kvx.KvError, match="layout"):
        kvx.ctrl_decode(bytes(bad))
    # the sender validates its tables like kv_block_table_update
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        kvx.ctrl_encode(lay, None, nt, [tables[0], tables[0][:1]])            # duplicate id
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        kvx.ctrl_encode(lay, None, nt, [tables[0][:-1], tables[1]])           # too few ids
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        kvx.ctrl_encode(lay, None, [8], [[50]])                              # out of range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPES = {   # name: (tp_p, tp_d, P dtype, D dtype)
    "c2": (2, 1, synth.F16, synth.F16),
    "c3": (4, 2, synth.BF16, synth.BF16),
    "c4": (4, 4, synth.BF16, synth.E4M3),
    "c5": (2, 4, synth.BF16, synth.BF16),
}


def _owner_view(shape, kind, r):
    """What rank r of instance `kind` chooses (seeded here; the receivers never see the seeds)."""
    tp_p, tp_d, sdt, ddt = SHAPES[shape]
    nt = [300, 17, 0, 64]
    B = 16
    NB = synth.pool_capacity(nt, B)
    seed = 11 if kind == "P" else 22
    tables = synth.block_tables(seed, nt, B, NB)
    tp, dt = (tp_p, sdt) if kind == "P" else (tp_d, ddt)
    sc = synth.pow2_scales(100 + r, 2, 8 // tp) if dt in synth.FP8 else None
    return dict(L=2, H=8, D=64, tp=tp, rank=r, B=B, NB=NB, dtype=dt,
                order=synth.P_ORDER if kind == "P" else synth.D_ORDER), sc, nt, tables


def _ctrl_worker(rank, world, port, shape, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import paper_2509_17542_b200 as kvx
        from paper_2509_17542_b200 import transfer as tr
        tp_p, tp_d = SHAPES[shape][:2]
        n_p, n_d = tr.present_ranks(tp_p, tp_d, world)
        me = tr.roles(world, n_p, n_d, allow_idle=True)[rank]
        pub = {}
        if me.kind in "PD":
            d, sc, nt, tables = _owner_view(shape, me.kind, me.tp_rank)
            lay = kvx.Layout.from_dict(d, None if sc is None else torch.from_numpy(sc.reshape(-1).copy()))
            cp = tr.ControlPlane(me, lay, sc, nt, tables, batch_id=5)
        else:
            cp = tr.ControlPlane(me)
        got = {}
        for (kind, r), m in cp.msgs.items():
            got[(kind, r)] = (m.desc, None if m.scales is None else m.scales.copy(), m.n_tokens,
                              [list(t) for t in m.tables], m.batch_id)
        other = {"P": "D", "D": "P"}.get(me.kind)
        pairs = tr.pair_plan(tp_p, tp_d, 8, p_ranks=set(range(n_p)), d_ranks=set(range(n_d)))
        if other:
            # the peer instance's tables and every peer layout this rank needs are usable
            nt, tb = cp.tables(other)
            peers = [q for p, q, _, _ in pairs if p == me.tp_rank] if me.kind == "P" else \
                [p for p, q, _, _ in pairs if q == me.tp_rank]
            for r in peers:
                pl = cp.layout(other, r, "cpu")
                pub[r] = pl.pool_bytes
        q.put((rank, me.kind, me.tp_rank, n_p, n_d, got, pub, cp.bytes_received))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, "c4"), (3, "c2"), (4, "c3"), (4, "c5"), (6, "c3"), (8, "c4"),
                                         (8, "c5")])
def test_control_plane_exchange(world, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ctrl_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tp_p, tp_d = SHAPES[shape][:2]
    n_p, n_d = res[0][3], res[0][4]
    if world >= tp_p + tp_d:
        assert (n_p, n_d) == (tp_p, tp_d), "the full transfer must fit"
    for rank, kind, tpr, _, _, got, pub, nbytes in res:
        # every present rank's message, exactly as its owner built it
        assert sorted(got) == sorted([("P", p) for p in range(n_p)] + [("D", d) for d in range(n_d)])
        for (k, r), (desc, sc, nt, tables, bid) in got.items():
            d, sc0, nt0, tb0 = _owner_view(shape, k, r)
            assert bid == 5 and nt == nt0 and tables == tb0
            for key in ("L", "H", "D", "tp", "rank", "B", "NB", "dtype"):
                assert desc[key] == d[key], key
            assert desc["order"] == tuple(d["order"])
            if sc0 is None:
                assert sc is None
            else:
                assert np.array_equal(sc.view(np.uint32), sc0.view(np.uint32))
        if kind in "PD":
            assert pub and all(v > 0 for v in pub.values())
        assert nbytes > 0
