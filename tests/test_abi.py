"""CPU checks of the C-ABI library: it loads, exports every symbol include/kvx.h declares,
and its host-side logic (validation, strides, re-shard plan, wire sizes, block-table
validation) behaves -- all without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvx():
    import __graft_entry__ as g   # builds libkvx.so by path (the package needs it to import)
    g.build()
    import paper_2509_17542_b200 as k
    return k


def _declared():
    src = open(os.path.join(ROOT, "include", "kvx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kv_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(kvx):
    from paper_2509_17542_b200 import _lib
    declared = _declared()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert sorted(_lib.EXPORTS) == declared
    assert b"sm_100a" in _lib.lib.kv_version()


def test_library_is_sm100a_only():
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2509_17542_b200", "libkvx.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _lay(kvx, **kw):
    d = dict(num_layers=2, num_kv_heads=8, head_dim=16, tp_degree=2, tp_rank=0, block_size=4, num_blocks=10,
             dtype=kvx.KV_BF16, axis_order=(0, 1, 2, 3, 4, 5))
    d.update(kw)
    return kvx.Layout(**d)


def test_describe_pool_bytes_and_errors(kvx):
    l = _lay(kvx)
    assert l.pool_bytes == 2 * 2 * 10 * 4 * 4 * 16 * 2
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        _lay(kvx, tp_degree=3)
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        _lay(kvx, tp_rank=2)
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        _lay(kvx, axis_order=(0, 1, 2, 3, 4, 4))
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        _lay(kvx, dtype=7)
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        _lay(kvx, dtype=kvx.KV_F8E4M3)  # fp8 needs scales
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        _lay(kvx, block_size=0)


@pytest.mark.parametrize("tp_p,tp_d,H", [(4, 2, 8), (2, 4, 8), (4, 4, 8), (1, 8, 8), (8, 1, 8), (6, 4, 12), (2, 1, 32)])
def test_plan_pairs_matches_oracle(kvx, o1, tp_p, tp_d, H):
    assert sorted(kvx.plan_pairs(tp_p, tp_d, H)) == sorted(o1.plan(tp_p, tp_d, H))


def test_plan_pairs_error(kvx):
    with pytest.raises(kvx.KvError):
        kvx.plan_pairs(3, 2, 8)


def test_wire_bytes_is_kv_size_formula(kvx, o1):
    """Per pair: 2 * L * |overlap| * T * D * bytes(wire dtype); summed over pairs = whole KV."""
    for tp_p, tp_d in [(4, 2), (2, 4), (4, 4), (1, 1)]:
        tot = 0
        for p, q, hb, he in kvx.plan_pairs(tp_p, tp_d, 8):
            s = _lay(kvx, tp_degree=tp_p, tp_rank=p, dtype=kvx.KV_BF16)
            d = _lay(kvx, tp_degree=tp_d, tp_rank=q, dtype=kvx.KV_F16)
            tot += kvx.wire_bytes(s, d, 100)
        assert tot == o1.kv_bytes(2, 8, 16, 100, 2)
    # narrowing: the wire carries the narrow dtype (cast on the sender)
    sc = 0x1000  # any non-null pointer value: describe never dereferences scales
    s = _lay(kvx, tp_degree=1, tp_rank=0)
    d = kvx.Layout(2, 8, 16, 1, 0, 4, 10, kvx.KV_F8E4M3, (0, 1, 2, 3, 4, 5), sc)
    assert kvx.wire_dtype(s, d) == kvx.KV_F8E4M3
    assert kvx.wire_bytes(s, d, 100) == o1.kv_bytes(2, 8, 16, 100, 1)
    assert kvx.wire_dtype(d, s) == kvx.KV_F8E4M3  # widening happens on the receiver
    # ranks without overlap move nothing
    s = _lay(kvx, tp_degree=2, tp_rank=0)
    d = _lay(kvx, tp_degree=2, tp_rank=1)
    assert kvx.wire_bytes(s, d, 100) == 0


def _table_update(kvx, lay, n_tokens, ids, buf_bytes=4096):
    from paper_2509_17542_b200._lib import Batch_t, lib
    bt = Batch_t()
    nt = np.asarray(n_tokens, np.int32)
    ids = np.asarray(ids, np.int32)
    return lib.kv_block_table_update(lay.handle, len(nt), nt.ctypes.data, ids.ctypes.data, len(ids), 0x10000,
                                     buf_bytes, C.byref(bt), None), lib.kv_last_error().decode()


def test_block_table_validation_fails_before_enqueue(kvx):
    lay = _lay(kvx)  # B=4, NB=10
    st, msg = _table_update(kvx, lay, [5, 4], [0, 1])
    assert st == 2 and "sum ceil" in msg
    st, msg = _table_update(kvx, lay, [5, 4], [0, 1, 10])
    assert st == 2 and "outside" in msg
    st, msg = _table_update(kvx, lay, [5, 4], [3, 1, 3])
    assert st == 2 and "twice" in msg
    st, msg = _table_update(kvx, lay, [5, -1], [3, 1])
    assert st == 1
    st, msg = _table_update(kvx, lay, [5, 4], [0, 1, 2], buf_bytes=8)
    assert st == 2 and "device buffer" in msg


def test_convert_validation(kvx):
    from paper_2509_17542_b200._lib import Batch_t, lib
    s0 = _lay(kvx, tp_degree=2, tp_rank=0)
    d0 = _lay(kvx, tp_degree=1, tp_rank=0)

    def bt(lay, n_req=1, tokens=5, digest=7):
        b = Batch_t()
        b.n_req, b.block_size, b.num_blocks = n_req, lay.block_size, lay.num_blocks
        b.total_tokens, b.total_blocks, b.token_digest = tokens, 2, digest
        b.tok_off = b.blk_off = b.blk_ids = b.blk_req = b.tok_req = 0x10000
        return b

    def call(src, dst, sbt, dbt, lb=0, le=2):
        S = (C.c_void_p * len(src))(*[l.handle.value for l in src])
        SP = (C.c_void_p * len(src))(*([0x20000] * len(src)))
        D = (C.c_void_p * len(dst))(*[l.handle.value for l in dst])
        DP = (C.c_void_p * len(dst))(*([0x30000] * len(dst)))
        st = lib.kv_convert_reshard(len(src), S, SP, C.byref(sbt), len(dst), D, DP, C.byref(dbt), lb, le, None)
        return st, lib.kv_last_error().decode()

    # merge 2 -> 1 with P rank 1 missing
    st, msg = call([s0], [d0], bt(s0), bt(d0))
    assert st == 2 and "missing source shard for P rank 1" in msg
    # mismatched requests between the P and D tables
    s1 = _lay(kvx, tp_degree=2, tp_rank=1)
    st, msg = call([s0, s1], [d0], bt(s0), bt(d0, digest=8))
    assert st == 2 and "different requests" in msg
    # layer range
    st, msg = call([s0, s1], [d0], bt(s0), bt(d0), 1, 3)
    assert st == 1
    # different models
    dm = _lay(kvx, tp_degree=1, tp_rank=0, head_dim=32)
    st, msg = call([s0, s1], [dm], bt(s0), bt(dm))
    assert st == 2 and "different models" in msg
    # table built for another pool
    d_other = _lay(kvx, tp_degree=1, tp_rank=0, num_blocks=11)
    st, msg = call([s0, s1], [d0], bt(s0), bt(d_other))
    assert st == 2 and "another block size" in msg


def test_wire_header_layout_roundtrip_and_check(kvx):
    """NEXT-2 wire header: documented byte offsets, parse round trip, and the
    check rejects every field that differs."""
    import struct
    from paper_2509_17542_b200 import replay
    s = _lay(kvx, tp_degree=4, tp_rank=1, dtype=kvx.KV_BF16)
    d = kvx.Layout(2, 8, 16, 2, 0, 4, 10, kvx.KV_F8E4M3, (0, 1, 2, 3, 4, 5), 0x1000)
    hdr = replay.header(s, d, [5, 7, 1])
    assert len(hdr) == 72 + 12
    magic, ver, hlen, wdt, H, D, lb, le, tps, tpr, tpd, tqr, hb, he, nreq, res, pay = struct.unpack_from(
        "<4sIIiiiiiiiiiiiiIQ", hdr, 0)
    assert (magic, ver, hlen) == (b"KVX1", 1, 84)
    assert (wdt, H, D, lb, le) == (kvx.KV_F8E4M3, 8, 16, 0, 2)
    assert (tps, tpr, tpd, tqr, hb, he, nreq, res) == (4, 1, 2, 0, 2, 4, 3, 0)
    assert pay == kvx.wire_bytes(s, d, 13) == 2 * 2 * 2 * 13 * 16 * 1
    assert struct.unpack_from("<3i", hdr, 72) == (5, 7, 1)
    info = replay.parse(hdr)
    assert info["n_tokens"] == [5, 7, 1] and info["payload_bytes"] == pay and info["head_end"] == 4
    replay.check_header(hdr, s, d, [5, 7, 1])
    with pytest.raises(kvx.KvError, match="token counts"):
        replay.check_header(hdr, s, d, [5, 7, 2])
    with pytest.raises(kvx.KvError, match="layer range"):
        replay.check_header(hdr, s, d, [5, 7, 1], (0, 1))
    s2 = _lay(kvx, tp_degree=4, tp_rank=0)
    with pytest.raises(kvx.KvError, match="P parallel strategy"):
        replay.check_header(hdr, s2, d, [5, 7, 1])
    with pytest.raises(kvx.KvError, match="bad magic"):
        replay.parse(b"XXXX" + hdr[4:])
    with pytest.raises(kvx.KvError, match="share no heads"):
        replay.header(_lay(kvx, tp_degree=4, tp_rank=3), d, [1])


def test_row_kernels_fit_four_ctas_per_sm():
    """Occupancy guard (CPU, from the cubin): every row-kernel instantiation uses <= 64
    registers and no local memory, so 4 CTAs of 256 threads fit an SM (the bf16 -> e4m3 one
    took 76 registers once and lost 8% of bandwidth); fp8 -> wider casts are capped at 3 CTAs
    (<= 80 registers, KVX_MINB_WIDEN: profiles/r01/minb_occupancy_ab.txt)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2509_17542_b200", "libkvx.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout
    fns = re.findall(r"Function (\S*k_convert_rows\S*):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
    assert len(fns) >= 16
    for name, reg, stack, local in fns:
        # 1-byte sources in 16-element chunks (4 x 16 B in flight) may keep a few bytes on the
        # stack; every other instantiation must stay in registers
        wide_fp8 = re.search(r"k_convert_rowsILi[24]ELi\dELi\dELi16E", name)
        widen = re.search(r"k_convert_rowsILi[24]ELi[013]E", name)
        assert int(reg) <= (80 if widen else 64) and int(local) == 0 and int(stack) <= (32 if wide_fp8 else 0), (name, reg, stack, local)


def test_layout_variants_describe_wire_and_header(kvx, o1):
    """NEXT-3 layout variants (reading 27): kv_part / dim_split validation, pool sizes equal
    the oracle's element counts, the wire carries only the K/V both pools hold, and the
    header's K/V field (offset 60) is written, parsed and checked."""
    import struct
    from paper_2509_17542_b200 import replay
    import synth
    order = (2, 4, 5, 3, 0, 1)   # BLOCK, HEAD, DIM(/x), SLOT, LAYER, KV: an x-packed key cache
    for kp, x in [(0, 0), (1, 8), (2, 0), (1, 4), (0, 16)]:
        l = kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, kv_part=kp, dim_split=x)
        d = synth.layout(2, 8, 16, 2, 1, 4, 10, synth.BF16, order, kv_part=kp, dim_split=x)
        assert l.pool_bytes == o1.pool_elems(d) * 2 == (1 if kp else 2) * 2 * 10 * 4 * 4 * 16 * 2
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, kv_part=3)
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, dim_split=3)    # not a power of two
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):
        kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, dim_split=32)   # does not divide head_dim
    both = _lay(kvx, tp_degree=2, tp_rank=1, dtype=kvx.KV_BF16)
    konly = kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, kv_part=1, dim_split=8)
    vonly = kvx.Layout(2, 8, 16, 2, 1, 4, 10, kvx.KV_BF16, order, kv_part=2)
    assert kvx.wire_bytes(both, konly, 100) == kvx.wire_bytes(both, both, 100) // 2 == 1 * 2 * 4 * 100 * 16 * 2
    assert kvx.wire_bytes(konly, vonly, 100) == 0          # nothing in common
    hdr = replay.header(both, vonly, [5, 7])
    assert struct.unpack_from("<I", hdr, 60)[0] == 2
    assert replay.parse(hdr)["kv_part"] == 2
    replay.check_header(hdr, both, vonly, [5, 7])
    with pytest.raises(kvx.KvError, match="K/V carried"):
        replay.check_header(hdr, both, konly, [5, 7])
    with pytest.raises(kvx.KvError, match="share neither"):
        replay.header(konly, vonly, [1])


def test_pull_and_stage_validation_fails_before_enqueue(kvx):
    """kv_pull / kv_stage / kv_pull_staged reject bad arguments synchronously (no GPU needed:
    nothing is enqueued on these paths)."""
    from paper_2509_17542_b200._lib import Batch_t, lib

    def bt(lay, tokens=5):
        b = Batch_t()
        b.n_req, b.block_size, b.num_blocks = 1, lay.block_size, lay.num_blocks
        b.total_tokens, b.total_blocks, b.token_digest = tokens, 2, 7
        b.tok_off = b.blk_off = b.blk_ids = b.blk_req = b.tok_req = 0x10000
        return b

    def arr(*xs):
        return (C.c_void_p * len(xs))(*xs)

    s = _lay(kvx, tp_degree=1, tp_rank=0)
    d = _lay(kvx, tp_degree=1, tp_rank=0)
    sb, db = bt(s), bt(d)
    err = 0x40000
    # kv_pull: a null ready flag
    st = lib.kv_pull(1, arr(s.handle.value), arr(0x20000), C.byref(sb), d.handle, 0x30000, C.byref(db),
                     arr(0), arr(0x50000), 1, 0, 2, 0, 10**9, err, None)
    assert st == 1 and "null flag" in lib.kv_last_error().decode()
    # kv_pull: K-only source, V-only destination -> nothing in common
    ks = kvx.Layout(2, 8, 16, 1, 0, 4, 10, kvx.KV_BF16, (0, 1, 2, 3, 4, 5), kv_part=1)
    vd = kvx.Layout(2, 8, 16, 1, 0, 4, 10, kvx.KV_BF16, (0, 1, 2, 3, 4, 5), kv_part=2)
    st = lib.kv_pull(1, arr(ks.handle.value), arr(0x20000), C.byref(bt(ks)), vd.handle, 0x30000, C.byref(bt(vd)),
                     arr(0x60000), arr(0x50000), 1, 0, 2, 0, 10**9, err, None)
    assert st == 2 and "share neither" in lib.kv_last_error().decode()
    # kv_stage: ring slots smaller than one layer chunk's wire
    need = kvx.wire_bytes(s, d, 5, (0, 1))
    st = lib.kv_stage(s.handle, 0x20000, C.byref(sb), 1, arr(d.handle.value), arr(0x70000, 0x80000), 2, need - 1,
                      arr(0x60000), arr(0x50000), None, 0, 0, 2, 1, 10**9, err, None)
    assert st == 2 and "ring slots smaller" in lib.kv_last_error().decode()
    # kv_stage: dynamic scales need an fp8 destination
    st = lib.kv_stage(s.handle, 0x20000, C.byref(sb), 1, arr(d.handle.value), arr(0x70000, 0x80000), 2, need,
                      arr(0x60000), arr(0x50000), arr(0x90000), 0, 0, 2, 1, 10**9, err, None)
    assert st == 1 and "dynamic scales" in lib.kv_last_error().decode()
    # kv_pull_staged: no ring slots
    st = lib.kv_pull_staged(1, arr(s.handle.value), arr(0x70000), 0, need, d.handle, 0x30000, C.byref(db),
                            arr(0x60000), arr(0x50000), None, 0, 0, 2, 1, 10**9, err, None)
    assert st == 1 and "bad argument" in lib.kv_last_error().decode()


@pytest.mark.parametrize("lb,le,lc,want", [
    (0, 80, 20, [(0, 20), (20, 40), (40, 60), (60, 80)]),
    (0, 80, 0, [(0, 80)]),
    (0, 80, -20, [(0, 2), (2, 7), (7, 17), (17, 37), (37, 57), (57, 77), (77, 80)]),
    (0, 80, -4, [(0, 1), (1, 2), (2, 4)] + [(l, l + 4) for l in range(4, 80, 4)]),
    (10, 40, -20, [(10, 30), (30, 40)]),          # fewer than two chunks: no ramp
    (0, 80, -3, [(l, min(80, l + 3)) for l in range(0, 80, 3)]),   # |layer_chunk| < 4: no ramp
    (5, 5, -20, []),
    (0, 80, -2**31, [(0, 80)]),                    # |INT32_MIN| saturates: one chunk
])
def test_chunk_count_and_schedule(kvx, lb, le, lc, want):
    """kv_chunk_count: the A10 chunk schedule of kv_stage / kv_pull_staged -- the
    chunks tile [lb, le) in order, uniform |layer_chunk| layers after an optional ramp of
    |layer_chunk|/8, /4, /2 (negative layer_chunk).  Here the expected chunk lists are
    written out by hand; the count must equal their number."""
    assert sum(b - a for a, b in want) == le - lb
    assert all(want[i][1] == want[i + 1][0] for i in range(len(want) - 1))
    assert kvx.chunk_count((lb, le), lc) == len(want)
