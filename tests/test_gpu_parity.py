"""GPU parity: the CUDA path (through the C ABI) against the oracle O1, element by element.

Bar (BASELINE north_star): bit-exact for layout / reshard / fp16 / bf16 / fp32 work; fp8
within 1 e4m3 ulp (ordered-integer distance on sign-magnitude codes, +-0 equal, NaN only
with NaN).  The fp8 path is in fact expected bit-exact (same op order on both sides,
reading 10), and the tests assert the 1-ulp bar plus report the exact-match count.
Whole destination pools are compared, so canary bytes outside the written blocks,
zero-filled tails and never-read source tails are all covered.
"""
import itertools

import numpy as np
import pytest
import torch

import synth
from synth import BF16, E4M3, F16, F32, FNUZ, FP8, LAYER, KV, BLOCK, SLOT, HEAD, DIM
from tests.kvcase import coord_fill, expected, make_case

pytestmark = pytest.mark.gpu

ALL_ORDERS = list(itertools.permutations(range(6)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g   # builds libkvx.so by path (the package needs it to import)
    g.build()


def e4m3_ulp_distance(a, b):
    """Ordered-integer distance between e4m3 codes (sign-magnitude -> two's-line)."""
    def ordv(x):
        x = x.astype(np.int32)
        mag = x & 0x7F
        return np.where(x & 0x80, -mag, mag)
    return np.abs(ordv(a) - ordv(b))


def assert_pools_match(got, want, dtype):
    for g, w in zip(got, want):
        assert g.shape == w.shape
        if dtype != E4M3:
            if not np.array_equal(g, w):
                bad = np.nonzero(g != w)[0]
                raise AssertionError(f"{len(bad)} mismatches, first at {bad[:5]}: got {g[bad[:5]]} want {w[bad[:5]]}")
        else:
            nan_w = (w & 0x7F) == 0x7F
            nan_g = (g & 0x7F) == 0x7F
            assert np.array_equal(nan_w, nan_g), "NaN positions differ"
            d = e4m3_ulp_distance(g[~nan_w], w[~nan_w])
            assert d.max(initial=0) <= 1, f"fp8 beyond 1 ulp: max {d.max()}"


def run_case(o1, case, layer_range=None):
    from tests.gpu_util import DevCase
    dc = DevCase(case)
    dc.convert(layer_range)
    want = expected(case, o1, layer_range)
    got = dc.dst_numpy()
    assert_pools_match(got, want, case["dst_lays"][0]["dtype"])
    return dc, got, want


def test_c1_tiny(o1):
    """configs[0]: 2 layers, 2 kv heads, D 64, 32 tokens, block 16 -> 32, fp16 -> bf16, TP1 -> 1."""
    c = synth.configs()["c1"]
    case = make_case(c.L, c.H, c.D, c.tp_p, c.tp_d, c.B_p, c.B_d, c.n_tokens, c.src_dtype, c.dst_dtype,
                     seed=c.seed, o1=o1)
    run_case(o1, case)


ALL_DT = (F16, BF16, E4M3, F32, FNUZ)


@pytest.mark.parametrize("sdt,ddt", [(s, d) for s in ALL_DT for d in ALL_DT])
def test_all_dtype_pairs(o1, sdt, ddt):
    """Every (src, dst) dtype pair (incl. the e4m3fnuz vendor format, NEXT-3), fast path,
    ragged requests, TP 2 -> 4 split."""
    case = make_case(3, 8, 64, 2, 4, 8, 16, [37, 5, 64, 1], sdt, ddt, seed=10 + 5 * sdt + ddt, o1=o1,
                     scales="amax")
    if sdt in FP8:  # fp8 sources need their own dequant scales
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(500 + i, lay["L"], lay["H"] // lay["tp"], -4, 4) * np.float32(0.75)
    run_case(o1, case)


@pytest.mark.parametrize("src_dt", [F16, BF16])
def test_exhaustive_cast_table_on_device(o1, src_dt):
    """All 65536 source bit patterns through the device cast (pins the NaN encodings,
    reading 12, by device observation)."""
    for dst_dt, scale in [(BF16 if src_dt == F16 else F16, None), (E4M3, 1.0), (E4M3, 5.5 / 448), (F32, None)]:
        L, H, D, B, T = 1, 1, 128, 16, 256
        src = synth.layout(L, H, D, 1, 0, B, T // B, src_dt, (LAYER, KV, BLOCK, SLOT, HEAD, DIM))
        sc = None if scale is None else np.full((L, 2, H), scale, np.float32)
        dst = synth.layout(L, H, D, 1, 0, B, T // B, dst_dt, (LAYER, KV, BLOCK, SLOT, HEAD, DIM), sc)
        pool = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
        from tests.kvcase import NPTYPE
        out = np.zeros(2 * T * D, dtype=NPTYPE[synth.NBYTES[dst_dt]])
        case = dict(src_lays=[src], src_pools=[pool], dst_lays=[dst], dst_pools=[out], n_tokens=[T],
                    src_tables=[list(range(T // B))], dst_tables=[list(range(T // B))])
        dc, got, want = run_case(o1, case)
        if dst_dt == E4M3:
            assert np.array_equal(got[0], want[0]), "fp8 path is expected bit-exact (reading 10)"


def test_exhaustive_fnuz_tables_on_device(o1):
    """e4m3fnuz (NEXT-3) through the device casts, compared bit for bit with O1: all 65536
    bf16 / f16 patterns -> fnuz at scales 1 and 5.5/240; all 256 fnuz codes -> bf16 / f16 /
    f32 / e4m3fn; all 256 e4m3fn codes -> fnuz (dequantise, then quantise: reading 26)."""
    from tests.kvcase import NPTYPE
    o = (LAYER, KV, BLOCK, SLOT, HEAD, DIM)
    runs = [(F16, FNUZ, None, 1.0), (BF16, FNUZ, None, 5.5 / 240), (FNUZ, BF16, 0.75, None),
            (FNUZ, F16, 2.0 ** -3, None), (FNUZ, F32, 1.0, None), (FNUZ, E4M3, 0.5, 1.0), (E4M3, FNUZ, 1.0, 2.0),
            (E4M3, FNUZ, 0.37, 1.3),
            # the fnuz decode folds an exact 2^7 into the source scale when 2^7 s is finite:
            # both sides of that test (2^125 and 1.7e37 overflow it), f32-subnormal scales
            (FNUZ, F32, 2.0 ** 125, None), (FNUZ, F32, 0.37, None), (FNUZ, BF16, 3.3e-41, None),
            (FNUZ, F16, 2.0 ** -140, None), (FNUZ, E4M3, 1.7e37, 3.1e37)]
    for sdt, ddt, ssc, dsc in runs:
        L, H, D, B = 1, 1, 128, 16
        n = 1 << (8 * synth.NBYTES[sdt])
        T = 2 * n // D if synth.NBYTES[sdt] == 2 else 2 * B   # K and V halves hold the patterns
        T = max(T // 2, B)
        pool = np.resize(np.arange(n, dtype=np.uint32).astype(NPTYPE[synth.NBYTES[sdt]]), 2 * T * D)
        s_sc = None if ssc is None else np.full((L, 2, H), ssc, np.float32)
        d_sc = None if dsc is None else np.full((L, 2, H), dsc, np.float32)
        src = synth.layout(L, H, D, 1, 0, B, T // B, sdt, o, s_sc)
        dst = synth.layout(L, H, D, 1, 0, B, T // B, ddt, o, d_sc)
        out = np.zeros(2 * T * D, dtype=NPTYPE[synth.NBYTES[ddt]])
        case = dict(src_lays=[src], src_pools=[pool], dst_lays=[dst], dst_pools=[out], n_tokens=[T],
                    src_tables=[list(range(T // B))], dst_tables=[list(range(T // B))])
        dc, got, want = run_case(o1, case)
        assert np.array_equal(got[0], want[0]), (sdt, ddt)


def test_s532_grid_coordinates(o1):
    """SPEC S:532 grid on the GPU: (tp_p, tp_d) in {1,2,4,8}^2, the 24 layouts, blocks {2,4,8,16},
    2 layers / 8 heads / 16 tokens; coordinate-coded values; D=8 keeps the fast path."""
    orders = [(KV, BLOCK) + p for p in itertools.permutations((LAYER, HEAD, SLOT, DIM))]
    k = 0
    for tp_p in (1, 2, 4, 8):
        for tp_d in (1, 2, 4, 8):
            for i in range(0, 24, 5):
                so, do = orders[i], orders[(i * 7 + tp_p + tp_d) % 24]
                Bp, Bd = (2, 4, 8, 16)[i % 4], (2, 4, 8, 16)[(i // 4 + tp_d) % 4]
                k += 1
                case = make_case(2, 8, 8, tp_p, tp_d, Bp, Bd, [16, 11], F16, F16, so, do, seed=k, o1=o1,
                                 tail_garbage=False)
                coord_fill(case, o1)
                run_case(o1, case)


@pytest.mark.parametrize("i", range(0, 720, 7))
def test_generic_axis_orders(o1, i):
    """Axis orders where head_dim is not innermost take the element-wise path; 103 src/dst
    order pairs spread over all 720 permutations."""
    so, do = ALL_ORDERS[i], ALL_ORDERS[(i * 13 + 5) % 720]
    case = make_case(2, 4, 8, 2, 1, 4, 2, [7, 3], BF16, F16, so, do, seed=i, o1=o1)
    run_case(o1, case)


def test_fast_path_many_layouts(o1):
    """DIM innermost on both sides: all 120 orders of the other five axes as the destination."""
    for i, p in enumerate(itertools.permutations((LAYER, KV, BLOCK, SLOT, HEAD))):
        case = make_case(2, 4, 16, 1, 2, 4, 8, [9, 20], BF16, E4M3, synth.P_ORDER, p + (DIM,), seed=i, o1=o1)
        run_case(o1, case)


def test_layer_chunk_invariance(o1):
    """A10: converting layer chunks separately == all at once (bit-identical)."""
    from tests.gpu_util import DevCase
    case = make_case(6, 8, 32, 4, 2, 16, 64, [100, 33, 64], BF16, BF16, seed=77, o1=o1)
    whole = DevCase(case)
    whole.convert()
    parts = DevCase(case)
    for lr in ((0, 1), (1, 4), (4, 6)):
        parts.convert(lr)
    for a, b in zip(whole.dst_numpy(), parts.dst_numpy()):
        assert np.array_equal(a, b)
    assert_pools_match(whole.dst_numpy(), expected(case, o1), BF16)


def test_subset_of_destination_ranks(o1):
    """Converting only D rank 1 touches only D rank 1 (per-pair dispatch)."""
    from tests.gpu_util import DevCase
    case = make_case(2, 8, 16, 4, 2, 4, 8, [13, 8], F16, BF16, seed=5, o1=o1)
    dc = DevCase(case)
    dc.convert(dst_idx=[1], src_idx=[2, 3])
    got = dc.dst_numpy()
    want = expected(case, o1)
    assert np.array_equal(got[0], case["dst_pools"][0])  # untouched canary
    assert np.array_equal(got[1], want[1])


def test_empty_and_degenerate(o1):
    """T_r = 0 requests, a single token, T a multiple of the block, B_p=1."""
    for n_tokens, Bp, Bd in [([0, 5, 0], 4, 4), ([1], 1, 16), ([32, 16], 16, 16), ([3], 16, 1)]:
        case = make_case(2, 2, 8, 1, 1, Bp, Bd, n_tokens, BF16, F16, seed=len(n_tokens), o1=o1)
        run_case(o1, case)


def test_pack_unpack_vs_flatten_restore(o1):
    """K2/K3 against the oracle's Fig. 5 flatten / restore, per pair, with a narrowing cast."""
    from tests.gpu_util import DevCase, dev_to_np
    import paper_2509_17542_b200 as kvx
    case = make_case(3, 8, 32, 2, 4, 8, 16, [21, 40, 7], BF16, E4M3, seed=3, o1=o1)
    dc = DevCase(case)
    for p, q, _, _ in kvx.plan_pairs(2, 4, 8):
        S, Dl = dc.src_lays[p], dc.dst_lays[q]
        nb = kvx.wire_bytes(S, Dl, dc.src_bt.total_tokens)
        wire = torch.empty(nb, dtype=torch.uint8, device="cuda")
        kvx.pack(S, dc.src_pools[p], dc.src_bt, Dl, wire)
        torch.cuda.synchronize()
        want_wire = o1.flatten(case["src_lays"][p], case["src_pools"][p], case["dst_lays"][q], case["n_tokens"],
                               case["src_tables"])
        assert np.array_equal(dev_to_np(wire, E4M3), want_wire)
        kvx.unpack(S, Dl, dc.dst_pools[q], dc.dst_bt, wire)
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)


def test_pack_unpack_widening_on_receiver(o1):
    """fp8 source -> bf16 destination: the wire carries fp8, the receiver dequantises."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    case = make_case(2, 4, 16, 1, 2, 4, 4, [9, 4], E4M3, BF16, seed=8, o1=o1)
    case["src_lays"][0]["scales"] = synth.pow2_scales(1, 2, 4, -3, 3) * np.float32(1.5)
    dc = DevCase(case)
    for q in range(2):
        S, Dl = dc.src_lays[0], dc.dst_lays[q]
        assert kvx.wire_dtype(S, Dl) == kvx.KV_F8E4M3
        wire = torch.empty(kvx.wire_bytes(S, Dl, dc.src_bt.total_tokens), dtype=torch.uint8, device="cuda")
        kvx.pack(S, dc.src_pools[0], dc.src_bt, Dl, wire)
        kvx.unpack(S, Dl, dc.dst_pools[q], dc.dst_bt, wire)
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), BF16)


@pytest.mark.parametrize("tp_p,tp_d,Bp,Bd,dorder,dt", [
    (4, 2, 16, 64, "head", BF16),   # merge, 4 source blocks per destination block (c3 shape)
    (2, 1, 16, 16, "head", F16),    # merge into one D rank, whole head rows (c2 shape)
    (2, 4, 8, 8, "slot", F16),      # split, D inner (SLOT, HEAD, DIM)
    (4, 4, 16, 32, "slot", BF16),   # 1:1, two source blocks per destination block
    (1, 1, 4, 4, "head", F32),      # fp32 rows
])
def test_tma_tile_path_forced(o1, monkeypatch, tp_p, tp_d, Bp, Bd, dorder, dt):
    """The same-dtype TMA tile path (KVX_TILE=2 forces it for every sub-tile size): tensor
    map in D's order, tail rows zeroed in smem, bulk stores; ragged requests incl. T = 0 and
    requests shorter than a block; also per-P-rank shares."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    monkeypatch.setenv("KVX_TILE", "2")
    d_order = synth.D_ORDER if dorder == "head" else (BLOCK, LAYER, KV, SLOT, HEAD, DIM)
    n_tokens = [Bd * 3 + 5, 0, 1, Bp - 1, Bd]
    case = make_case(3, 8, 64, tp_p, tp_d, Bp, Bd, n_tokens, dt, dt, synth.P_ORDER, d_order,
                     seed=40 + tp_p + Bd, o1=o1)
    kvx.launch_count_reset()
    run_case(o1, case)
    # the same transfer as per-P-rank shares (distributed push primitive)
    case2 = make_case(3, 8, 64, tp_p, tp_d, Bp, Bd, n_tokens, dt, dt, synth.P_ORDER, d_order,
                      seed=40 + tp_p + Bd, o1=o1)
    dc = DevCase(case2)
    for p, q, _, _ in kvx.plan_pairs(tp_p, tp_d, 8):
        kvx.convert_share(dc.src_lays[p], dc.src_pools[p], dc.src_bt, [dc.dst_lays[q]], [dc.dst_pools[q]], dc.dst_bt)
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case2, o1), dt)


def test_tma_tile_and_row_paths_agree(o1, monkeypatch):
    """KVX_TILE=0 (row kernel) and KVX_TILE=2 (TMA tile) give identical pools on a c2-shaped case."""
    from tests.gpu_util import DevCase
    case = make_case(4, 32, 128, 2, 1, 16, 16, [300, 17], F16, F16, seed=9, o1=o1)
    outs = []
    for mode in ("0", "2"):
        monkeypatch.setenv("KVX_TILE", mode)
        dc = DevCase(case)
        dc.convert()
        outs.append(dc.dst_numpy())
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert_pools_match(outs[1], expected(case, o1), F16)


@pytest.mark.parametrize("vec_path", [True, False])
def test_redzones_untouched(o1, vec_path):
    """compute-sanitizer is closed on this pool, so out-of-bounds writes are caught with
    red zones: every pool (and the wire) sits inside a larger canary-filled buffer and the
    bytes around it must survive a convert, a pack and an unpack."""
    import paper_2509_17542_b200 as kvx
    RZ = 4096
    order_p = synth.P_ORDER if vec_path else (LAYER, KV, BLOCK, DIM, SLOT, HEAD)
    case = make_case(3, 8, 32, 2, 4, 8, 16, [21, 9], BF16, E4M3, order_p, synth.D_ORDER, seed=17, o1=o1,
                     scales="pow2")

    def embed(arr):
        raw = np.ascontiguousarray(arr).view(np.uint8)
        big = torch.full((raw.size + 2 * RZ,), 0x5A, dtype=torch.uint8, device="cuda")
        big[RZ:RZ + raw.size] = torch.from_numpy(raw.copy()).cuda()
        return big, big[RZ:RZ + raw.size]

    def intact(big, n):
        return bool((big[:RZ] == 0x5A).all()) and bool((big[RZ + n:] == 0x5A).all())

    src = [embed(p) for p in case["src_pools"]]
    dst = [embed(p) for p in case["dst_pools"]]
    S = [kvx.Layout.from_dict(l) for l in case["src_lays"]]
    Dl = [kvx.Layout.from_dict(l, torch.from_numpy(np.asarray(l["scales"], np.float32)).cuda()) for l in case["dst_lays"]]
    sbt = kvx.Batch(S[0], case["n_tokens"], case["src_tables"])
    dbt = kvx.Batch(Dl[0], case["n_tokens"], case["dst_tables"])
    kvx.convert_reshard(S, [v for _, v in src], sbt, Dl, [v for _, v in dst], dbt)
    nb = kvx.wire_bytes(S[0], Dl[0], sbt.total_tokens)
    wbig = torch.full((nb + 2 * RZ,), 0x5A, dtype=torch.uint8, device="cuda")
    kvx.pack(S[0], src[0][1], sbt, Dl[0], wbig[RZ:RZ + nb])
    kvx.unpack(S[0], Dl[0], dst[0][1], dbt, wbig[RZ:RZ + nb])
    torch.cuda.synchronize()
    for big, view in src + dst:
        assert intact(big, view.numel())
    assert intact(wbig, nb)
    got = [v.cpu().numpy().view(np.uint8) for _, v in dst]
    want = expected(case, o1)
    assert_pools_match([g for g in got], [w.view(np.uint8) for w in want], E4M3)


def test_launch_count_and_errors():
    import paper_2509_17542_b200 as kvx
    kvx.launch_count_reset()
    lay = kvx.Layout(1, 2, 8, 1, 0, 4, 4, kvx.KV_BF16, synth.P_ORDER)
    bt = kvx.Batch(lay, [5], [[0, 1]])
    pools = [lay.new_pool(fill=0), lay.new_pool(fill=0)]
    kvx.convert_reshard([lay], [pools[0]], bt, [lay], [pools[1]], bt)
    torch.cuda.synchronize()
    assert kvx.launch_count() == 1
    with pytest.raises(kvx.KvError, match="KV_ESHAPE"):
        kvx.Batch(lay, [5], [[0, 9]])


@pytest.mark.parametrize("tp_p,tp_d,sdt,ddt", [(2, 1, F16, F16), (1, 2, BF16, E4M3), (4, 2, BF16, BF16)])
def test_pipeline_stage_reshard(o1, tp_p, tp_d, sdt, ddt):
    """NEXT-2: P stages [0,2),[2,4) -> D stages [0,3),[3,4), one device call per overlapping
    stage pair over the intersection, == the oracle's staged transfer (pinned against O2)."""
    from tests.gpu_util import DevCase
    from tests.test_oracle_pp import D_STAGES, P_STAGES, _pools_for, _staged, staged_transfer
    import paper_2509_17542_b200 as kvx
    base = make_case(4, 8, 64, tp_p, tp_d, 16, 32, [70, 5], sdt, ddt, seed=tp_p + 7 * tp_d, o1=None,
                     tail_garbage=False, scales="pow2")
    src, dst = _staged(base, P_STAGES, "src"), _staged(base, D_STAGES, "dst")
    case = dict(src_lays=src, src_pools=_pools_for(src, 300, sdt), dst_lays=dst,
                dst_pools=_pools_for(dst, 0, ddt, canary=True), n_tokens=base["n_tokens"],
                src_tables=base["src_tables"], dst_tables=base["dst_tables"])
    dc = DevCase(case)
    for sf, se in P_STAGES:
        si = [i for i, d in enumerate(src) if d["first_layer"] == sf]
        for df, de in D_STAGES:
            lb, le = max(sf, df), min(se, de)
            if lb < le:
                di = [i for i, d in enumerate(dst) if d["first_layer"] == df]
                kvx.convert_reshard([dc.src_lays[i] for i in si], [dc.src_pools[i] for i in si], dc.src_bt,
                                    [dc.dst_lays[i] for i in di], [dc.dst_pools[i] for i in di], dc.dst_bt, (lb, le))
    torch.cuda.synchronize()
    want = [p.copy() for p in case["dst_pools"]]
    staged_transfer(o1, src, case["src_pools"], dst, want, case["n_tokens"], case["src_tables"], case["dst_tables"])
    assert_pools_match(dc.dst_numpy(), want, ddt)
    with pytest.raises(kvx.KvError, match="KV_EINVAL"):  # range outside the P stage
        kvx.convert_reshard(dc.src_lays[:tp_p], dc.src_pools[:tp_p], dc.src_bt, dc.dst_lays[:tp_d],
                            dc.dst_pools[:tp_d], dc.dst_bt, (1, 3))


@pytest.mark.parametrize("tp_p,tp_d,ddt", [(4, 2, BF16), (2, 4, E4M3), (4, 4, E4M3), (2, 1, F16), (1, 2, F16)])
def test_convert_share_per_p_rank(o1, tp_p, tp_d, ddt):
    """Distributed push primitive: each P rank converts only its own heads into every D rank
    it shares heads with (fan-in and fan-out); all shares together == the whole transfer."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    case = make_case(3, 8, 64, tp_p, tp_d, 16, 32, [45, 16, 3], F16 if ddt == F16 else BF16, ddt,
                     seed=30 + tp_p * 5 + tp_d, o1=o1, scales="pow2")
    dc = DevCase(case)
    pairs = kvx.plan_pairs(tp_p, tp_d, 8)
    for p in range(tp_p):
        qs = sorted(q for pp, q, _, _ in pairs if pp == p)
        kvx.convert_share(dc.src_lays[p], dc.src_pools[p], dc.src_bt, [dc.dst_lays[q] for q in qs],
                          [dc.dst_pools[q] for q in qs], dc.dst_bt)
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), ddt)
    if tp_p > tp_d > 1:  # a D rank that P rank 0 does not feed is refused
        with pytest.raises(kvx.KvError, match="holds no head"):
            kvx.convert_share(dc.src_lays[0], dc.src_pools[0], dc.src_bt, [dc.dst_lays[tp_d - 1]],
                              [dc.dst_pools[tp_d - 1]], dc.dst_bt)


def test_replay_from_file_and_hidden_state(o1, tmp_path):
    """NEXT-2: every (p, q) share packed, saved as header + payload, loaded back, header-checked
    and unpacked == the oracle; a mismatching receiver is refused.  Plus the opaque hidden
    state copy."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    from paper_2509_17542_b200 import replay
    case = make_case(3, 8, 32, 4, 2, 8, 16, [19, 40], BF16, E4M3, seed=12, o1=o1, scales="pow2")
    dc = DevCase(case)
    for p, q, _, _ in kvx.plan_pairs(4, 2, 8):
        path = str(tmp_path / f"kv_{p}_{q}.kvx")
        replay.save(path, dc.src_lays[p], dc.src_pools[p], dc.src_bt, dc.dst_lays[q])
        info = replay.load(path, dc.src_lays[p], dc.dst_lays[q], dc.dst_pools[q], dc.dst_bt)
        assert info["src_tp_rank"] == p and info["dst_tp_rank"] == q
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)
    with pytest.raises(kvx.KvError, match="P parallel strategy"):
        replay.load(str(tmp_path / "kv_0_0.kvx"), dc.src_lays[1], dc.dst_lays[0], dc.dst_pools[0], dc.dst_bt)
    h = torch.randint(0, 255, (16384 + 3,), dtype=torch.uint8, device="cuda")
    out = torch.zeros(16384 + 8, dtype=torch.uint8, device="cuda")
    replay.copy_hidden(out[5:], h)  # misaligned destination on purpose
    torch.cuda.synchronize()
    assert torch.equal(out[5:5 + h.numel()], h) and int(out[:5].sum()) == 0


@pytest.mark.parametrize("sdt", [F16, BF16, E4M3])
def test_dynamic_scales_then_convert(o1, sdt):
    """NEXT-1: device amax/448 scales == oracle bit-exactly; converting with them == oracle."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    case = make_case(3, 8, 64, 4, 2, 16, 32, [70, 13, 1], sdt, E4M3, seed=60 + sdt, o1=o1, scales=1.0)
    if sdt == E4M3:
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(80 + i, 3, 2, -3, 3) * np.float32(1.25)
    dc = DevCase(case)
    for q, dl in enumerate(dc.dst_lays):
        out = torch.full((3, 2, 4), -1.0, dtype=torch.float32, device="cuda")
        kvx.compute_scales(dc.src_lays, dc.src_pools, dc.src_bt, dl, out)
        torch.cuda.synchronize()
        want = o1.amax_scales(case["src_lays"], case["src_pools"], case["dst_lays"][q], case["n_tokens"],
                              case["src_tables"])
        assert np.array_equal(out.cpu().numpy(), want)
        # use them: the destination layout now carries the dynamic scales
        case["dst_lays"][q]["scales"] = want
        dl.scales.copy_(out.view(dl.scales.shape))
    dc.convert()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), E4M3)


@pytest.mark.parametrize("order_i,ddt", [(0, E4M3), (201, E4M3), (0, FNUZ), (517, FNUZ)])
def test_dynamic_scales_row_and_generic_paths(o1, order_i, ddt):
    """kv_compute_scales on both amax kernels -- the row path (head_dim innermost) and the
    element-wise path (any other source order) -- against O1, for e4m3fn (amax/448) and
    e4m3fnuz (amax/240) destinations, with a ragged batch over several token groups."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    so = synth.P_ORDER if order_i == 0 else ALL_ORDERS[order_i]
    case = make_case(2, 4, 32, 2, 1, 8, 16, [700, 33, 1, 290], BF16, ddt, so, seed=90 + order_i, o1=o1, scales=1.0)
    dc = DevCase(case)
    out = torch.full((2, 2, 4), -1.0, dtype=torch.float32, device="cuda")
    kvx.compute_scales(dc.src_lays, dc.src_pools, dc.src_bt, dc.dst_lays[0], out)
    torch.cuda.synchronize()
    want = o1.amax_scales(case["src_lays"], case["src_pools"], case["dst_lays"][0], case["n_tokens"],
                          case["src_tables"])
    assert np.array_equal(out.cpu().numpy(), want)


# ---- NEXT-3 layout variants (reading 27): K-only / V-only pools, x-split head_dim ---------
_HELD = {0: (0, 1), 1: (0,), 2: (1,)}


@pytest.mark.parametrize("seed", range(12))
def test_layout_variants_convert_and_wire(o1, seed):
    """Random K-only / V-only / both pools with and without an x-split head_dim on either
    side, every path: the fused convert and pack -> unpack per pair, bit-exact vs O1."""
    from tests.gpu_util import DevCase, dev_to_np
    import paper_2509_17542_b200 as kvx
    rng = np.random.default_rng(2000 + seed)
    tp_p, tp_d = [(2, 1), (1, 2), (2, 2), (4, 2)][seed % 4]
    pk = int(rng.integers(0, 3))
    dk = int(rng.choice([k for k in range(3) if set(_HELD[k]) & set(_HELD[pk])]))
    px, dx = int(rng.choice([0, 8, 16])), int(rng.choice([0, 8, 16]))
    sdt, ddt = [(BF16, BF16), (BF16, E4M3), (F16, FNUZ), (E4M3, BF16)][seed % 4]
    so, do = ALL_ORDERS[int(rng.integers(720))], ALL_ORDERS[int(rng.integers(720))]
    case = make_case(2, 8, 32, tp_p, tp_d, 4, 8, [13, 40, 1], sdt, ddt, so, do, seed=seed, o1=o1, scales="pow2",
                     p_kv_part=pk, d_kv_part=dk, p_split=px, d_split=dx)
    if sdt in FP8:
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(600 + i, 2, 8 // tp_p, -3, 3)
    run_case(o1, case)
    dc = DevCase(case)
    for p, q, _, _ in kvx.plan_pairs(tp_p, tp_d, 8):
        S, Dl = dc.src_lays[p], dc.dst_lays[q]
        wire = torch.empty(max(16, kvx.wire_bytes(S, Dl, dc.src_bt.total_tokens)), dtype=torch.uint8, device="cuda")
        kvx.pack(S, dc.src_pools[p], dc.src_bt, Dl, wire)
        torch.cuda.synchronize()
        want_wire = o1.flatten(case["src_lays"][p], case["src_pools"][p], case["dst_lays"][q], case["n_tokens"],
                               case["src_tables"])
        assert np.array_equal(dev_to_np(wire, kvx.wire_dtype(S, Dl))[:want_wire.size], want_wire)
        kvx.unpack(S, Dl, dc.dst_pools[q], dc.dst_bt, wire)
    torch.cuda.synchronize()
    assert_pools_match(dc.dst_numpy(), expected(case, o1), ddt)


def test_other_vendor_prefill_to_nvidia_decode(o1):
    """The multi-vendor pairing end to end on one GPU: a P instance whose engine keeps an
    x-packed key cache ([LAYER], BLOCK, HEAD, D/8, SLOT, x=8) and a head_dim-major value
    cache ([LAYER], BLOCK, HEAD, DIM, SLOT) in two pools, fp8 e4m3fnuz with per-head scales, TP2 ->
    a D instance with one block-major K+V pool in OCP e4m3fn, TP1 (merge), block 16 -> 32.
    Two convert calls (K, then V) == O1 on the same pools."""
    from tests.gpu_util import DevCase
    import paper_2509_17542_b200 as kvx
    korder = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)   # per-layer tensors, KV extent 1; x-split below
    vorder = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)   # head_dim-major: k_convert_tr
    args = (3, 8, 64, 2, 1, 16, 32, [70, 5, 33], FNUZ, E4M3)
    kw = dict(d_order=synth.D_ORDER, seed=77, o1=o1, scales="pow2")
    kc = make_case(*args, p_order=korder, p_kv_part=1, p_split=8, **kw)
    vc = make_case(*args, p_order=vorder, p_kv_part=2, **kw)
    for c in (kc, vc):
        for i, lay in enumerate(c["src_lays"]):
            lay["scales"] = synth.pow2_scales(700 + i, 3, 4, -2, 2)
    # one D pool receives both calls
    dk_ = DevCase(kc)
    dv_ = DevCase(vc)
    dv_.dst_pools = dk_.dst_pools
    dk_.convert()
    assert kvx.last_kernel() == "k_convert_tr8"       # x-split (D/x, SLOT, x) tiles: register sub-blocks
    dv_.convert()
    assert kvx.last_kernel() == "k_convert_tr8"       # head_dim-major: register 8 x 8 transposes
    want = expected(kc, o1)
    want = [w.copy() for w in want]
    o1.convert(vc["src_lays"], vc["src_pools"], vc["dst_lays"], want, vc["n_tokens"], vc["src_tables"],
               vc["dst_tables"])
    assert_pools_match(dk_.dst_numpy(), want, E4M3)


@pytest.mark.parametrize("dt,Bp,Bd,D", [(BF16, 16, 16, 128), (BF16, 32, 64, 64), (F16, 8, 16, 128), (E4M3, 16, 32, 64)])
@pytest.mark.parametrize("tr", ["0", "1"])
def test_head_dim_major_source_tiles(o1, monkeypatch, tr, dt, Bp, Bd, D):
    """A head_dim-major ((DIM, SLOT) innermost) source through both transpose kernels
    (KVX_TR=0: k_convert_tr, shared-memory tiles; 1: k_convert_tr8, register 8 x 8
    sub-blocks), 2-byte and fp8 sources, ragged requests, TP 2 -> 1."""
    import paper_2509_17542_b200 as kvx
    monkeypatch.setenv("KVX_TR", tr)
    vorder = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)
    ddt = BF16 if dt == E4M3 else E4M3
    case = make_case(2, 4, D, 2, 1, Bp, Bd, [70, 1, 33, 0], dt, ddt, vorder, synth.D_ORDER, seed=Bp + D, o1=o1,
                     scales="pow2")
    if dt in FP8:
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(800 + i, 2, 2, -2, 2)
    run_case(o1, case)
    tb = tr == "1" and dt != F32 and Bp == Bd == 16 and D in (64, 128, 256)
    assert kvx.last_kernel() == ("k_convert_tb" if tb else "k_convert_tr8" if tr == "1" else "k_convert_tr")


_VCOL = (LAYER, KV, BLOCK, HEAD, DIM, SLOT)   # head_dim-major tile (other vendors' value cache)
# side forms: (axis order, x-split): rows = head_dim innermost, col = (DIM, SLOT) innermost,
# x8 / x16 = (D/x, SLOT, x) innermost (other vendors' key cache)
_FORMS = {"rows_p": (synth.P_ORDER, 0), "rows_d": (synth.D_ORDER, 0), "col": (_VCOL, 0), "x8": (_VCOL, 8),
          "x16": (_VCOL, 16)}


@pytest.mark.parametrize("sf,df,sdt,ddt,Bp,Bd,tp", [
    ("col", "rows_d", BF16, E4M3, 16, 16, (2, 1)),
    ("x8", "rows_d", BF16, E4M3, 16, 16, (2, 1)),
    ("rows_p", "col", E4M3, BF16, 8, 32, (1, 2)),
    ("rows_p", "x16", F16, F16, 16, 64, (2, 2)),
    ("col", "col", FNUZ, E4M3, 8, 16, (2, 1)),
    ("x16", "col", F32, BF16, 16, 16, (1, 1)),
    ("col", "x8", E4M3, FNUZ, 16, 32, (4, 2)),
    ("x8", "x16", BF16, BF16, 8, 8, (1, 2)),
    ("col", "rows_d", F32, F32, 8, 64, (2, 1)),
    ("col", "rows_d", E4M3, E4M3, 32, 32, (1, 1)),
])
def test_tr8_forms(o1, monkeypatch, sf, df, sdt, ddt, Bp, Bd, tp):
    """k_convert_tr8 over every pairing of side forms (rows / head_dim-major / x-packed),
    each dtype width on the transpose (1, 2, 4 bytes), block growth with several source
    blocks per destination block, ragged requests (0, 1 and non-multiple-of-8 tokens), TP
    split and merge: bit-exact vs O1, and identical to the shared-memory kernel."""
    import paper_2509_17542_b200 as kvx
    monkeypatch.setenv("KVX_TB", "0")   # the register kernel itself (k_convert_tb: test_tb_tiles)
    (so, px), (do, dx) = _FORMS[sf], _FORMS[df]
    case = make_case(2, 8, 64, tp[0], tp[1], Bp, Bd, [70, 0, 1, 37, 129], sdt, ddt, so, do, seed=Bp * 7 + Bd,
                     o1=o1, scales="pow2", p_split=px, d_split=dx)
    if sdt in FP8:
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(900 + i, 2, 8 // tp[0], -2, 2)
    got = {}
    for tr in ("1", "0"):
        monkeypatch.setenv("KVX_TR", tr)
        _, got[tr], _ = run_case(o1, case)
        assert kvx.last_kernel() == ("k_convert_tr8" if tr == "1" else "k_convert_tr")
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("sdt,ddt,Bp,Bd,tp,do", [
    (BF16, BF16, 16, 16, (2, 1), "rows_d"),
    (F16, BF16, 16, 64, (1, 2), "rows_p"),
    (BF16, F16, 32, 32, (2, 2), "x8"),
])
def test_tr8_w16(o1, monkeypatch, sdt, ddt, Bp, Bd, tp, do):
    """k_convert_tr8's W16 sub-blocks (2-byte head_dim-major source, 2-byte destination,
    blocks of >= 16 slots: one 256-bit load per 32-B head_dim row, two 8 x 8 transposes),
    ragged requests, on and off (KVX_TR_W16=0): bit-exact vs O1 both ways."""
    import paper_2509_17542_b200 as kvx
    monkeypatch.setenv("KVX_TB", "0")
    (so, _), (dord, dx) = _FORMS["col"], _FORMS[do]
    case = make_case(2, 8, 64, tp[0], tp[1], Bp, Bd, [70, 0, 1, 37, 129, 16], sdt, ddt, so, dord, seed=Bp + Bd + 5,
                     o1=o1, d_split=dx)
    for w in ("1", "0"):
        monkeypatch.setenv("KVX_TR_W16", w)
        run_case(o1, case)
        assert kvx.last_kernel() == "k_convert_tr8"


@pytest.mark.parametrize("sdt,ddt,D,tp,n_tokens,split", [
    (BF16, E4M3, 128, (2, 1), [70, 0, 1, 37, 129, 16], 0),
    (BF16, BF16, 128, (1, 1), [300, 15, 17], 0),
    (F16, FNUZ, 64, (2, 4), [33, 64, 1], 0),
    (BF16, F32, 256, (1, 2), [48, 5], 0),
    (F16, F16, 128, (4, 2), [1000, 3, 0, 31], 0),
    (E4M3, BF16, 128, (2, 1), [70, 0, 1, 37], 0),
    (FNUZ, E4M3, 128, (2, 2), [129, 16, 3], 0),
    (FNUZ, F32, 64, (1, 2), [40, 17], 0),
    (E4M3, E4M3, 256, (2, 1), [33, 1], 0),
    # x-packed (D/x, SLOT, x) tiles with x = 16 bytes (other vendors' key cache)
    (BF16, E4M3, 128, (2, 1), [70, 0, 1, 37], 8),
    (F16, BF16, 64, (2, 4), [129, 16], 8),
    (BF16, F32, 256, (1, 2), [17, 48], 8),
])
def test_tb_tiles(o1, monkeypatch, sdt, ddt, D, tp, n_tokens, split):
    """k_convert_tb (head_dim-major 1- or 2-byte source tiles of 16 slots through TMA, swizzled
    shared-memory stages, warp-specialised producer / consumers) into D's rows: bit-exact vs
    O1 and identical to k_convert_tr8 (KVX_TB=0), ragged requests (0, 1, 15, 17 tokens),
    TP merge and split, every destination dtype width."""
    import paper_2509_17542_b200 as kvx
    case = make_case(3, 8, D, tp[0], tp[1], 16, 16, n_tokens, sdt, ddt, _VCOL, synth.D_ORDER,
                     seed=D + tp[0] * 10 + tp[1] + sdt + split, o1=o1, scales="pow2", p_split=split)
    if sdt in FP8:
        for i, lay in enumerate(case["src_lays"]):
            lay["scales"] = synth.pow2_scales(950 + i, 3, 8 // tp[0], -2, 2)
    got = {}
    for tb in ("1", "0"):
        monkeypatch.setenv("KVX_TB", tb)
        _, got[tb], _ = run_case(o1, case)
        assert kvx.last_kernel() == ("k_convert_tb" if tb == "1" else "k_convert_tr8")
    for a, b in zip(got["1"], got["0"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("sdt,ddt", [(FNUZ, E4M3), (E4M3, FNUZ)])
@pytest.mark.parametrize("codes", ["random", "all"])
@pytest.mark.parametrize("form", ["col", "xpack"])
def test_tb_requant_tables(o1, monkeypatch, sdt, ddt, codes, form):
    """fp8 -> other fp8 from other vendors' tiles -- head_dim-major V (form="col") and
    x-packed K with x = 16 codes (form="xpack"; through tb for e4m3fn -> fnuz only):
    k_convert_tb's per-item code tables (two heads per TMA box) vs its arithmetic cast
    (KVX_TB_LUT=0) and vs k_convert_tr8 (KVX_TB=0)
    -- all identical and equal to O1: random non-power-of-two scales on both sides, NaN
    codes, and (codes="all") every one of the 256 codes in every tile, ragged requests, TP
    split."""
    import paper_2509_17542_b200 as kvx
    so, split = (_VCOL, 0) if form == "col" else ((LAYER, KV, BLOCK, HEAD, DIM, SLOT), 16)
    case = make_case(3, 8, 128, 2, 4, 16, 16, [129, 16, 3, 0, 40], sdt, ddt, so, synth.D_ORDER, seed=77,
                     o1=o1, scales="amax", p_split=split)
    rng = np.random.default_rng(78)
    for lay in case["src_lays"]:
        lay["scales"] = np.exp(rng.uniform(np.log(0.01), np.log(100), size=(3, 2, 4))).astype(np.float32)
    for p_ in case["src_pools"]:
        if codes == "all":
            p_.view(np.uint8)[:] = (np.arange(p_.size) * 7 % 256).astype(np.uint8)
        else:
            p_[::97] = 0x80 if sdt == FNUZ else 0x7F
            p_[5::101] = 0xFF if sdt == E4M3 else 0x7F
    got = {}
    runs = [("1", "1"), ("1", "0"), ("0", "1"), ("0", "0")]   # (KVX_TB, table paths on)
    for tb, lut in runs:
        monkeypatch.setenv("KVX_TB", tb)
        monkeypatch.setenv("KVX_TB_LUT", lut)
        _, got[(tb, lut)], _ = run_case(o1, case)
        want_k = "k_convert_tb" if tb == "1" and (form == "col" or ddt == FNUZ) else "k_convert_tr8"
        assert kvx.last_kernel() == want_k
    for r in runs[1:]:
        for a, b in zip(got[runs[0]], got[r]):
            assert np.array_equal(a, b), r


@pytest.mark.parametrize("tp_p,tp_d", [(1, 1), (1, 2), (2, 1)])
def test_tile_copy_head_groups(o1, tp_p, tp_d):
    """k_tile_copy with sub-tiles over 64 KB (32 heads x 16 slots x 256 B): split into
    head groups, each with its own P rank and local head offsets (and the share path)."""
    import paper_2509_17542_b200 as kvx
    from tests.gpu_util import DevCase
    case = make_case(2, 64, 128, tp_p, tp_d, 16, 16, [40, 3, 16], BF16, BF16, seed=30 + tp_p * 3 + tp_d, o1=o1)
    run_case(o1, case)
    assert kvx.last_kernel() == "k_tile_copy"
    if tp_p > tp_d:   # per P rank share (the distributed-push primitive) over head groups
        dc = DevCase(case)
        for p in range(tp_p):
            kvx.convert_share(dc.src_lays[p], dc.src_pools[p], dc.src_bt, dc.dst_lays, dc.dst_pools, dc.dst_bt)
        torch.cuda.synchronize()
        assert_pools_match(dc.dst_numpy(), expected(case, o1), BF16)


@pytest.mark.parametrize("codes", ["random", "all"])
@pytest.mark.parametrize("sdt,ddt", [(FNUZ, E4M3), (E4M3, FNUZ)])
@pytest.mark.parametrize("tp,L", [((2, 4), 3), ((4, 2), 2), ((1, 1), 200)])
def test_requant_tables(o1, monkeypatch, sdt, ddt, tp, L, codes):
    """fp8 -> other fp8 through shared-memory code tables (k_requant_rows: 128 magnitude
    entries per table, the sign and the special codes restored per byte): bit-identical to
    the arithmetic row kernel (KVX_LUT=0) and to O1, random codes including the NaN codes of
    both formats (codes="all": every one of the 256 codes in every row region, both signs of
    zero and of every underflow), random (non-power-of-two) scales on both sides, ragged
    requests, TP split / merge, and a layer count whose tables exceed one launch (200 layers
    x 2 x 8 heads)."""
    import paper_2509_17542_b200 as kvx
    case = make_case(L, 8, 64, tp[0], tp[1], 16, 16, [37, 0, 16, 1], sdt, ddt, seed=60 + L + tp[0],
                     o1=o1, scales="amax")
    rng = np.random.default_rng(61)
    for lay in case["src_lays"]:
        lay["scales"] = np.exp(rng.uniform(np.log(0.01), np.log(100), size=(L, 2, 8 // tp[0]))).astype(np.float32)
    for p_ in case["src_pools"]:   # NaN codes too (synth avoids them): 0x7F / 0xFF in fn, 0x80 in fnuz
        if codes == "all":         # 7 is odd: each 64-element row holds 64 distinct codes, all 256 cycle
            p_.view(np.uint8)[:] = (np.arange(p_.size) * 7 % 256).astype(np.uint8)
            continue
        p_[::97] = 0x80 if sdt == FNUZ else 0x7F
        p_[5::101] = 0xFF if sdt == E4M3 else 0x7F
    got = {}
    for lut in ("2", "0"):   # 2: tables whatever the direction; 0: the arithmetic row kernel
        monkeypatch.setenv("KVX_LUT", lut)
        _, got[lut], _ = run_case(o1, case)
        assert kvx.last_kernel() == ("k_requant_rows" if lut == "2" else "k_convert_rows")
    for a, b in zip(got["2"], got["0"]):
        assert np.array_equal(a, b)
