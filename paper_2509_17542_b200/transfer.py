"""P -> D transfer across GPUs of one box (A8, A10, A11): roles, pair plan, control-plane
exchange and the data-plane modes (bench.py default: pull).

* ``push`` (the fused kernel K4): each D rank exports its pool and a completion
  flag through CUDA IPC; each P rank maps them and runs ``convert_reshard`` with the
  *peer-mapped* D pool as destination -- one kernel gathers from local HBM, converts and
  stores straight into the D rank's HBM across NVLink -- then ``signal``s the flag with a
  system-scope release.  The D rank ``wait``s (acquire) on its local flag.  The cast
  happens on the sender, so a narrowing cast halves the NVLink bytes (hard
  part 2).  D keeps control of placement: its block table (and fp8 scales) travel to P
  through the control plane (``ControlPlane``, A3).
* ``pull`` (the paper's direction, "read(local, remote, location)"): each P rank
  exports its pool (same-width / widening cast) or a staging ring (narrowing cast) plus a
  flag array; each D rank maps them and reads across NVLink.  Without narrowing, D runs
  ``kv.pull`` -- one convert_reshard per layer chunk with the peer-mapped P pools as
  sources -- after P's ready flag, then releases P with a done flag.  With narrowing, P
  ``kv.stage``s (packs + casts) each layer chunk into a ring slot and D ``kv.pull_staged``s
  it (unpack reading the peer slot), so the link carries the narrow bytes.  SM loads from
  a peer move more user bytes per second than SM stores to a peer.
* ``nccl`` (baseline): P ``pack``s each pair's share into a wire buffer (canonical
  Fig. 5 order), ``Comm.send``s it; D ``recv``s and ``unpack``s; per-layer chunks are
  pipelined on two streams (pack chunk k+1 while chunk k is on the wire).

Ranks: the first ``n_p`` ranks of the job are the P instance's TP ranks, the next ``n_d``
the D instance's (disjoint GPU groups, north_star).  The pair plan is A2.
torch.distributed is the control plane only (object exchange, barriers).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import kv


@dataclass
class Role:
    kind: str        # "P" or "D"
    tp_rank: int     # rank inside its instance
    world_rank: int


def roles(world_size: int, n_p: int, n_d: int, allow_idle: bool = False):
    """Global rank -> Role; P ranks first, then D ranks (disjoint GPU groups); with
    allow_idle, ranks beyond n_p + n_d are idle ("X": they only join the barriers)."""
    if n_p + n_d != world_size and not (allow_idle and n_p + n_d < world_size):
        raise ValueError(f"world_size {world_size} != n_p {n_p} + n_d {n_d}")
    return [Role("P", r, r) if r < n_p else Role("D", r - n_p, r) if r < n_p + n_d else Role("X", -1, r)
            for r in range(world_size)]


def present_ranks(tp_p: int, tp_d: int, world_size: int):
    """How many P and D TP ranks a job of world_size GPUs can run as a complete sub-transfer
    (every present D rank has all the P ranks holding its heads): (n_p, n_d).
    Merge (tp_p >= tp_d): each D rank needs tp_p/tp_d P ranks; split: each P rank feeds
    tp_d/tp_p D ranks.  With world_size >= tp_p + tp_d this is the full transfer."""
    if tp_p >= tp_d:
        ratio = tp_p // tp_d
        n_d = min(tp_d, world_size // (1 + ratio))
        return n_d * ratio, n_d
    ratio = tp_d // tp_p
    n_p = min(tp_p, world_size // (1 + ratio))
    return n_p, n_p * ratio


@dataclass
class StreamRole:
    kind: str        # "P" or "D"
    inst: int        # P instance (P ranks); -1 for D ranks
    tp_rank: int


class StreamPlan:
    """Roles and wiring of the c5 stream (several P instances feeding one D instance; the
    paper's DP-replicated prefill): world ranks [0, n_p) are P ranks -- instance
    rank // per_inst, TP rank rank % per_inst -- and [n_p, n_p + n_d) the D instance's TP
    ranks.  Requests alternate over the instances (request r belongs to instance r % n_inst).
    Completion words: every rank owns an int32 flag array of ``flag_words`` words; the word a
    peer signals in it is the peer's world rank (``flag_word``)."""

    def __init__(self, world: int, tp_p: int, tp_d: int, num_kv_heads: int, n_req: int):
        self.world, self.tp_p, self.tp_d, self.H, self.n_req = world, tp_p, tp_d, num_kv_heads, n_req
        self.n_p = self.n_d = world // 2
        self.n_inst = 2 if self.n_p >= 2 else 1
        self.per_inst = self.n_p // self.n_inst
        self.flag_words = max(world, 1)
        if self.n_p < 1 or self.per_inst < 1:
            raise ValueError(f"the stream needs at least 2 GPUs, got {world}")

    def role(self, rank: int) -> StreamRole:
        if rank < self.n_p:
            return StreamRole("P", rank // self.per_inst, rank % self.per_inst)
        return StreamRole("D", -1, rank - self.n_p)

    def requests_of(self, inst: int):
        return list(range(inst, self.n_req, self.n_inst))

    def inst_of(self, r: int) -> int:
        return r % self.n_inst

    def p_index(self, inst: int, tp_rank: int) -> int:
        """Control-plane key of a P rank (unique over the instances) = its world rank."""
        return inst * self.per_inst + tp_rank

    def d_world(self, q: int) -> int:
        return self.n_p + q

    def d_peers(self, p_world: int):
        """D TP ranks (present) the P rank at world rank p_world feeds (A2 pairs of its TP rank)."""
        tp = self.role(p_world).tp_rank
        return sorted({q for p, q, _hb, _he in kv.plan_pairs(self.tp_p, self.tp_d, self.H) if p == tp and q < self.n_d})

    def p_sources(self, d_world: int):
        """World ranks of the P ranks (every instance) that feed the D rank at world rank d_world."""
        q = self.role(d_world).tp_rank
        return [pr for pr in range(self.n_p) if q in self.d_peers(pr)]

    def flag_word(self, world_rank: int) -> int:
        return world_rank


def pair_plan(tp_p: int, tp_d: int, num_kv_heads: int, p_ranks=None, d_ranks=None):
    """A2 pairs restricted to the ranks present: [(p, q, h_begin, h_end)]."""
    pairs = kv.plan_pairs(tp_p, tp_d, num_kv_heads)
    return [x for x in pairs if (p_ranks is None or x[0] in p_ranks) and (d_ranks is None or x[1] in d_ranks)]


def exchange(obj, group=None):
    """all_gather_object over the control-plane group (gloo or nccl)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


class ControlPlane:
    """A3: the control-plane exchange before a transfer ("control plane information
    interaction"; P:125 D obtains P's "GPU ranks and parallel strategy").

    Collective over the job (or ``group``).  Every P / D rank publishes one kv_ctrl message
    (``kv.ctrl_encode``): its layout descriptor, its fp8 scales when its pool is fp8 (a D
    rank's scales are what P's sender-side cast quantises with) and, if it passes them, the
    batch's block tables its instance chose.  Afterwards every rank holds every other rank's
    parsed message: ``layout(kind, r, device)`` rebuilds a peer's layout (scales uploaded to
    this rank's GPU) and ``batch(kind, device)`` the peer instance's validated tables.  The
    bytes travel through torch.distributed (object all-gather); nothing is regenerated from
    seeds on the receiving side."""

    def __init__(self, role: Role, layout=None, scales=None, n_tokens=None, tables=None, batch_id=0, group=None):
        mine = None
        if role.kind in ("P", "D") and layout is not None:
            mine = {"kind": role.kind, "r": role.tp_rank,
                    "msg": kv.ctrl_encode(layout, scales, n_tokens, tables, batch_id)}
        allv = exchange(mine, group)
        self.role = role
        self.msgs = {(e["kind"], e["r"]): kv.ctrl_decode(e["msg"]) for e in allv if e is not None}
        self.bytes_received = sum(len(e["msg"]) for e in allv if e is not None)

    def ranks(self, kind):
        return sorted(r for k, r in self.msgs if k == kind)

    def message(self, kind, r):
        return self.msgs[(kind, r)]

    def layout(self, kind, r, device="cuda"):
        """kv_layout_describe of rank r of instance `kind` (its scales on `device`)."""
        return self.msgs[(kind, r)].layout(device)

    def tables(self, kind):
        """(n_tokens, tables) the instance published; every rank of it must agree (one block
        table per instance, shared by its TP ranks)."""
        got = [(m.n_tokens, m.tables) for (k, _), m in sorted(self.msgs.items()) if k == kind and m.tables is not None]
        if not got:
            raise ValueError(f"no {kind} rank published block tables")
        nt0, tb0 = got[0]
        for nt, tb in got[1:]:
            if nt != nt0 or len(tb) != len(tb0) or any(list(a) != list(b) for a, b in zip(tb, tb0)):
                raise ValueError(f"{kind} ranks published different block tables")
        return nt0, tb0

    def batch(self, kind, layout, device="cuda", stream=None):
        """kv_block_table_update of instance `kind`'s published tables against `layout` (a
        layout of that instance: block size and pool capacity are validated)."""
        nt, tb = self.tables(kind)
        return kv.Batch(layout, nt, tb, device, stream)


class PushChannel:
    """IPC-mapped D pools + flags for the fused push (K4/K5).

    Every rank calls the constructor collectively.  D ranks pass their pool tensor and a
    4-byte flag tensor; P ranks pass None.  Afterwards P ranks hold ``peer_pool[q]`` and
    ``peer_flag[q]`` (device addresses in the P process) for every D rank q."""

    def __init__(self, role: Role, pool=None, flag=None, group=None, ipc_export=None, ipc_open=None):
        ipc_export = ipc_export or kv.ipc_export
        ipc_open = ipc_open or kv.ipc_open
        mine = None
        if role.kind == "D":
            mine = {"q": role.tp_rank, "pool": ipc_export(pool), "flag": ipc_export(flag)}
        allv = exchange(mine, group)
        self.role = role
        self.peer_pool, self.peer_flag, self._mapped = {}, {}, []
        if role.kind == "P":
            for ent in allv:
                if ent is None:
                    continue
                q = ent["q"]
                self.peer_pool[q] = ipc_open(*ent["pool"])
                self.peer_flag[q] = ipc_open(*ent["flag"])
                self._mapped += [(self.peer_pool[q], ent["pool"][1]), (self.peer_flag[q], ent["flag"][1])]

    def close(self):
        for ptr, off in self._mapped:
            kv.ipc_close(ptr, off)
        self._mapped = []


class PullChannel:
    """IPC maps for the D-initiated read (kv_pull / kv_stage + kv_pull_staged).

    Collective.  Every rank passes its role and a local int32 flag array: on a D rank one
    ready word per P rank (P writes it), on a P rank one done / free word per D rank (D
    writes it).  P ranks also pass ``pool`` (direct pull) or ``ring`` (a uint8 tensor of
    len(ring_dst) * ring_slots * slot_bytes bytes; slot b for D rank ring_dst[i] starts at
    (i * ring_slots + b) * slot_bytes).  Afterwards a D rank holds, per P rank p,
    ``src_pool[p]`` / ``src_ring[p]`` (its ring_slots slot addresses) and ``peer_flag[p]``
    (the word it signals in p's flag array); a P rank holds ``peer_flag[q]`` per D rank q and,
    when D ranks pass ``scales`` (their fp8 scale arrays, for dynamic scales shipped by P),
    ``peer_scales[q]``."""

    def __init__(self, role: Role, flags, pool=None, ring=None, ring_dst=(), ring_slots=0, slot_bytes=0,
                 group=None, ipc_export=None, ipc_open=None, scales=None):
        ipc_export = ipc_export or kv.ipc_export
        ipc_open = ipc_open or kv.ipc_open
        mine = {"kind": role.kind, "r": role.tp_rank, "flags": ipc_export(flags) if role.kind in "PD" else None,
                "pool": ipc_export(pool) if pool is not None else None,
                "ring": ipc_export(ring) if ring is not None else None, "ring_dst": list(ring_dst),
                "ring_slots": ring_slots, "slot_bytes": slot_bytes,
                "scales": ipc_export(scales) if scales is not None else None}
        allv = exchange(mine, group)
        self.role = role
        self.src_pool, self.src_ring, self.peer_flag, self._mapped = {}, {}, {}, []
        self.slot_bytes = {}   # D side: P rank p's ring slot size
        self.peer_scales = {}  # P side: D rank q's scale array
        if role.kind not in "PD":
            return
        other = "P" if role.kind == "D" else "D"
        for ent in allv:
            if ent["kind"] != other:
                continue
            if role.kind == "P":
                # my word in D rank q's ready array is index p
                base = ipc_open(*ent["flags"])
                self._mapped.append((base, ent["flags"][1]))
                self.peer_flag[ent["r"]] = base + 4 * role.tp_rank
                if ent["scales"] is not None:
                    self.peer_scales[ent["r"]] = ipc_open(*ent["scales"])
                    self._mapped.append((self.peer_scales[ent["r"]], ent["scales"][1]))
                continue
            p, q = ent["r"], role.tp_rank
            if ent["pool"] is None and (ent["ring"] is None or q not in ent["ring_dst"]):
                continue
            base = ipc_open(*ent["flags"])
            self._mapped.append((base, ent["flags"][1]))
            self.peer_flag[p] = base + 4 * q
            if ent["pool"] is not None:
                self.src_pool[p] = ipc_open(*ent["pool"])
                self._mapped.append((self.src_pool[p], ent["pool"][1]))
            if ent["ring"] is not None:
                rb = ipc_open(*ent["ring"])
                self._mapped.append((rb, ent["ring"][1]))
                i, R, sb = ent["ring_dst"].index(q), ent["ring_slots"], ent["slot_bytes"]
                self.src_ring[p] = [rb + (i * R + b) * sb for b in range(R)]
                self.slot_bytes[p] = sb

    def close(self):
        for ptr, off in self._mapped:
            kv.ipc_close(ptr, off)
        self._mapped = []


def push_step(src_layout, src_pool, src_batch, dst_layouts, peer_pools, dst_batch, peer_flags, epoch,
              layer_chunk=None, stream=None, flag_slot=0):
    """P side of one push transfer (native kv_push): one fused gather/convert/NVLink-store
    launch per layer chunk covering every paired D rank (A10), then a release flag per D
    rank (A11).  With fan-in (several P ranks feeding one D rank) each P rank writes its own
    flag word ``flag_slot`` of the D rank's flag array."""
    qs = sorted(dst_layouts)
    kv.push(src_layout, src_pool, src_batch, [dst_layouts[q] for q in qs], [peer_pools[q] for q in qs], dst_batch,
            [peer_flags[q] + 4 * flag_slot for q in qs], epoch, None, layer_chunk or 0, stream)


def nccl_send_step(comm, src_layout, src_pool, src_batch, dst_layouts, dst_world, wires, layer_chunk, pack_stream,
                   send_stream, events=None, stream=None):
    """P side of the NCCL mode (native kv_send_pipelined): pack layer chunk k+1 on
    pack_stream while chunk k is on the wire; wires[(q, b)] double buffers per peer."""
    qs = sorted(dst_layouts)
    cap = min(wires[(q, b)].numel() for q in qs for b in range(2))
    comm.send_pipelined(src_layout, src_pool, src_batch, [dst_layouts[q] for q in qs], [dst_world[q] for q in qs],
                        [wires[(q, b)] for q in qs for b in range(2)], cap, layer_chunk, None, stream, pack_stream,
                        send_stream)


def nccl_recv_step(comm, src_layouts, dst_layout, dst_pool, dst_batch, src_world, wires, layer_chunk, recv_stream,
                   unpack_stream, events=None, stream=None):
    """D side of the NCCL mode (native kv_recv_pipelined): receive layer chunk k+1 from
    every paired P rank (grouped, so fan-in links run concurrently) while chunk k is
    unpacked."""
    ps = sorted(src_layouts)
    cap = min(wires[(p, b)].numel() for p in ps for b in range(2))
    comm.recv_pipelined([src_layouts[p] for p in ps], [src_world[p] for p in ps], dst_layout, dst_pool, dst_batch,
                        [wires[(p, b)] for p in ps for b in range(2)], cap, layer_chunk, None, stream, recv_stream,
                        unpack_stream)


class HostStaged:
    """The paper's own transport (P:95 steps 3/5/6), kept as the baseline the NVLink
    path replaces (NEXT-3): P packs each layer chunk (Fig. 5 flatten + the sender-side cast)
    and copies it into a pinned host "CPU buffer"; the transfer engine moves it to D's CPU
    buffer (here both instances share one host, so the buffer is shared: the stand-in RDMA
    read costs nothing, which makes this the fastest host-staged path the box allows); D
    copies it up and unpacks it into its pool.  Every chunk is a chain of device work with
    event edges only (no host round trip): P's stream packs and copies down, D's stream waits
    for that copy, copies up and unpacks; a host slot is reused after the copy up that read it.
    P and D may be the same GPU or two GPUs of one process."""

    def __init__(self, src_layout, dst_layout_at_p, dst_layout, total_tokens, layer_range, layer_chunk, p_device,
                 d_device, slots=3):
        import torch
        lb, le = layer_range
        self.chunks = [(l0, min(le, l0 + layer_chunk)) for l0 in range(lb, le, layer_chunk)]
        self.nbytes = [kv.wire_bytes(src_layout, dst_layout, total_tokens, c) for c in self.chunks]
        cap = max(self.nbytes + [16])
        self.R = max(1, min(slots, len(self.chunks)))
        self.wp = [torch.empty(cap, dtype=torch.uint8, device=p_device) for _ in range(self.R)]
        self.wd = [torch.empty(cap, dtype=torch.uint8, device=d_device) for _ in range(self.R)]
        self.host = [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(self.R)]
        self.sp = torch.cuda.Stream(device=p_device)
        self.sd = torch.cuda.Stream(device=d_device)
        self.p_device, self.d_device = p_device, d_device
        self.S, self.Dp, self.D = src_layout, dst_layout_at_p, dst_layout

    def step(self, src_pool, src_batch, dst_pool, dst_batch, stream_p=None, stream_d=None):
        """Enqueue one transfer; stream_p / stream_d (optional) wait for all of it."""
        import torch
        sp, sd = self.sp, self.sd
        if stream_p is not None:
            sp.wait_stream(stream_p)
        if stream_d is not None:
            sd.wait_stream(stream_d)
        up_done = [None] * self.R
        for k, (lr, n) in enumerate(zip(self.chunks, self.nbytes)):
            b = k % self.R
            with torch.cuda.device(self.p_device), torch.cuda.stream(sp):
                if up_done[b] is not None:
                    sp.wait_event(up_done[b])       # D copied this host slot up already
                kv.pack(self.S, src_pool, src_batch, self.Dp, self.wp[b], lr, sp, wire_nbytes=n)
                self.host[b][:n].copy_(self.wp[b][:n], non_blocking=True)   # P -> CPU buffer
                down = torch.cuda.Event()
                down.record(sp)
            with torch.cuda.device(self.d_device), torch.cuda.stream(sd):
                sd.wait_event(down)
                self.wd[b][:n].copy_(self.host[b][:n], non_blocking=True)  # CPU buffer -> D
                up_done[b] = torch.cuda.Event()
                up_done[b].record(sd)
                kv.unpack(self.S, self.D, dst_pool, dst_batch, self.wd[b], lr, sd, wire_nbytes=n)
        if stream_p is not None:
            stream_p.wait_stream(sp)
        if stream_d is not None:
            stream_d.wait_stream(sd)
