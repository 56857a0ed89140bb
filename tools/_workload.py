"""Single-process workload holder for the measurement tools (tools/*.py): every P and D rank
of one configuration that lives in this process, both instances' tables (the tools run P
and D in one process, so no control plane is involved), and a sampled oracle check.  Built
from bench.py's input helpers (synth: seeded, no method arithmetic)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import (d_tables, dst_bytes, make_d_rank, make_p_rank, o1_compare, p_tables, sample_of,  # noqa: E402
                   src_bytes)


class Workload:
    def __init__(self, cfg, p_ranks, d_ranks, device, contiguous=False):
        import torch
        import paper_2509_17542_b200 as kvx
        self.cfg, self.device = cfg, device
        c = cfg
        self.NB_p = synth.pool_capacity(c.n_tokens, c.B_p)
        self.NB_d = synth.pool_capacity(c.n_tokens, c.B_d)
        self.src_tables = p_tables(c, self.NB_p, contiguous)
        self.dst_tables = d_tables(c, self.NB_d, contiguous)
        self.p_ranks, self.d_ranks = list(p_ranks), list(d_ranks)
        self.src_dicts, self.src_lays, self.src_pools = {}, {}, {}
        for p in self.p_ranks:
            self.src_dicts[p], self.src_lays[p], self.src_pools[p] = make_p_rank(c, p, self.NB_p, device)
        self.dst_dicts, self.dst_lays, self.dst_pools, self.scales = {}, {}, {}, {}
        for q in self.d_ranks:
            self.dst_dicts[q], self.dst_lays[q], self.dst_pools[q], self.scales[q] = make_d_rank(c, q, self.NB_d, device)
        any_src = self.src_lays[self.p_ranks[0]] if self.p_ranks else kvx.Layout.from_dict(
            synth.layout(c.L, c.H, c.D, c.tp_p, 0, c.B_p, self.NB_p, c.src_dtype, c.p_order))
        any_dst = self.dst_lays[self.d_ranks[0]] if self.d_ranks else make_d_rank(c, 0, self.NB_d, device)[1]
        self._keep = (any_src, any_dst)
        self.src_bt = kvx.Batch(any_src, c.n_tokens, self.src_tables, device)
        self.dst_bt = kvx.Batch(any_dst, c.n_tokens, self.dst_tables, device)
        del torch

    def src_bytes(self, p_ranks=None):
        return src_bytes(self.cfg, None if p_ranks is None else len(p_ranks))

    def dst_bytes(self, d_ranks=None):
        return dst_bytes(self.cfg, None if d_ranks is None else len(d_ranks))


def sample_parity(w, layers, req, p_ranks, d_ranks, dst_pool_of=None):
    """O1 on request `req`, layers [lb, le) of the given ranks vs the device pools -> (ok, detail)."""
    dst_pool_of = dst_pool_of or (lambda q: w.dst_pools[q])
    ss = [sample_of(w.src_pools[p], w.src_dicts[p], w.src_tables, [req], layers) for p in p_ranks]
    ds = [sample_of(dst_pool_of(q), w.dst_dicts[q], w.dst_tables, [req], layers) for q in d_ranks]
    res = o1_compare(ss, ds, [w.cfg.n_tokens[req]], w.cfg.dst_dtype)
    res["sample"] = f"request {req}, layers [{layers[0]},{layers[1]}), P ranks {list(p_ranks)} -> D ranks {list(d_ranks)}"
    return res["ok"], res
