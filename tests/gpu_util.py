"""Move a tests.kvcase case onto the GPU and run the CUDA path through the C ABI."""
from __future__ import annotations

import numpy as np
import torch

from tests.kvcase import NPTYPE
from synth import NBYTES


def np_to_dev(a: np.ndarray, device="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(device)


def dev_to_np(t: torch.Tensor, dtype_code):
    return t.cpu().numpy().view(NPTYPE[NBYTES[dtype_code]])


class DevCase:
    def __init__(self, case, device="cuda"):
        import paper_2509_17542_b200 as kvx
        self.kvx = kvx
        self.case = case
        self.src_lays = []
        for lay in case["src_lays"]:
            sc = None if lay.get("scales") is None else torch.from_numpy(np.asarray(lay["scales"], np.float32)).to(device)
            self.src_lays.append(kvx.Layout.from_dict(lay, sc))
        self.dst_lays = []
        for lay in case["dst_lays"]:
            sc = None if lay.get("scales") is None else torch.from_numpy(np.asarray(lay["scales"], np.float32)).to(device)
            self.dst_lays.append(kvx.Layout.from_dict(lay, sc))
        self.src_pools = [np_to_dev(p, device) for p in case["src_pools"]]
        self.dst_pools = [np_to_dev(p, device) for p in case["dst_pools"]]
        self.src_bt = kvx.Batch(self.src_lays[0], case["n_tokens"], case["src_tables"], device)
        self.dst_bt = kvx.Batch(self.dst_lays[0], case["n_tokens"], case["dst_tables"], device)

    def convert(self, layer_range=None, dst_idx=None, src_idx=None):
        di = range(len(self.dst_lays)) if dst_idx is None else dst_idx
        si = range(len(self.src_lays)) if src_idx is None else src_idx
        self.kvx.convert_reshard([self.src_lays[i] for i in si], [self.src_pools[i] for i in si], self.src_bt,
                                 [self.dst_lays[i] for i in di], [self.dst_pools[i] for i in di], self.dst_bt,
                                 layer_range)
        torch.cuda.synchronize()

    def dst_numpy(self):
        return [dev_to_np(t, l["dtype"]) for t, l in zip(self.dst_pools, self.case["dst_lays"])]
