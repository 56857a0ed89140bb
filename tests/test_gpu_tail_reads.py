"""SPEC S:274 ("never read beyond T_r") in the memory-access sense, reading 5: the source
tail slots of a request's last block are not read by any kernel whose source has head_dim
innermost (the TMA tile paths load a partial sub-tile's valid rows by plain loads).  Each
case runs in a child process (tests/guard_child.py) whose P pool ends its valid data at the
end of a virtual-memory mapping, with the tail slots unmapped: a read of them would fault.

Sources whose slots are interleaved with head_dim inside 32-B sectors (head_dim-major V,
x-packed K: k_convert_tr8 / k_convert_tb) read whole sectors by construction; they are not
covered here (reading 5)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["copy", "cast", "rows", "pack", "copy_slotmajor", "cast_slotmajor"])
def test_no_source_tail_reads(mode):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, "-m", "tests.guard_child", mode], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "OK" in out.stdout, (out.stdout[-2000:], out.stderr[-3000:])
