"""Out-of-bounds guard for every convert kernel (SURVEY T3 without compute-sanitizer, which
this pool's GPUs do not allow): each P and D pool in its own virtual-memory mapping with
unmapped address space on both sides, so one byte read or written outside any pool faults.
Groups: "tile" and "vendor" (every convert kernel), "wire" (k_pack / k_pack_rows into a wire
buffer that ends at an unmapped page, k_unpack_rows back into guarded D pools, k_amax over
guarded P pools).  Runs tests/guard_pools.py in a child process per group (a fault must not
take the test process's CUDA context with it); each case also matches O1 element by element."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("group", ["tile", "vendor", "wire"])
def test_guarded_pools(group):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, "-m", "tests.guard_pools", group], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, (out.stdout[-2000:], out.stderr[-3000:])
