"""Multi-GPU parity at BASELINE.json's full sizes, in exactly the launch configuration
bench.py times: torchrun of bench.py itself (one process per GPU, layouts / tables / scales
exchanged through the control plane), each D rank checking a sample of its received pool
against the oracle (request 0, layers [0, 2), the P rank's source sample shipped over the
control plane) and K6 checking every element of every D pool -- for the default pull
transport and the push / NCCL baselines."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(n, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"), "--gpus", str(n),
           "--steps", "2", "--warmup", "1", "--no-e2e", *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = out.stdout.splitlines()  # exactly one line, nothing else (native banners go to stderr)
    assert len(lines) == 1 and lines[0].startswith("{"), out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("mode", ["pull", "push", "nccl"])
def test_c4_pair_fullsize(mode):
    """c4 (70B GQA, 32 x 4096 tokens, bf16 -> e4m3) on one 1:1 pair."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    d = _bench(2, "--mode", mode)
    assert d["parity"] and all(p["ok"] for p in d["parity"]), d["parity"]
    assert d["parity"][0]["mismatches"] == 0
    assert d["fullsize"]["ok"] is True, d["fullsize"]


@pytest.mark.parametrize("workload", ["c3", "c2"])
def test_fan_in_fullsize_pull(workload):
    """c3' / c2: two P ranks -> one D rank (fan-in 2), the D rank pulling both peer pools."""
    if torch.cuda.device_count() < 3:
        pytest.skip("needs 3 GPUs")
    d = _bench(min(4, torch.cuda.device_count()), "--workload", workload, "--mode", "pull")
    assert d["parity"] and all(p["ok"] for p in d["parity"]), d["parity"]
    assert d["fullsize"]["ok"] is True, d["fullsize"]


def test_c4_pair_dynamic_scales():
    """The staged pull with per-chunk amax scales computed on P and shipped with the codes."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    d = _bench(2, "--mode", "pull", "--dynamic-scales")
    assert d["parity"] and all(p["ok"] for p in d["parity"]), d["parity"]
    assert d["parity"][0].get("dynamic_scales_ok") is True


def test_c5_stream_pull():
    """c5' (two P instances' requests, alternating, into one D instance) with K6 full-size."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    d = _bench(4, "--workload", "c5", "--mode", "pull")
    assert d["fullsize"]["ok"] is True, d["fullsize"]


@pytest.mark.parametrize("workload", ["c4", "c5"])
def test_world8_oversubscribed(workload):
    """The full 8-rank configurations (c4: P TP4 -> D TP4, four pairs; c5: two P instances x
    TP2 -> D TP4) as 8 processes on the GPUs available (two or more ranks per GPU, same role
    per GPU, gloo control plane): parity and K6 on every D rank (not a performance run)."""
    # c5's P pools are ~45 GB per rank: four of them on one GPU do not fit, two do
    need = 4 if workload == "c5" else 2
    if torch.cuda.device_count() < need:
        pytest.skip(f"needs {need} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"), "--gpus", "8",
           "--oversubscribe", "--steps", "1", "--warmup", "1", "--no-e2e", "--no-nvlink-probe", "--workload", workload]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.splitlines()[0])
    assert d["n_gpus"] == 8 and d["config"]["oversubscribed"]
    assert d["fullsize"]["ok"] is True, d["fullsize"]
    if workload == "c4":
        assert len(d["parity"]) == 4 and all(p["ok"] for p in d["parity"]), d["parity"]
