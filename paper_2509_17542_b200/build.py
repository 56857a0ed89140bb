"""Build libkvx.so in-tree with nvcc for sm_100a (no torch JIT cache, so the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkvx.so")
INCLUDE = os.path.join(ROOT, "include")


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers from the torch wheel (nvidia/nccl) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "kvx.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    # several processes (torchrun ranks, pytest workers) may ask at once: one builds, the
    # others wait on the lock and then find the library up to date
    import fcntl
    with open(os.path.join(CSRC, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not needs_build():
            return LIB
        return _build_locked(verbose)


def _build_locked(verbose: bool) -> str:
    """One nvcc -c per translation unit, in parallel, then one shared-library link."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    nccl_inc, nccl_lib = _nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    common = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-O3,-Wall", "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC, "-I", nccl_inc]
    common += os.environ.get("KVX_NVCC_FLAGS", "").split()
    if verbose:
        common.insert(1, "-Xptxas=-v")
    with tempfile.TemporaryDirectory(prefix="kvx_build_") as tmp:
        objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in sources()]

        def cc(pair):
            src, obj = pair
            cmd = common + ["-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            return subprocess.run(cmd, capture_output=not verbose, text=True)

        with ThreadPoolExecutor(len(objs)) as ex:
            res = list(ex.map(cc, zip(sources(), objs)))
        for src, r in zip(sources(), res):
            if r.returncode != 0:
                sys.stderr.write((r.stdout or "") + (r.stderr or ""))
                raise subprocess.CalledProcessError(r.returncode, f"nvcc -c {src}")
        link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_lib, "-o", LIB + ".tmp"]
        subprocess.check_call(link[:4] + objs + link[4:])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
