"""CPU oracle for the heterogeneous-compatible KV transmission path (arXiv 2509.17542).

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything here.
The product package (``paper_2509_17542_b200``) never touches it, and it shares
no code with the CUDA path.

* ``o1``          -- ctypes wrapper around ``kv_oracle.c`` (O1, plain C loops
                     written from SURVEY.md 8(c); see that file's header for the
                     passages it follows).
* ``bruteforce``  -- O2, pure Python, source-driven enumeration and nearest-code
                     casts; tiny shapes only.

Parity status: every function is pinned (tests/test_oracle_*.py); see DESIGN.md
section "Oracle and pins".  The NaN output encodings (reading 12) are pinned by
device observation only.
"""
