"""ORACLE — test infrastructure only.

Two CPU checkers for the GPU engine, neither ever on the product path:

* ``oracle/_ref/libmigsched_ref.so`` — the unmodified reference library
  (/root/reference/proj/src) compiled by oracle/Makefile with its own Release
  flags (no FMA), behind a C-ABI shim (ref_shim.cpp).
* ``oracle/_port/liboracle_port.so`` — oracle_port.c, a plain-C restatement
  of the reference algorithm, each function citing the reference file:line
  it follows; pinned against the reference library and the golden vectors in
  tests/golden/.

Only tests/, ``__graft_entry__.smoke()`` (as the checker) and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this package.
"""
