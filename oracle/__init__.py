"""TEST INFRASTRUCTURE ONLY — CPU oracle for the SlimSell BFS-SpMV path.

Two checkers live here, both loaded through ctypes:

* ``port``      — ``liboracle.so``, the plain-C restatement in
  ``slimsell_oracle.c`` (each function cites the reference file:line).
* ``reference`` — ``_ref/libslimsell_ref.so``, the unmodified reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``
  plus the C-ABI shim ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference arm may import this package, and only as the checker or the timed
CPU baseline — never as the product path.
"""
from .cpu import (  # noqa: F401
    KINF,
    TROPICAL,
    REAL,
    BOOLEAN,
    SELMAX,
    VARIANTS,
    OracleError,
    port_available,
    reference_available,
    Port,
    Reference,
    build,
)
