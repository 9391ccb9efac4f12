"""CPU ORACLE -- test infrastructure, not the product.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this package.  It wraps
``oracle/bp_oracle.c`` (a plain-C restatement of the reference binpaths
algorithms, see that file's header for the file:line citations) through
ctypes.  It is pinned against golden vectors made by importing the unmodified
reference (tools/make_goldens.py -> tests/golden/).
"""
from .oracle import (  # noqa: F401
    KIND_BITS,
    build,
    exact,
    exact_range,
    lib,
    mc_bits,
    mc_range,
    mc_shared,
    mc_strata,
    philox4x32_10,
)
