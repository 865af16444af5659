"""rmips-b200: exact reverse k-MIPS (Simpfer, arXiv 2110.07131) hot path for one B200 (sm_100a).

The product is the C ABI in include/rmips.h, implemented by librmips.so (csrc/*.cu).
`paper_2110_07131_b200.rmips` is a thin ctypes binding with the same names.  Importing it
requires the compiled library: there is no CPU fallback.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librmips.so")


def load():
    """Import the binding (raises ImportError if librmips.so is missing)."""
    from . import rmips
    return rmips
