"""Seeded synthetic workloads.

This package holds ONLY input generation: it contains none of the method's
arithmetic (no inner products, norms-for-ranking, top-k or decisions).  It is
the one module shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (tests, bench, smoke).
"""
from .generator import CONFIGS, Workload, make_workload, table1, sha256_arrays  # noqa: F401
