"""fp64 CPU oracle for exact reverse k-MIPS (arXiv 2110.07131).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg are the only callers.  The product package
(paper_2110_07131_b200) never imports this package, and this package never
imports the product.  See oracle/oracle.c for the arithmetic and its citations.
"""
from .oracle import *  # noqa: F401,F403
