"""Development check: overflow rows and candidates per user of the k_max = 128 test shapes
(tests/test_gpu_parity.py::test_kmax_128_lists_without_fallback).  Usage: python tools/ovf_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import generator as gen  # noqa: E402

for d in (50, 100):
    for kind, n, m, km in (("skewed", 3000, 2500, 128), ("skewed", 20000, 50000, 128), ("gaussian", 20000, 50000, 100)):
        U, P = gen.random_instance(90 + d, n, m, d, kind)
        idx = rmips.rmips_build_index(torch.from_numpy(U).cuda(), torch.from_numpy(P).cuda(), km)
        idx.refresh_info()
        print("%s n %d m %d d %d k_max %d: overflow rows %d cand/user %.1f kernel %d slots %d"
              % (kind, n, m, d, km, idx.overflow_rows, idx.cand_total / n, idx.build_kernel, idx.cand_slots), flush=True)
        idx.close()
