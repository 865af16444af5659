"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the
d <= 64 build (k_build_tc), the CTA-pair build (k_build_tc2cta, d = 100), the 1-CTA tcgen05 build with
256-slot lists (k_max = 96), the d > 256 streamed kernels, a P' index (scan path), and every query
output path; each checked against the oracle.  Usage: compute-sanitizer --tool X python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import generator as gen  # noqa: E402

dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)  # noqa: E731
bad = 0
for (n, m, d, kmax, k, pp) in [(300, 200, 50, 10, 5, 0), (300, 200, 100, 10, 5, 0), (260, 150, 40, 96, 90, 0),
                               (150, 120, 300, 8, 4, 0), (300, 200, 50, 10, 5, 20)]:
    U, P = gen.random_instance(n + d, n, m, d, "skewed")
    Qy = np.concatenate([P[:7], gen.random_instance(7, 5, 1, d, "skewed")[0]])
    idx = rmips.rmips_build_index_pprime(t(U), t(P), kmax, pp) if pp else rmips.rmips_build_index(t(U), t(P), kmax)
    want = oracle.sets_from_member(oracle.rkmips_naive(U, P, Qy, k))
    for fl in (0, rmips.RMIPS_FLAG_KEY_SORT, rmips.RMIPS_FLAG_VERIFY_SCAN | rmips.RMIPS_FLAG_FORCE_VERIFY):
        got = rmips.split_sets(*rmips.rmips_query(idx, t(Qy), k, fl))
        bad += sum(not np.array_equal(a, b) for a, b in zip(got, want))
    idx.close()
torch.cuda.synchronize()
print("sanitize cases done, %d mismatching sets" % bad)
sys.exit(1 if bad else 0)
