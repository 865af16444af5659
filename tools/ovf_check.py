"""Development check: build time split and overflow rows (rows sent to the O(m d) exact fallback) across
the shape domain (configs[4] recipe).  Usage: python tools/ovf_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth.generator import make_workload  # noqa: E402

SHAPES = [(148000, 1000000, 256, 50), (148000, 1000000, 240, 50), (60000, 1200000, 300, 50),
          (60000, 1200000, 200, 50), (148000, 1000000, 200, 100), (148000, 1000000, 64, 50),
          (148000, 1000000, 120, 50), (148000, 300000, 1000, 50)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for (n, m, d, km) in SHAPES:
    w = make_workload(4, n=n, m=m, d=d, nq=16)
    U = torch.from_numpy(w.U).cuda()
    P = torch.from_numpy(w.P).cuda()
    for r in range(2):
        idx = rmips.rmips_build_index(U, P, km, rmips.RMIPS_BUILD_TIMING)
        pt = idx.phase_times()
        idx.refresh_info()
        if r:
            print("n %d m %d d %d k_max %d: build %.1f ms (prep %.1f contraction %.1f select %.1f) overflow rows %d "
                  "cand/user %.1f kernel %d slots %d" % (n, m, d, km, pt[3], pt[0], pt[1], pt[2], idx.overflow_rows,
                                                         idx.cand_total / n, idx.build_kernel, idx.cand_slots), flush=True)
        idx.close()
    del U, P
    torch.cuda.empty_cache()
