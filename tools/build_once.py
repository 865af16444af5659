"""One timed build of a configs[N] shape after a warm-up build (for ncu launch lists of the build kernels).
Usage: [RMIPS_LIB=...] python tools/build_once.py N [k_max]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth.generator import make_workload  # noqa: E402

w = make_workload(int(sys.argv[1]))
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else w.spec.k_max
U, P = torch.from_numpy(w.U).cuda(), torch.from_numpy(w.P).cuda()
for _ in range(2):
    idx = rmips.rmips_build_index(U, P, kmax, rmips.RMIPS_BUILD_TIMING)
    print("contraction %.3f ms, tiles %d" % (idx.phase_times()[1], idx.tiles_done), flush=True)
    idx.close()
