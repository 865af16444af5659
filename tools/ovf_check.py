import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2110_07131_b200 import rmips
from synth.generator import make_workload
for (n, m, d) in ((148000, 1000000, 300), (148000, 1000000, 200), (148000, 200000, 300), (148000, 1000000, 513)):
    w = make_workload(4, n=n, m=m, d=d, nq=16)
    U = torch.from_numpy(w.U).cuda(); P = torch.from_numpy(w.P).cuda()
    for r in range(2):
        idx = rmips.rmips_build_index(U, P, 50, rmips.RMIPS_BUILD_TIMING)
        pt = idx.phase_times(); idx.refresh_info()
        if r: print("n %d m %d d %d: build %.1f ms (prep %.1f contraction %.1f select %.1f) overflow rows %d cand/user %.1f kernel %d slots %d" % (
            n, m, d, pt[3], pt[0], pt[1], pt[2], idx.overflow_rows, idx.cand_total / n, idx.build_kernel, idx.cand_slots))
        idx.close()
