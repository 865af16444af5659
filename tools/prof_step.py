"""Run N full steps (build + query) of a config; used under ncu for kernel captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--simt", action="store_true")
ap.add_argument("--qflags", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--pprime", type=int, default=0, help="P' index over the first C * k_max items")
a = ap.parse_args()
w = make_workload(a.config, n=a.n or None)
U = torch.from_numpy(w.U).cuda()
P = torch.from_numpy(w.P).cuda()
Q = torch.from_numpy(w.Qy).cuda()
for _ in range(a.steps):
    bf = rmips.RMIPS_BUILD_SIMT if a.simt else 0
    if a.pprime:
        idx = rmips.rmips_build_index_pprime(U, P, w.spec.k_max, a.pprime * w.spec.k_max, bf)
    else:
        idx = rmips.rmips_build_index(U, P, w.spec.k_max, bf)
    for b0 in range(0, Q.shape[0], w.spec.batch):  # the bench's query calls (configs[4]: 40 of 256)
        off, ids = rmips.rmips_query(idx, Q[b0:b0 + w.spec.batch], w.spec.ks[-1], a.qflags)
    idx.close()
torch.cuda.synchronize()
print("ok", int(ids.numel()))
