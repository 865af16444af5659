"""Development probe: host time of every API call over repeated bench-like steps (build + query calls),
printing outliers, to locate sporadic stalls.  Usage: python tools/stall_probe.py [config] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = make_workload(cfg)
spec = w.spec
U, P, Q = (torch.from_numpy(a).cuda() for a in (w.U, w.P, w.Qy))
Qb = [Q[a:a + spec.batch] for a in range(0, spec.nq, spec.batch)]
k = spec.ks[-1]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for s in range(steps):
    flush.zero_()
    torch.cuda.synchronize()
    rec = []
    t0 = time.perf_counter()
    idx = rmips.rmips_build_index(U, P, spec.k_max, rmips.RMIPS_BUILD_TIMING)
    rec.append(("build", time.perf_counter() - t0))
    for j, q in enumerate(Qb):
        t1 = time.perf_counter()
        off, ids = rmips.rmips_query(idx, q, k, rmips.RMIPS_FLAG_TIMING)
        rec.append(("q%d" % j, time.perf_counter() - t1))
        t2 = time.perf_counter()
        idx.phase_times(), idx.stats()
        rec.append(("rd%d" % j, time.perf_counter() - t2))
    t3 = time.perf_counter()
    idx.close()
    rec.append(("close", time.perf_counter() - t3))
    tot = time.perf_counter() - t0
    med = np.median([r[1] for r in rec if r[0].startswith("q")])
    out = [(n, round(v * 1e3, 3)) for n, v in rec if (n.startswith("q") and v > 3 * med) or (not n.startswith("q") and v > 2e-3)]
    print("step %d: %.2f ms total; query median %.3f ms; outliers %s" % (s, tot * 1e3, med * 1e3, out), flush=True)
