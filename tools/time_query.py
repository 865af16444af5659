"""Development timing of the query path on a BASELINE config (librmips_dev.so switches read at every
launch): per variant, the median over calls of the filter kernel's own time (k_query_tc, CUDA events
right around it) and of the whole call.
Usage: RMIPS_LIB=.../librmips_dev.so python tools/time_query.py CFG [reps] [VAR=1,VAR2=1 ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import make_workload  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variants = sys.argv[3:] or ["default"]
w = make_workload(cfg)
U = torch.from_numpy(w.U).cuda()
P = torch.from_numpy(w.P).cuda()
Q = torch.from_numpy(w.Qy).cuda()
k = w.spec.ks[-1]
idx = rmips.rmips_build_index(U, P, w.spec.k_max)
# warm-up pass (discarded): the first variant measured in a process otherwise includes the clock ramp
# (configs[4]: 99 vs 83 us per call for the same kernel)
for b0 in range(0, Q.shape[0], w.spec.batch):
    rmips.rmips_query(idx, Q[b0:b0 + w.spec.batch], k, rmips.RMIPS_FLAG_TIMING)
for b0 in range(0, Q.shape[0], w.spec.batch):
    rmips.rmips_query(idx, Q[b0:b0 + w.spec.batch], k, rmips.RMIPS_FLAG_TIMING)
keys = set()
for v in variants:
    keys |= {kv.split("=")[0] for kv in v.split(",") if "=" in kv}
for v in variants:
    for k_ in keys:
        os.environ.pop(k_, None)
    for kv in v.split(","):
        if "=" in kv:
            a, b = kv.split("=")
            os.environ[a] = b
    kern, call = [], []
    dev = getattr(rmips.lib, "rmips_debug_qdev", None) if hasattr(rmips.lib, "rmips_debug_qdev") else None
    qd = (ctypes.c_ulonglong * 4)()
    if dev:
        dev(qd, 1)
    for r in range(reps + 1):
        for b0 in range(0, Q.shape[0], w.spec.batch):
            rmips.rmips_query(idx, Q[b0:b0 + w.spec.batch], k, rmips.RMIPS_FLAG_TIMING)
            pt = idx.phase_times()
            if r:
                kern.append(pt[13])
                call.append(pt[12])
    extra = ""
    if dev:
        dev(qd, 0)
        extra = "  flagged warp-chunks %.2f%% of %d" % (100.0 * qd[0] / max(1, qd[1]), qd[1])
    print("cfg%d %-32s filter kernel %.1f us/call  call %.1f us (median of %d)%s" %
          (cfg, v, 1e3 * float(np.median(kern)), 1e3 * float(np.median(call)), len(kern), extra), flush=True)
idx.close()
