"""Development timing of one build shape (synthetic cfg4 recipe, custom n / m / d): median contraction
and build times over a few builds, for several dev-switch variants in ONE process (the RMIPS_DEV switches
of librmips_dev.so are read at every launch).
Usage: RMIPS_LIB=.../librmips_dev.so python tools/time_build.py n m d [k_max] [reps] [VAR=1,VAR2=1 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth.generator import make_workload  # noqa: E402

n, m, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kmax = int(sys.argv[4]) if len(sys.argv) > 4 else 50
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
variants = sys.argv[6:] or ["default"]
w = make_workload(4, n=n, m=m, d=d, nq=16)
U = torch.from_numpy(w.U).cuda()
P = torch.from_numpy(w.P).cuda()
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
    ts = []
    for r in range(reps + 1):
        idx = rmips.rmips_build_index(U, P, kmax, rmips.RMIPS_BUILD_TIMING)
        pt = idx.phase_times()
        if r:
            ts.append((pt[1], pt[3], idx.tiles_done))
        idx.close()
    c = float(np.median([t[0] for t in ts]))
    tiles = ts[-1][2]
    kst = 16 * ((d + 15) // 16)
    print("%-40s n %d m %d d %d: contraction %.3f ms build %.3f ms tiles %d -> %.1f TFLOP/s (MMA K=%d), %.0f ns/tile/SM"
          % (v, n, m, d, c, float(np.median([t[1] for t in ts])), tiles,
             2.0 * tiles * 128 * 128 * kst / (c / 1e3) / 1e12, kst, c * 1e6 * 148 / max(1, tiles)), flush=True)
