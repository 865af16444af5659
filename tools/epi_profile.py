"""Development-only: per item-tile profile of the build epilogue (librmips_prof.so, built with
-DRMIPS_EPI_PROFILE).  Prints, per range of item-tile index, the epilogue's average wait cycles,
work cycles, passing warp-chunks and appends per row."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["RMIPS_LIB"] = os.path.join(ROOT, "paper_2110_07131_b200", "librmips_prof.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth import make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = make_workload(cfg)
U = torch.from_numpy(w.U).cuda()
P = torch.from_numpy(w.P).cuda()
buf = (ctypes.c_ulonglong * (4 * 256))()
for rep in range(2):
    rmips.lib.rmips_debug_epi_profile(buf, 1)
    idx = rmips.rmips_build_index(U, P, w.spec.k_max, rmips.RMIPS_BUILD_TIMING)
    pt = idx.phase_times()
    idx.close()
torch.cuda.synchronize()
rmips.lib.rmips_debug_epi_profile(buf, 0)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 256).astype(np.float64)
n, m = w.spec.n, w.spec.m
ut = (n + 127) // 128
nit = (m + 127) // 128
warps = ut * 4  # epilogue warp-tiles per item-tile index
print("cfg%d contraction %.3f ms; per item-tile index (averaged over %d epilogue warps):" % (cfg, pt[1], warps))
edges = [0, 1, 2, 4, 8, 16, 32, 64, 128, 256]
for lo, hi in zip(edges[:-1], edges[1:]):
    hi = min(hi, nit, 256)
    if lo >= hi:
        break
    s = slice(lo, hi)
    k = hi - lo
    print("tiles %3d-%3d: wait %7.0f cyc  work %7.0f cyc" % (
        lo, hi, a[0, s].sum() / warps / k, a[1, s].sum() / warps / k))
print("slow path per warp-sweep: passing chunks %.1f  append cycles %.0f  refresh cycles %.0f  refreshes %.2f" % (
    a[2, 0] / warps, a[2, 1] / warps, a[2, 2] / warps, a[2, 3] / warps))
tot = a[0].sum() + a[1].sum()
print("total wait %.1f%%  work %.1f%%" % (100 * a[0].sum() / tot, 100 * a[1].sum() / tot))
