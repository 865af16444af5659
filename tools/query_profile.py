"""Development-only: where the tcgen05 query kernel waits (librmips_prof.so, -DRMIPS_EPI_PROFILE):
MMA warp cycles waiting for Q_FULL / ACC_EMPTY / A_FULL, epilogue warps waiting for ACC_FULL,
producer waiting for A_EMPTY, summed over CTAs."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["RMIPS_LIB"] = os.path.join(ROOT, "paper_2110_07131_b200", "librmips_prof.so")
import numpy as np, torch
from paper_2110_07131_b200 import rmips
from synth import make_workload
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = make_workload(cfg)
U = torch.from_numpy(w.U).cuda(); P = torch.from_numpy(w.P).cuda(); Q = torch.from_numpy(w.Qy).cuda()
idx = rmips.rmips_build_index(U, P, w.spec.k_max)
buf = (ctypes.c_ulonglong * 8)()
for rep in range(3):
    rmips.lib.rmips_debug_query_profile(buf, 1)
    off, ids = rmips.rmips_query(idx, Q, w.spec.ks[0], rmips.RMIPS_FLAG_TIMING)
    torch.cuda.synchronize()
rmips.lib.rmips_debug_query_profile(buf, 0)
a = np.frombuffer(buf, dtype=np.uint64).astype(np.float64)
pt = idx.phase_times()
cyc = pt[9] * 1e-3 * 1.965e9 * 148
print("cfg%d filter %.3f ms (%.3g SM-cycles); per CTA-role share of the kernel time:" % (cfg, pt[9], cyc))
for i, name in enumerate(["MMA wait Q_FULL", "MMA wait ACC_EMPTY", "MMA wait A_FULL", "epilogue wait ACC_FULL (per warp)", "producer wait A_EMPTY"]):
    scale = 8 if i == 3 else 1
    print("  %-36s %5.1f%%" % (name, 100 * a[i] / scale / cyc))
