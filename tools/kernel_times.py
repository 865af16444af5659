"""Warm per-kernel device times of one bench-shaped step (build + query) via the CUDA activity
trace of torch.profiler (CUPTI): unlike the ncu launch list these are not serialised or cold-cache.
Usage: python tools/kernel_times.py [config] [steps]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2110_07131_b200 import rmips  # noqa: E402
from synth.generator import make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = make_workload(cfg)
dev = torch.device("cuda", 0)
U = torch.from_numpy(w.U).to(dev)
P = torch.from_numpy(w.P).to(dev)
Qy = torch.from_numpy(w.Qy).to(dev)
k = w.spec.ks[0]


def step():
    idx = rmips.rmips_build_index(U, P, w.spec.k_max)
    rmips.rmips_query(idx, Qy, k)
    idx.close()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name if len(e.name) < 70 else e.name[:67] + "..."
        tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[name] += 1
allt = sum(tot.values())
print("config %d, %d steps, per-step device time by kernel (us):" % (cfg, steps))
for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("%9.1f  %5.1f%%  x%-3d %s" % (t / steps, 100 * t / allt, cnt[name] // steps, name))
print("%9.1f  total" % (allt / steps))

# idle gaps on the device between consecutive activities (where the GPU waits for the host)
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
gaps = collections.defaultdict(float)
gcount = collections.Counter()
span = (evs[-1].time_range.end - evs[0].time_range.start) if evs else 0
idle = 0.0
for a, b_ in zip(evs, evs[1:]):
    g = b_.time_range.start - a.time_range.end
    if g > 0:
        idle += g
        key = "%s -> %s" % (a.name[:40], b_.name[:40])
        gaps[key] += g
        gcount[key] += 1
print("device span %.1f us/step, idle %.1f us/step; largest idle gaps (us/step):" % (span / steps, idle / steps))
for key, g in sorted(gaps.items(), key=lambda kv: -kv[1])[:20]:
    print("%8.1f  x%-3d %s" % (g / steps, gcount[key] // steps, key))
