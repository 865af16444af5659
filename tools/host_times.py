import collections, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2110_07131_b200 import rmips
from synth.generator import make_workload
w = make_workload(1)
dev = torch.device("cuda", 0)
U = torch.from_numpy(w.U).to(dev); P = torch.from_numpy(w.P).to(dev); Qy = torch.from_numpy(w.Qy).to(dev)
k = w.spec.ks[0]
T = collections.defaultdict(list)
def step():
    t0 = time.perf_counter(); idx = rmips.rmips_build_index(U, P, w.spec.k_max); t1 = time.perf_counter()
    rmips.rmips_query(idx, Qy, k); t2 = time.perf_counter(); idx.close(); t3 = time.perf_counter()
    T["build"].append(t1 - t0); T["query"].append(t2 - t1); T["close"].append(t3 - t2)
for _ in range(5): step()
T.clear()
for _ in range(10): step()
for kk, v in T.items(): print("host %s %.1f us" % (kk, 1e6 * sorted(v)[len(v) // 2]))
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
tot = collections.defaultdict(float); cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cu"):
        tot[e.name] += e.cpu_time_total; cnt[e.name] += 1
for n, t in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print("%8.1f us/step  x%-3d %s" % (t / 3, cnt[n] // 3, n))

# one step's host runtime-API timeline (start offset, duration) to locate host-side stalls
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cu")],
            key=lambda e: e.time_range.start)
syncs = [i for i, e in enumerate(ev) if e.name == "cudaStreamSynchronize"]
if len(syncs) >= 4:
    lo, hi = syncs[2], syncs[5] if len(syncs) > 5 else len(ev) - 1
    t0 = ev[lo].time_range.start
    prev_end = t0
    for e in ev[lo:hi + 1]:
        print("%9.1f %+8.1f %7.1f  %s" % (e.time_range.start - t0, e.time_range.start - prev_end,
                                          e.time_range.end - e.time_range.start, e.name))
        prev_end = e.time_range.end
