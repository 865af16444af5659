"""Summarise a round's GPU evidence into profiles/ (tracked):
  profiles/<round>_launches_cfg<c>.md   per-kernel device time and share (ncu launch list)
  profiles/<round>_ncu_cfg<c>.md        key ncu --set full metrics per hot kernel
  profiles/traffic.json                 dram bytes per launch of each hot kernel (bench.py roofline.traffic)
Usage: python tools/summarize_profiles.py r01 [cfg]"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
g = os.path.join(ROOT, "gpurun_out")


def short(name):
    name = name.replace("rmips::", "")
    if "cub::" in name:
        return "cub::" + name.split("cub::")[1].split("<")[0] + (" (64-bit keys)" if "double" in name or "unsigned long" in name else "")
    return name.split("(")[0]


# ---------------------------------------------------------------- launch list
rows = list(csv.reader(open(os.path.join(g, "launches_cfg%d.csv" % cfg))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
    v *= scale
    agg[short(r[ki])][0] += 1
    agg[short(r[ki])][1] += v
    total += v
    seq.append((short(r[ki]), v))
lines = ["# %s — ncu launch list, cfg%d, `tools/prof_step.py --config %d --steps 2`" % (rnd, cfg, cfg), "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare SHARES, "
         "not absolutes).  Two full steps (build + 1,000-query batch); %d launches, %.1f us total." % (len(seq), total),
         "", "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append("| `%s` | %d | %.1f | %.1f%% |" % (k, c, v, 100 * v / total))
open(os.path.join(out_dir, "%s_launches_cfg%d.md" % (rnd, cfg)), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

# ---------------------------------------------------------------- ncu --set full
rep = os.path.join(g, "prof_cfg%d.ncu-rep" % cfg)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rr[0], rr[1], rr[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
col = {w: hdr.index(w) for w in want if w in hdr}
kn = hdr.index("Kernel Name")
traffic = {}
lines = ["# %s — ncu --set full, cfg%d (one launch of each hot kernel, second step)" % (rnd, cfg), "",
         "`ncu --set full --clock-control none --import-source on -k 'regex:k_build_tc|k_query_tc|k_exact_select' "
         "-s 3 -c 3` on `tools/prof_step.py --config %d --steps 2`; report `gpurun_out/prof_cfg%d.ncu-rep` "
         "(scratch, not tracked)." % (cfg, cfg), ""]
for d in data:
    name = short(d[kn])
    lines.append("## `%s`" % name)
    lines.append("")
    lines.append("| metric | value | unit |")
    lines.append("|---|---:|---|")
    for w, i in col.items():
        lines.append("| %s | %s | %s |" % (w, d[i], units[i]))
    lines.append("")

    def val(w):
        v = float(d[col[w]].replace(",", ""))
        u = units[col[w]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    if "dram__bytes_read.sum" in col:
        traffic[name] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
open(os.path.join(out_dir, "%s_ncu_cfg%d.md" % (rnd, cfg)), "w").write("\n".join(lines) + "\n")
tj_path = os.path.join(out_dir, "traffic.json")
tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
tj["cfg%d" % cfg] = {"tc": traffic.get("void k_build_tc<1>"), "kernels": traffic,
                     "source": "%s_ncu_cfg%d.md (dram__bytes_read.sum + dram__bytes_write.sum, one launch)" % (rnd, cfg)}
json.dump(tj, open(tj_path, "w"), indent=1)
print("\n".join(lines[:60]))
