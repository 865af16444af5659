"""Round-2 profile summaries into profiles/ (tracked): the launch list of the headline bench step and the
key ncu --set full metrics of every captured hot kernel; profiles/traffic.json gets the DRAM bytes per
launch of the roofline kernels (bench.py roofline.traffic).  Usage: python tools/summarize_r02.py"""
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
KEYS = [("gpu__time_duration.sum", "duration"), ("sm__cycles_elapsed.avg", "SM cycles"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("lts__t_sector_hit_rate.pct", "L2 hit rate"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__inst_executed.sum", "instructions"), ("launch__registers_per_thread", "registers"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def short(name):
    name = name.replace("rmips::", "")
    if "cub::" in name:
        return "cub::" + name.split("cub::")[1].split("<")[0]
    return name.split("(")[0].replace("void ", "")


def launches(csv_path, title):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                             "msecond": 1e3}[r[ui]]
        agg[short(r[ki])][0] += 1
        agg[short(r[ki])][1] += v
        total += v
    lines = [title, "", "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare "
             "SHARES, not absolutes); %d launches, %.1f ms of kernel time (warm-up + 2 timed steps)."
             % (sum(c for c, _ in agg.values()), total / 1e3), "", "| kernel | launches | total ms | share |",
             "|---|---:|---:|---:|"]
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append("| `%s` | %d | %.3f | %.1f%% |" % (k, c, v / 1e3, 100 * v / total))
    return lines


def ncu(rep, title, how):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rr[0], rr[1], rr[2:]
    lines = [title, "", how, ""]
    out = {}
    for row in data:
        name = short(row[hdr.index("Kernel Name")])
        lines += ["## `%s`" % name, "", "| metric | value | unit |", "|---|---:|---|"]
        rec = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append("| %s (`%s`) | %s | %s |" % (label, key, row[i], units[i]))
                rec[key] = (row[i], units[i])
        lines.append("")
        out.setdefault(name, rec)
    return lines, out


def mbytes(v):
    val, unit = v
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    open(os.path.join(OUT, "r02_launches_cfg4.md"), "w").write("\n".join(launches(
        os.path.join(G, "r02_launches_cfg4.csv"),
        "# r02 -- launch list of the headline bench step (configs[4]): `bench.py --extra '' --steps 2`")) + "\n")
    traffic = json.load(open(os.path.join(OUT, "traffic.json"))) if os.path.exists(os.path.join(OUT, "traffic.json")) else {}
    caps = [("r02_cfg4_query", "# r02 -- ncu --set full, configs[4] query path (full size, one 256-query call)",
             "`tools/gpu_profile_r02.sh`: `ncu --set full -k regex:'k_query_tc|k_exact_select|k_exact_decide|k_bits_emit' -s 4 -c 5` on `tools/prof_step.py --config 4 --steps 1`."),
            ("r02_cfg4_build", "# r02 -- ncu --set full, configs[4]-shaped build (k_build_tc2cta)",
             "`tools/prof_step.py --config 4 --n 37888` (d = 200, m = 1,000,000; n cut to 296 user tiles = one pair per CTA pair twice)."),
            ("r02_cfg3", "# r02 -- ncu --set full, configs[3] (full size)", "`tools/prof_step.py --config 3 --steps 1`, -s 1 -c 3."),
            ("r02_cfg3_scan", "# r02 -- ncu --set full, configs[3] P' index (|P'| = 2 k_max): Alg. 2's verification scan",
             "`tools/prof_step.py --config 3 --steps 1 --pprime 2` (P32 = 100,000 x 56 x 4 B = 22 MB: L2-resident, so the scan's fraction is of L2, not HBM)."),
            ("r02_cfg1", "# r02 -- ncu --set full, configs[1] (full size)", "`tools/prof_step.py --config 1 --steps 2`, -s 3 -c 3."),
            ("r02_cfg4_prep", "# r02 -- ncu --set full, configs[4] build prep (norms, permute + convert)",
             "`tools/prof_step.py --config 4 --steps 1`, -k regex:'k_norms|k_prep_users|k_prep_items' -c 3.")]
    for rep, title, how in caps:
        p = os.path.join(G, rep + ".ncu-rep")
        if not os.path.exists(p):
            continue
        lines, out = ncu(p, title, how)
        open(os.path.join(OUT, rep.replace("r02_", "r02_ncu_") + ".md"), "w").write("\n".join(lines) + "\n")
        cfg = "cfg" + rep.split("cfg")[1][0]
        for name, rec in out.items():
            if "dram__bytes_read.sum" in rec:
                t = mbytes(rec["dram__bytes_read.sum"]) + mbytes(rec["dram__bytes_write.sum"])
                traffic.setdefault(cfg, {}).setdefault("kernels", {})[name] = t
                if name.startswith("k_build_tc"):
                    if "37888" not in how:
                        traffic[cfg]["tc"] = t
                    else:
                        traffic[cfg]["tc_note"] = "k_build_tc2cta on n = 37,888 users (296 tiles): %.0f bytes" % t
                if name.startswith("k_query_tc"):
                    traffic[cfg]["query"] = t
        traffic.setdefault(cfg, {})["source"] = "r02 ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum, one launch)"
    json.dump(traffic, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
