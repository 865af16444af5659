"""Regenerate the performance table of DESIGN.md §12 and the results rows of BASELINE.md §4 from
profiles/r02_bench.json (the committed bench line).  Usage: python tools/refresh_tables.py"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.loads(open(os.path.join(ROOT, "profiles", "r02_bench.json")).read().strip().splitlines()[-1])
c = d["configs"]


def design_row(name, x):
    b, q, r, rq = x["build"], x["query"], x["roofline"], x.get("roofline_query", {})
    return "| %s | %.2f | %.2f (%.2f / %.2f / %.2f) | %.3f (%.3f) | %.3f %s | %s | %d / %d |" % (
        name, x["ms_per_step"], b["ms"], b["contraction_ms"], b["select_blocks_ms"], b["prep_ms"], q["ms"],
        q["filter_ms"], r["frac"], "sustained" if "sustained" in r.get("peak_src", "") else "burst",
        ("%.3f" % rq["frac"]) if rq and rq.get("bound") == "hbm" else "L2-resident",
        x["parity"]["disagreements"], x["parity"]["in_band_pairs"])


p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
tab = ["| cfg | step ms | build ms (contraction / select+blocks / prep) | query ms (filter kernel) | build frac | "
       "query filter frac of HBM | disagreements / in-band |", "|---|---|---|---|---|---|---|",
       design_row("4 (headline)", d)] + [design_row(k[-1], c[k]) for k in ("cfg3", "cfg2", "cfg1", "cfg0")]
a = s.index("| cfg | step ms | build ms (contraction")
b = s.index("\n\n", a)
s = s[:a] + "\n".join(tab) + s[b:]
s = re.sub(r"Headline: [0-9.]+ ms per step, [0-9.e+]+ inner products/s \(round 1: 172 ms\); e2e through the host-buffer API [0-9.]+ ms",
           "Headline: %.1f ms per step, %.3g inner products/s (round 1: 172 ms); e2e through the host-buffer API %.1f ms"
           % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"]), s)
open(p, "w").write(s)

p = os.path.join(ROOT, "BASELINE.md")
s = open(p).read()
ks = c["cfg2"]["k_sweep"]
k2 = " / ".join("%.3g" % ks[k]["query"]["queries_per_s"] for k in ("k1", "k5", "k10", "k25")) + \
    " / %.3g" % c["cfg2"]["query"]["queries_per_s"]
R = {"0": c["cfg0"], "1": c["cfg1"], "2": c["cfg2"], "3": c["cfg3"], "4": d}
rows = [
    "| 0 | 10 | %.6f | %.3g | 0.5 %% (latency-bound) | %.3g (100) | L2-resident | < 0.1 (16) | — | 0 / %d (all 2,000 users) |"
    % (R["0"]["build"]["ms"] / 1e3, R["0"]["build"]["inner_products_per_s"], R["0"]["query"]["queries_per_s"],
       R["0"]["parity"]["in_band_pairs"]),
    "| 1 | 10 | %.5f | %.3g | %.1f %% of burst | %.3g (256) | L2-resident | 4.1 (16), r01 reference arm | — | 0 / %d (%d users) |"
    % (R["1"]["build"]["ms"] / 1e3, R["1"]["build"]["inner_products_per_s"], 100 * R["1"]["roofline"]["frac"],
       R["1"]["query"]["queries_per_s"], R["1"]["parity"]["in_band_pairs"], R["1"]["parity"]["users_sampled"]),
    "| 2 | 1,5,10,25,50 | %.5f | %.3g | %.1f %% of burst | %s (256) | L2-resident | ~14 (16), extrapolated | — | 0 at every k (%d users) |"
    % (R["2"]["build"]["ms"] / 1e3, R["2"]["build"]["inner_products_per_s"], 100 * R["2"]["roofline"]["frac"], k2,
       R["2"]["parity"]["users_sampled"]),
    "| 3 | 10 | %.4f | %.3g | %.1f %% of burst | %.3g (256) | %.1f %% | ~330 (16), extrapolated | — | 0 / %d (%d users) |"
    % (R["3"]["build"]["ms"] / 1e3, R["3"]["build"]["inner_products_per_s"], 100 * R["3"]["roofline"]["frac"],
       R["3"]["query"]["queries_per_s"], 100 * R["3"]["roofline_query"]["frac"], R["3"]["parity"]["in_band_pairs"],
       R["3"]["parity"]["users_sampled"]),
    "| 4 | 50 | %.4f | %.3g | **%.1f %% of sustained** | %.3g (256) | **%.1f %%** | ~8,400 (16), extrapolated from a 250-user sample (%.3g ip/s) | %.2g per 250 users | 0 / %d (250 users x 10,000 queries) |"
    % (d["build"]["ms"] / 1e3, d["build"]["inner_products_per_s"], 100 * d["roofline"]["frac"], d["query"]["queries_per_s"],
       100 * d["roofline_query"]["frac"], d["cpu_baseline"]["phase1_inner_products_per_s"],
       d["cpu_baseline"]["phase2_queries_per_s"], d["parity"]["in_band_pairs"])]
a = s.index("| 0 | 10 |")
b = s.index("\n\n", a)
s = s[:a] + "\n".join(rows) + s[b:]
s = re.sub(r"call\): [0-9.]+ ms,\n  [0-9.e+]+ inner products/s; e2e through the host-buffer API [0-9.]+ ms",
           "call): %.1f ms,\n  %.3g inner products/s; e2e through the host-buffer API %.1f ms"
           % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"]), s)
open(p, "w").write(s)
print("headline %.2f ms, %.4g ip/s" % (d["ms_per_step"], d["value"]))
