"""NEXT-3: the paper's experiment axes on synthetic data, on one B200.

Axes, on the configs[1] recipe (MovieLens-shaped MF vectors, d = 50, k_max = 50, 1,000 queries from P):
  blocks ablation  Lemma 3 on / off (RMIPS_FLAG_NO_BLOCKS), exact index and P' index
  k sweep  k in {1, 5, 10, 25, 50}
  |Q| sweep  n in {25k, 50k, 100k, 200k}
  |P| sweep  m in {6.25k, 12.5k, 25k, 50k}
For each point: build and query device times (CUDA events, median of 3 after a warm-up), and the
Theorem 3 counters: alpha = block-query pairs pruned by Lemma 3 / all, m' = items per
scan, #ip = inner products evaluated (build n x |P'| + query pairs scored + items scanned).
Both indexes answer identically (the parity tests); here only cost is measured.
Writes profiles/<round>_experiments.{md,json}.  Usage: python tools/experiments.py r01
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_07131_b200 import rmips  # noqa: E402
from synth.generator import make_workload  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
dev = torch.device("cuda", 0)


def run_point(n, m, k, pprime, blocks=True, reps=3):
    w = make_workload(1, n=n, m=m)
    U = torch.from_numpy(w.U).to(dev)
    P = torch.from_numpy(w.P).to(dev)
    Qy = torch.from_numpy(w.Qy).to(dev)
    k_max = w.spec.k_max
    qflags = rmips.RMIPS_FLAG_TIMING | (0 if blocks else rmips.RMIPS_FLAG_NO_BLOCKS)
    res = []
    for r in range(reps + 1):
        if pprime:
            idx = rmips.rmips_build_index_pprime(U, P, k_max, pprime * k_max, rmips.RMIPS_BUILD_TIMING)
        else:
            idx = rmips.rmips_build_index(U, P, k_max, rmips.RMIPS_BUILD_TIMING)
        tb = idx.phase_times()[3]
        off, ids = rmips.rmips_query(idx, Qy, k, qflags)
        tq = idx.phase_times()[12]
        st = idx.stats()
        idx.close()
        if r:
            res.append((tb, tq, st))
    tb = float(np.median([x[0] for x in res]))
    tq = float(np.median([x[1] for x in res]))
    st = res[-1][2]
    mp = min(m, pprime * k_max) if pprime else m
    bp = max(1, st["block_query_pairs"])
    return {"n": n, "m": m, "k": k, "index": "P'=%d" % mp if pprime else "exact", "blocks": blocks,
            "build_ms": tb, "query_ms": tq, "total_ms": tb + tq,
            "alpha": st["block_query_pruned"] / bp, "pairs_scored": st["pairs_scored"],
            "pairs_undecided": st["pairs_undecided"], "scans": st["scans"],
            "m_prime_per_scan": st["items_scanned"] / max(1, st["scans"]),
            "ip": n * mp + st["pairs_scored"] + st["items_scanned"], "result_total": st["result_total"]}


rows = {"blocks": [], "k": [], "Q": [], "P": []}
for pp in (0, 2):
    for b in (True, False):
        rows["blocks"].append(run_point(100_000, 25_000, 10, pp, b))
for pp in (0, 2):
    for k in (1, 5, 10, 25, 50):
        rows["k"].append(run_point(100_000, 25_000, k, pp))
for pp in (0, 2):
    for n in (25_000, 50_000, 100_000, 200_000):
        rows["Q"].append(run_point(n, 25_000, 10, pp))
for pp in (0, 2):
    for m in (6_250, 12_500, 25_000, 50_000):
        rows["P"].append(run_point(100_000, m, 10, pp))

os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(rows, open(os.path.join(ROOT, "profiles", "%s_experiments.json" % rnd), "w"), indent=1)
cols = ["index", "n", "m", "k", "blocks", "build_ms", "query_ms", "total_ms", "alpha", "pairs_scored", "scans",
        "m_prime_per_scan", "ip", "result_total"]
titles = {"blocks": "Blocks ablation (Lemma 3 on/off; P:611-617), k = 10",
          "k": "k sweep (P:620-643)", "Q": "|Q| sweep (P:693-703), k = 10", "P": "|P| sweep (P:731-739), k = 10"}
out = ["# %s — the paper's experiment axes on the configs[1] recipe (one B200)" % rnd, "",
       "`tools/experiments.py`: device times (CUDA events, median of 3 after a warm-up; no L2 flush), Theorem 3 "
       "counters (P:531-560): alpha = (block, query) pairs pruned by Lemma 3 / all, m' = items per scan, "
       "#ip = inner products evaluated (build n x |P'| + query pairs scored + items scanned).  'exact' = the "
       "hot-path index (lists over all of P); \"P'\" = Alg. 1 as printed with |P'| = 2 k_max (NEXT-1).", ""]
for key in ("blocks", "k", "Q", "P"):
    out += ["## " + titles[key], "", "| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for r in rows[key]:
        vals = []
        for c in cols:
            v = r[c]
            vals.append("%.3f" % v if isinstance(v, float) else str(v))
        out.append("| " + " | ".join(vals) + " |")
    out.append("")
open(os.path.join(ROOT, "profiles", "%s_experiments.md" % rnd), "w").write("\n".join(out))
print("\n".join(out))
