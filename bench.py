#!/usr/bin/env python3
"""bench.py -- one JSON line per run for the exact reverse k-MIPS hot path on B200.

A step = one pass of the whole hot path (SURVEY §8(a) rows B1-B6 + Q1-Q6) over one batch of
synthetic input: rmips_build_index over (Q, P), then rmips_query over the config's whole query set
in calls of the config's batch size (BASELINE.json configs[4]: 10,000 fresh queries "in batches of
256" = 40 calls), then rmips_free_index.  Inputs are device-resident when the timed region starts;
L2 (126 MB) is flushed before every timed step (a 512 MiB memset).

Default workload: BASELINE.json configs[4] -- d = 200, |Q| = 1,000,000 users, |P| = 1,000,000 items,
lognormal(0, 0.75) norms, k_max = 50, k = 50 -- the largest single-GPU configuration ("index build
dominated"); BASELINE.json's metric names no config.  configs[0..3] run after it as extra keys
("configs"), each with its own parity block (the small oracle case and the paper-shaped ones).

value = inner products evaluated exactly per second over the whole step:
        (n*m  [index build, Alg. 1 over all of P]  +  nq*n  [query x user]) / step time.
The JSON also carries the build rate (n*m / build time) and queries/s separately.

parity: the timed step's own output, checked against the fp64 oracle (oracle/) on a fixed user
sample (every query's decision for those users), with SURVEY §8(c)'s borderline bookkeeping:
disagreements and in-band pairs (|q.u - tau'_k(u)| <= 1e-5 |q||u|, reading R9).

--impl reference runs the reference arm: the fp64 CPU oracle, the only reference this paper has,
on a bounded user sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reverse k-MIPS queries/sec + index-build inner products/sec; % of roofline"
UNIT = "inner products/s (build n*m + query nq*n, whole step)"
BAND = 1e-5  # BASELINE north star: borderline users |q.u - tau_k(u)| <= 1e-5 |q||u|


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML initialisation) can stall CUDA work for ~0.2 s: wait for its
            # first samples so that it happens before the timed region
            t0 = time.perf_counter()
            while len(self.lines) < 3 and time.perf_counter() - t0 < 10:
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if t0 is not None and not (t0 <= ts <= t1):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _batches(nq, bs):
    return [(b0, min(nq, b0 + bs)) for b0 in range(0, nq, bs)]


# ------------------------------------------------------------------------------ the oracle legs

def oracle_sample(w, k, users: int, threads: int, seed: int):
    """The fp64 oracle on a fixed user sample of the workload: phase 1 = exact top-(k_max + 1) lists
    over all of P (Alg. 1 lines 7-9 over P, the index build's analogue), phase 2 = every query's
    decision for those users (two-phase form, equal to Def. 2 by reading R8).  Timed separately."""
    import oracle
    spec = w.spec
    rng = np.random.default_rng(seed)
    sample = np.sort(rng.choice(spec.n, min(users, spec.n), replace=False))
    Us = np.ascontiguousarray(w.U[sample])
    t0 = time.perf_counter()
    vals, ids = oracle.topk(Us, w.P, spec.k_max + 1, threads=threads)
    t1 = time.perf_counter()
    member = oracle.rkmips_twophase(Us, np.ascontiguousarray(vals[:, :spec.k_max]), w.Qy, k, threads=threads)
    t2 = time.perf_counter()
    return sample, vals, ids, member, t1 - t0, t2 - t1


def cpu_baseline(w, k, users: int, users_1t: int, seed: int = 2):
    """The oracle as it stands, timed on the host: all cores on `users` sampled users, and one thread on
    `users_1t` of them (phase 1 inner products/s and phase 2 queries/s reported separately)."""
    spec = w.spec
    cores = os.cpu_count() or 1
    sample, vals, ids, member, p1, p2 = oracle_sample(w, k, users, cores, seed)
    s1 = oracle_sample(w, k, users_1t, 1, seed + 1)
    S, S1 = len(sample), len(s1[0])
    units = S * spec.m + spec.nq * S
    out = {"value": units / (p1 + p2), "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
           "sample": "%d of %d users: exact fp64 top-%d over all %d items (phase 1, %.2f s) + %d query decisions "
                     "each (phase 2, %.2f s), %d threads" % (S, spec.n, spec.k_max + 1, spec.m, p1, spec.nq, p2, cores),
           "phase1_inner_products_per_s": S * spec.m / p1,
           "phase2_queries_per_s": spec.nq / p2, "phase2_note": "decisions for the %d sampled users per query" % S,
           "one_thread": {"users": S1, "phase1_inner_products_per_s": S1 * spec.m / s1[4],
                          "phase2_queries_per_s": spec.nq / s1[5], "value": (S1 * spec.m + spec.nq * S1) / (s1[4] + s1[5])}}
    return out, (sample, vals, ids, member)


def parity_block(w, k, sets, sample, vals, ids, member, threads):
    """SURVEY §8(c) comparison procedure on the sampled users: per query, GPU set restricted to the
    sample vs the oracle's; every disagreement's margin; in-band pairs over all (query, sampled user)."""
    import oracle
    spec = w.spec
    nq = len(sets)
    assert nq == spec.nq
    mine = np.zeros((nq, len(sample)), bool)
    ascending = True
    for qi, s_ in enumerate(sets):
        ascending &= bool((np.diff(s_) > 0).all())
        mine[qi] = np.isin(sample, s_, assume_unique=True)
    dis = np.argwhere(mine != member)
    qq, jj = np.meshgrid(np.arange(nq, dtype=np.int64), np.arange(len(sample), dtype=np.int64), indexing="ij")
    pairs = np.stack([qq.ravel(), jj.ravel()], axis=1)
    mu = oracle.margins_from_lists(w.U[sample], w.P, w.Qy, vals, ids, pairs, k, threads=threads)
    inband = int((np.abs(mu) <= BAND).sum())
    dis_mu = mu[dis[:, 0] * len(sample) + dis[:, 1]] if len(dis) else np.zeros(0)
    excused = int((np.abs(dis_mu) <= BAND).sum())
    return {"users_sampled": int(len(sample)), "queries": nq, "pairs_checked": int(nq * len(sample)),
            "disagreements": int(len(dis)), "excused_borderline": excused, "hard_failures": int(len(dis)) - excused,
            "in_band_pairs": inband, "sets_ascending": ascending,
            "oracle_members": int(member.sum()), "gpu_members": int(mine.sum()),
            "rule": "identical sets except |q.u - tau'_k(u)| <= 1e-5 |q||u| (tau' over P minus copies of q, R9)"}


# ------------------------------------------------------------------------------ reference arm (oracle)

def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from synth import make_workload
    w = make_workload(args.config)
    spec = w.spec
    k = args.k or spec.ks[-1]
    cores = os.cpu_count() or 1
    S = args.ref_users or (64 if spec.m * spec.d > 1e8 else 1000)
    times = []
    for it in range(args.warmup + args.steps):
        _, _, _, _, p1, p2 = oracle_sample(w, k, S, cores, 100 + it)
        if it >= args.warmup:
            times.append(p1 + p2)
    units = S * spec.m + spec.nq * S
    t = sum(times) / len(times)
    v = units / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY Appendix C generator, seed 0)",
            "config": _config_dict(spec, k, ws) | {"ref_user_sample": S},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
                             "sample": "%d of %d users per step: exact fp64 top-%d over all %d items + %d query "
                                       "decisions each" % (S, spec.n, spec.k_max + 1, spec.m, spec.nq)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _config_dict(spec, k, ws):
    return {"workload": spec.name, "n": spec.n, "m": spec.m, "d": spec.d, "k_max": spec.k_max, "queries": spec.nq,
            "k": k, "query_batch": "%d batches of <= %d queries" % (len(_batches(spec.nq, spec.batch)), spec.batch),
            "l2": "flushed (512 MiB memset) before every timed step", "parallelism": "user-shard x%d" % ws}


# ------------------------------------------------------------------------------ our arm

def run_config(cfg, args, dev, rank, ws, steps, warmup, parity_users, e2e=True, cpu=True, k=None):
    import torch
    from paper_2110_07131_b200 import rmips
    from synth import make_workload

    from paper_2110_07131_b200.shard import gather_csr, user_shard
    from synth.generator import CONFIGS

    # N > 1: ONE problem sharded by users -- rank 0 generates the workload and
    # broadcasts the users, the items and the queries over NCCL; each rank keeps its contiguous user
    # range [a, b), builds its own index and answers every query batch; the per-query lists are
    # exchanged device-side (shard.gather_csr) inside the timed step.  Strong scaling: the total work is
    # the config's, whatever N.
    spec = CONFIGS[cfg]
    w = make_workload(cfg, seed=0) if rank == 0 else None
    k = k or args.k or spec.ks[-1]
    if ws > 1:
        nq_eff = spec.nq if spec.query_mode != "from_p" else min(spec.nq, spec.m)
        Uf = torch.from_numpy(w.U).to(dev) if rank == 0 else torch.empty(spec.n, spec.d, device=dev)
        P = torch.from_numpy(w.P).to(dev) if rank == 0 else torch.empty(spec.m, spec.d, device=dev)
        Qy = torch.from_numpy(w.Qy).to(dev) if rank == 0 else torch.empty(nq_eff, spec.d, device=dev)
        for t_ in (Uf, P, Qy):
            torch.distributed.broadcast(t_, 0)
        sa, sb = user_shard(spec.n, ws, rank)
        U = Uf[sa:sb].contiguous()
        del Uf
    else:
        sa, sb = 0, spec.n
        U = torch.from_numpy(w.U).to(dev)
        P = torch.from_numpy(w.P).to(dev)
        Qy = torch.from_numpy(w.Qy).to(dev)
    batches = _batches(spec.nq, spec.batch)
    Qb = [Qy[a:b] for a, b in batches]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    bflags = rmips.RMIPS_BUILD_TIMING | (rmips.RMIPS_BUILD_SIMT if args.simt else 0)
    qflags = rmips.RMIPS_FLAG_TIMING | (rmips.RMIPS_FLAG_SIMT if args.simt else 0)
    stream = torch.cuda.current_stream()
    m_prime = args.pprime * spec.k_max if args.pprime else 0
    cap = [None]  # learned during the warm-up steps (the first call sizes itself: rmips.py retries once)
    host_build_ms = []

    def step():
        """One pass of the hot path: build + every query call.  Per-call phase times and counters are
        read right after each call (host reads of values the call already synchronised on)."""
        tb0 = time.perf_counter()
        if m_prime:
            idx = rmips.rmips_build_index_pprime(U, P, spec.k_max, m_prime, bflags)
        else:
            idx = rmips.rmips_build_index(U, P, spec.k_max, bflags)
        host_build_ms.append((time.perf_counter() - tb0) * 1e3)
        outs, qph = [], []
        if args.query_api == "batches":  # every batch of the config in one call, one host sync
            qsets = [(Qy, rmips.rmips_query_batches)]
        else:  # one rmips_query call (and host sync) per batch
            qsets = [(q, None) for q in Qb]
        for q, fn in qsets:
            if fn is not None:
                off, ids = fn(idx, q, spec.batch, k, qflags, capacity=cap[0])
            else:
                off, ids = rmips.rmips_query(idx, q, k, qflags, capacity=cap[0])
            qph.append((idx.phase_times(), idx.stats()))
            if ws > 1:  # the exchange step: every rank gets the global lists (NCCL all_gathers)
                off, ids = gather_csr(off, ids, sa)
            outs.append((off, ids))
        return idx, outs, qph

    def readout(idx, outs, qph):
        pt = idx.phase_times()  # build phases (ms[0..3], launches ms[14]) survive the queries
        rec = {"prep": pt[0], "contraction": pt[1], "select": pt[2], "build": pt[3], "build_launches": pt[14],
               "cand_per_user": idx.cand_total / max(1, spec.n), "tiles_issued": idx.tiles_done,
               "build_kernel": idx.build_kernel,
               "q_prep": sum(p[8] for p, _ in qph), "q_filter": sum(p[9] for p, _ in qph),
               "q_exact": sum(p[10] for p, _ in qph), "q_output": sum(max(0.0, p[11]) for p, _ in qph),
               "q_total": sum(p[12] for p, _ in qph), "q_launches": sum(p[15] for p, _ in qph),
               "q_kernel": sum(max(0.0, p[13]) for p, _ in qph),
               "tiles_scored": sum(s["tiles_scored"] for _, s in qph), "scans": sum(s["scans"] for _, s in qph),
               "items_scanned": sum(s["items_scanned"] for _, s in qph),
               "undecided": sum(s["pairs_undecided"] for _, s in qph),
               "filter_kernel": min(s["filter_kernel"] for _, s in qph),
               "result_total": sum(s["result_total"] for _, s in qph)}
        need = max(int(o[1].numel()) for o in outs)
        if cap[0] is None or need > cap[0] // 2:
            cap[0] = max(1 << 16, 2 * need)
        idx.close()
        return rec

    # the clock sampler starts before the warm-up steps: nvidia-smi's start-up (NVML initialisation)
    # stalled CUDA calls for ~0.2 s when it overlapped the first timed steps
    sampler = ClockSampler(dev.index)
    sampler.__enter__()
    ts0 = time.perf_counter()
    for _ in range(warmup):
        readout(*step())
    while time.perf_counter() - ts0 < 2.0:  # at least 2 s of sampling before the timed region
        if ws > 1:  # (every rank must run the same steps: their collectives pair up)
            time.sleep(0.05)
        else:
            readout(*step())
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    step_ms, recs, host_ms = [], [], []
    last = None
    import gc
    gc.collect()
    gc.disable()  # (no collector pause inside the timed region; re-enabled right after it)
    try:
        tw0 = time.perf_counter()
        for si in range(steps):
            flush.zero_()                               # L2 flush, outside the timed region
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            th0 = time.perf_counter()
            idx, outs, qph = step()
            host_ms.append((time.perf_counter() - th0) * 1e3)
            e1.record(stream)
            torch.cuda.synchronize()
            recs.append(readout(idx, outs, qph))        # (frees the index: stream-ordered, after e1)
            step_ms.append(e0.elapsed_time(e1))
            if si == steps - 1:
                last = outs  # (only the last step's lists are kept: the device memory of every step is
                             # reused by the next, so no step allocates more than the warm-up ones did)
            del outs
        tw1 = time.perf_counter()
    finally:
        sampler.__exit__(None, None, None)
    gc.enable()
    clocks = sampler.summary(tw0, tw1)
    torch.cuda.synchronize()
    t_rank = sum(step_ms)
    if ws > 1:
        t = torch.tensor([t_rank], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        t_max = t_rank
    units_step = spec.n * spec.m + spec.nq * spec.n  # the whole config, split over the ws ranks
    value = units_step * steps / (t_max / 1e3)
    ms_per_step = t_max / steps
    med = lambda key: float(np.median([r[key] for r in recs]))  # noqa: E731
    peaks = _peaks()

    # ---- roofline of the dominant kernel: the build contraction (B4), tensor-core bound.
    # achieved = algorithmic flops of the (user tile, item tile) contractions actually issued (2 d per
    # user-item pair; tiles skipped by the Cauchy-Schwarz exit are not counted) / the contraction time;
    # effective = 2 n m d / time counts the pruned pairs too.
    kern_ms = med("contraction")
    tiles = med("tiles_issued")
    flops_eff = 2.0 * spec.n * spec.m * spec.d
    flops = 2.0 * tiles * 128 * 128 * spec.d if tiles > 0 else flops_eff
    achieved = flops / (kern_ms / 1e3) / 1e12
    # burst peak for a kernel timed alone (ms-scale), the sustained peak (back-to-back matmul for 4 s,
    # power-capped clocks) for one that runs for tens of ms inside a long step
    sustained = kern_ms > 20.0 and peaks.get("bf16_tflops_sustained")
    peak = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    kname = {0: "k_build_simt", 1: "k_build_tc", 2: "k_build_tcq", 3: "k_build_tcq (streamed A)",
             4: "k_build_tc2cta (CTA pairs, cta_group::2; head pass + regrouped main pass when n >= 4 x 148 x 128"
                ", m >= 512 x 128)"}.get(recs[-1]["build_kernel"], "?")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get("cfg%d" % cfg, {}).get("simt" if args.simt else "tc")
    roof = {"bound": "tensor", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_src": ("MEASURED_PEAKS.json %s (fp16 has the bf16 dense rate)"
                         % ("bf16_tflops_sustained" if sustained else "bf16_tflops (burst)"))
            if peaks["src"] == "measured" else "fallback (B200_PROFILING.md)",
            "flops_per_launch": flops, "flop_unit": "2 d per (user, item) pair of the issued 128 x 128 tiles",
            "tiles_issued": tiles, "kernel_ms": kern_ms,
            "launches_per_build": 2 if recs[-1]["build_kernel"] == 4 and spec.n >= 4 * 148 * 128 and spec.m >= 512 * 128 else 1,
            "time_basis": "the build's contraction phase (CUDA events): every contraction launch of the build (head + "
                          "regrouped main pass where they apply) and the regroup sort / gather between them; flops "
                          "are those of all issued tiles (seed-pass repeats not counted)",
            "effective_tflops_incl_pruned": flops_eff / (kern_ms / 1e3) / 1e12,
            "share_of_step": kern_ms / ms_per_step}

    # ---- the query filter (Q2+Q3, k_query_tc): HBM-bound stream of the users' fp16 rows + thresholds
    qf_ms = med("q_kernel") if med("q_kernel") > 0 else med("q_filter")  # the kernel alone, else the phase
    qbytes = med("tiles_scored") * 128 * (2 * spec.d + 4)
    ubytes = spec.n * (2 * spec.d + 4)
    roof_q = {"bound": "hbm" if ubytes > 126e6 else "l2 (user rows fit in the 126 MB L2)",
              "kernel": "k_query_simt" if args.simt else "k_query_tc",
              "achieved": qbytes / (qf_ms / 1e3) / 1e9 if qf_ms > 0 else None, "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": (qbytes / (qf_ms / 1e3) / 1e9) / peaks["hbm_gbs"] if qf_ms > 0 else None,
              "bytes_per_step": qbytes, "byte_unit": "(2 d + 4) B per user of every 128-user tile Lemma 3 keeps, "
                                                      "per query call", "kernel_ms_per_step": qf_ms,
              "timing": "CUDA events right around each k_query_tc launch, summed over the step's calls",
              "phase_ms_per_step": med("q_filter"),
              "calls": len(batches)}
    # the same kernel against the tensor roofline: at d = 200 a 256-query call is ~1.1e11 flop of MMA for
    # ~0.4 GB of user rows, so the filter is co-bound (upper bound of the issued flops: MMA N = the Lemma 3
    # prefix <= the sub-batch's queries)
    qcols = min(256, max(b_ - a_ for a_, b_ in batches)) if batches else 0
    qflops = med("tiles_scored") * 128 * qcols * 2 * (16 * ((spec.d + 15) // 16))
    # (sustained peak when the calls run inside a long, power-capped step, as the build's)
    qpeak = peaks["bf16_tflops_sustained"] if ms_per_step > 20.0 and peaks.get("bf16_tflops_sustained") else peaks["bf16_tflops"]
    if qf_ms > 0 and not args.simt:
        roof_q["tensor"] = {"achieved": qflops / (qf_ms / 1e3) / 1e12, "peak": qpeak, "unit": "TFLOP/s",
                            "frac": qflops / (qf_ms / 1e3) / 1e12 / qpeak,
                            "flop_unit": "2 K_pad per (user, query) slot of every scored 128-user x <= 256-query tile",
                            "peak_src": "bf16_tflops_sustained" if qpeak == peaks.get("bf16_tflops_sustained") else "bf16_tflops (burst)"}

    # ---- the verification scan (Q5, k_verify_scan), P' index only
    roof_s = None
    if m_prime:
        ex_ms = med("q_exact")
        sbytes = med("items_scanned") * 4 * (((spec.d + 7) // 8) * 8)
        p32 = spec.m * 4 * (((spec.d + 7) // 8) * 8)
        roof_s = {"bound": "hbm" if p32 > 126e6 else "l2 (P32 fits in the 126 MB L2)",
                  "kernel": "k_exact_decide_pp + k_verify_scan", "kernel_ms": ex_ms, "scans": med("scans"),
                  "items_scanned": med("items_scanned"), "bytes_per_step": sbytes,
                  "achieved": sbytes / (ex_ms / 1e3) / 1e9 if ex_ms > 0 else None, "peak": peaks["hbm_gbs"],
                  "unit": "GB/s", "frac": (sbytes / (ex_ms / 1e3) / 1e9) / peaks["hbm_gbs"] if ex_ms > 0 else None}

    res = {"value": value, "ms_per_step": ms_per_step, "steps": steps, "warmup": warmup,
           "step_ms": [round(x, 3) for x in step_ms], "host_ms": [round(x, 3) for x in host_ms],
           "host_build_ms": [round(x, 3) for x in host_build_ms[-steps:]],
           "config": _config_dict(spec, k, ws) | {"kernels": "simt" if args.simt else "tcgen05"},
           "build": {"ms": med("build"), "inner_products_per_s": spec.n * spec.m / (med("build") / 1e3),
                     "contraction_ms": kern_ms, "prep_ms": med("prep"), "select_blocks_ms": med("select"),
                     "candidates_per_user": med("cand_per_user")},
           "query": {"ms": med("q_total"), "queries_per_s": spec.nq / (med("q_total") / 1e3), "calls": len(batches),
                     "api": "rmips_query_batches (one call, %d batches)" % len(batches) if args.query_api == "batches"
                     else "%d rmips_query calls" % len(batches),
                     "prep_ms": med("q_prep"), "filter_ms": qf_ms, "filter_phase_ms": med("q_filter"), "exact_ms": med("q_exact"),
                     "output_ms": med("q_output"), "undecided_pairs": med("undecided"),
                     "result_ids": recs[-1]["result_total"], "filter_kernel_tcgen05": bool(recs[-1]["filter_kernel"]),
                     "wall_ms_incl_host": ms_per_step - med("build")},
           "roofline": roof, "roofline_query": roof_q, "clocks": clocks,
           "gpu_launches": int(med("build_launches") + med("q_launches")) * steps}
    if m_prime:
        res["roofline_scan"] = roof_s
        res["index"] = "P' over the first %d items (Alg. 1 line 6)" % m_prime

    # ---- parity of the last timed step's output against the oracle (sampled users), rank 0
    sets = None
    if parity_users and rank == 0:
        sets = []
        for off, ids in last:
            sets += rmips.split_sets(off, ids)
    del last

    # ---- end to end through the public API with HOST buffers (copies inside the timed region)
    if e2e:
        Uh = U.cpu().pin_memory()  # this rank's users (all of them at N = 1)
        Ph = P.cpu().pin_memory()
        Qh = [Qy.cpu().pin_memory()] if args.query_api == "batches" else [Qy[a:b].cpu().pin_memory() for a, b in batches]
        offh = [torch.empty(q.shape[0] + 1, dtype=torch.int64).pin_memory() for q in Qh]
        idsh = torch.empty(cap[0], dtype=torch.int32).pin_memory()
        e2e_ms, d2h = [], 0
        for it in range(warmup + steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            idx = rmips.rmips_build_index_host(Uh, Ph, spec.k_max)
            d2h = 0
            for j, q in enumerate(Qh):
                if args.query_api == "batches":
                    off, ids = rmips.rmips_query_batches_host(idx, q, spec.batch, k, out_offsets=offh[j], out_ids=idsh,
                                                              capacity=idsh.numel())
                else:
                    off, ids = rmips.rmips_query_host(idx, q, k, out_offsets=offh[j], out_ids=idsh,
                                                      capacity=idsh.numel())
                if ws > 1:  # the exchange: this rank's host lists -> device -> NCCL gather -> host
                    g_off, g_ids = gather_csr(off.to(dev, non_blocking=True), ids.to(dev, non_blocking=True), sa)
                    off, ids = g_off.cpu(), g_ids.cpu()
                d2h += 8 * int(off.numel()) + 4 * int(len(ids))
            e1.record(stream)
            torch.cuda.synchronize()
            idx.close()
            if it >= warmup:
                e2e_ms.append(e0.elapsed_time(e1))
        t_e2e = sum(e2e_ms)
        if ws > 1:
            t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            t_e2e = float(t.item())
        res["e2e"] = {"value": units_step * steps / (t_e2e / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": 4 * spec.d * ((sb - sa) + spec.m + spec.nq), "d2h_bytes_per_step": d2h,
                      "ms_per_step": t_e2e / steps,
                      "api": ("rmips_build_index_host + rmips_query_batches_host (%d batches, pinned host buffers)%s"
                              if args.query_api == "batches" else
                              "rmips_build_index_host + %d rmips_query_host calls (pinned host buffers)%s")
                             % (len(batches), " + shard.gather_csr" if ws > 1 else "")}
    del U, P, Qy, Qb, flush
    torch.cuda.empty_cache()

    if rank == 0 and (cpu or parity_users):
        if w is None:
            w = make_workload(cfg, seed=0)
        cores = os.cpu_count() or 1
        if cpu and ws == 1:
            base, orc = cpu_baseline(w, k, parity_users, args.cpu_users_1t)
            res["cpu_baseline"] = base
        else:
            s_, v_, i_, m_, _, _ = oracle_sample(w, k, parity_users, cores, 2)
            orc = (s_, v_, i_, m_)
        if sets is not None:
            res["parity"] = parity_block(w, k, sets, *orc, threads=cores)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rmips", choices=["rmips", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--k", type=int, default=0, help="0 = the config's k (the last of its sweep for configs[2])")
    ap.add_argument("--extra", default="0,1,2,3", help="configs run after the headline one (extra keys); '' = none")
    ap.add_argument("--extra-steps", type=int, default=5)
    ap.add_argument("--simt", action="store_true", help="CUDA-core build/query kernels instead of tcgen05")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parity-users", type=int, default=0, help="oracle user sample (0 = per-config default)")
    ap.add_argument("--cpu-users-1t", type=int, default=8, help="users of the one-thread oracle timing")
    ap.add_argument("--ref-users", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pprime", type=int, default=0,
                    help="NEXT-1: build the P' index over the first C * k_max items (Alg. 1 as printed) "
                         "and answer through Lemmas 1-2 and Alg. 2's scan; 0 = exact index over all of P")
    ap.add_argument("--query-api", default="batches", choices=["batches", "calls"],
                    help="batches: one rmips_query_batches call per step (the config's batches back to back, one "
                         "host sync); calls: one rmips_query call per batch")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)

    import __graft_entry__
    __graft_entry__.build()

    def pusers(cfg, budget=1.5e10):
        """oracle user sample: about `budget` fp64 MAC of phase 1 (~2-6 s on the box's cores)"""
        if args.parity_users:
            return args.parity_users
        from synth.generator import CONFIGS
        s = CONFIGS[cfg]
        return int(min(s.n, max(64, budget / (s.m * s.d))))

    head = run_config(args.config, args, dev, rank, ws, args.steps, args.warmup, pusers(args.config, 5e10),
                      e2e=not args.no_e2e, cpu=not args.no_cpu_baseline)
    line = {"metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "fp16 filter (fp32 accumulate) + f64 exact decisions",
            "data": "synthetic (SURVEY Appendix C generator, seed 0; at N > 1 one problem split by users); stands in "
                    "for the paper's MF vectors (P:571-587), configs[4] is beyond the paper"}
    for key in ("step_ms", "host_ms", "host_build_ms", "config", "build", "query", "roofline", "roofline_query", "roofline_scan", "index", "clocks",
                "gpu_launches", "e2e", "cpu_baseline", "parity"):
        if key in head:
            line[key] = head[key]
    extras = {}
    for c in [int(x) for x in args.extra.split(",") if x.strip() != ""]:
        if c == args.config:
            continue
        r = run_config(c, args, dev, rank, ws, args.extra_steps, 3, pusers(c), e2e=False, cpu=False)
        extras["cfg%d" % c] = {kk: r[kk] for kk in ("value", "ms_per_step", "step_ms", "host_ms", "host_build_ms", "config", "build", "query", "roofline",
                                                    "roofline_query", "clocks", "parity") if kk in r}
        if c == 2 and args.k == 0:  # configs[2] sweeps k over {1, 5, 10, 25, 50}: the other k values
            from synth.generator import CONFIGS
            sweep = {}
            for kk in CONFIGS[2].ks[:-1]:
                r2 = run_config(c, args, dev, rank, ws, 3, 3, pusers(c), e2e=False, cpu=False, k=kk)
                sweep["k%d" % kk] = {x: r2[x] for x in ("value", "ms_per_step", "query", "parity") if x in r2}
            extras["cfg2"]["k_sweep"] = sweep
    if extras:
        line["configs"] = extras
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
