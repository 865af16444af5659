"""Pinned synthetic generator for the five BASELINE.json configs.

Follows SURVEY.md Appendix C bit-for-bit (numpy PCG64 via SeedSequence.spawn):

    ss = SeedSequence(seed); rng_u, rng_p, rng_q = default_rng(s) for s in ss.spawn(3)
    vecs(rng, count, d, sigma, offset) = N(0,1) direction * lognormal(0, sigma) norm + offset  -> fp32

The data ARE the fp32 values returned here.  Stand-in for the paper's LIBMF
matrix-factorisation vectors (§5.1: d = 50 vectors,
"randomly chose 1,000 vectors as query vectors from P"), which are not in the
container.  Table 2 sizes are mirrored by configs 1-3.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    name: str
    d: int
    n: int            # |Q| users
    m: int            # |P| items
    sigma: float      # lognormal sigma of vector norms
    item_offset: float
    k_max: int
    nq: int           # number of queries
    ks: tuple         # k values evaluated
    query_mode: str   # "from_p" | "half_fresh" | "fresh"
    batch: int        # query batch size used by the bench / parity tests


# BASELINE.json "configs" restated.
CONFIGS = {
    0: ConfigSpec("cfg0-tiny", 50, 2_000, 1_000, 0.5, 0.0, 10, 100, (10,), "from_p", 100),
    1: ConfigSpec("cfg1-movielens-shape", 50, 100_000, 25_000, 0.5, 0.1, 50, 1_000, (10,), "from_p", 256),
    2: ConfigSpec("cfg2-netflix-shape", 50, 480_000, 18_000, 0.5, 0.1, 50, 1_000, (1, 5, 10, 25, 50), "from_p", 256),
    3: ConfigSpec("cfg3-amazon-shape-heavytail", 50, 2_000_000, 100_000, 1.0, 0.1, 25, 1_000, (10,), "half_fresh", 256),
    4: ConfigSpec("cfg4-d200-1Mx1M", 200, 1_000_000, 1_000_000, 0.75, 0.0, 50, 10_000, (50,), "fresh", 256),
}


@dataclasses.dataclass
class Workload:
    spec: ConfigSpec
    U: np.ndarray            # [n, d] fp32 users (Q in the paper)
    P: np.ndarray            # [m, d] fp32 items
    Qy: np.ndarray           # [nq, d] fp32 query items
    q_item: np.ndarray       # [nq] int64: index into P if the query was drawn from P, else -1
    seed: int


def vecs(rng: np.random.Generator, count: int, d: int, sigma: float, offset: float) -> np.ndarray:
    g = rng.standard_normal((count, d))
    r = rng.lognormal(mean=0.0, sigma=sigma, size=count)
    v = g / np.linalg.norm(g, axis=1, keepdims=True) * r[:, None] + offset
    return v.astype(np.float32)


def make_workload(cfg, seed: int = 0, n: Optional[int] = None, m: Optional[int] = None,
                  nq: Optional[int] = None, d: Optional[int] = None) -> Workload:
    """Generate a config's inputs. n/m/nq/d overrides shrink a config for tests
    (same recipe, different sizes: the bytes then differ from the full config)."""
    spec = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if any(v is not None for v in (n, m, nq, d)):
        spec = dataclasses.replace(spec, n=n or spec.n, m=m or spec.m, nq=nq or spec.nq, d=d or spec.d,
                                   name=spec.name + "-resized")
    ss = np.random.SeedSequence(seed)
    rng_u, rng_p, rng_q = [np.random.default_rng(s) for s in ss.spawn(3)]
    U = vecs(rng_u, spec.n, spec.d, spec.sigma, 0.0)
    P = vecs(rng_p, spec.m, spec.d, spec.sigma, spec.item_offset)
    if spec.query_mode == "from_p":
        nq_eff = min(spec.nq, spec.m)
        idx = rng_q.choice(spec.m, nq_eff, replace=False)
        Qy = P[idx].copy()
        q_item = idx.astype(np.int64)
    elif spec.query_mode == "half_fresh":
        h = min(spec.nq // 2, spec.m)
        idx = rng_q.choice(spec.m, h, replace=False)
        fresh = vecs(rng_q, spec.nq - h, spec.d, spec.sigma, spec.item_offset)
        Qy = np.concatenate([P[idx], fresh]).astype(np.float32)
        q_item = np.concatenate([idx.astype(np.int64), -np.ones(spec.nq - h, np.int64)])
    elif spec.query_mode == "fresh":
        Qy = vecs(rng_q, spec.nq, spec.d, spec.sigma, spec.item_offset)
        q_item = -np.ones(spec.nq, np.int64)
    else:
        raise ValueError(spec.query_mode)
    return Workload(spec, np.ascontiguousarray(U), np.ascontiguousarray(P), np.ascontiguousarray(Qy), q_item, seed)


def random_instance(seed: int, n: int, m: int, d: int, dist: str = "gaussian"):
    """Small random instances for the oracle-equivalence sweeps (SPEC.md line 452 ranges).

    dist: "gaussian" (N(0,1)), "uniform" (U[-1,1]), "skewed" (gaussian direction, lognormal(0,1) norm)."""
    rng = np.random.default_rng(seed)
    if dist == "gaussian":
        U = rng.standard_normal((n, d))
        P = rng.standard_normal((m, d))
    elif dist == "uniform":
        U = rng.uniform(-1, 1, (n, d))
        P = rng.uniform(-1, 1, (m, d))
    elif dist == "skewed":
        U = vecs(rng, n, d, 1.0, 0.0)
        P = vecs(rng, m, d, 1.0, 0.0)
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(U, np.float32), np.ascontiguousarray(P, np.float32)


def table1():
    """PAPER.md Table 1 (lines 80-84): users u1..u4 and items p1..p5, 2-d, as fp32."""
    U = np.array([[3.1, 0.1], [2.5, 2.0], [1.5, 2.2], [1.8, 3.2]], dtype=np.float32)
    P = np.array([[2.8, 0.6], [2.5, 1.8], [3.2, 1.0], [1.4, 2.6], [0.5, 3.4]], dtype=np.float32)
    return U, P


def sha256_arrays(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
