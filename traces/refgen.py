"""Reference-compatible trace generation and JSONL I/O (INPUT PREPARATION, not product).

``load_trace``/``save_trace`` read and write the reference's JSON-lines trace
format (workload.py:232-313).  ``generate_trace`` reproduces the reference's
generator (workload.py:100-229) draw for draw on the same numpy RNG stream,
so a given ``WorkloadConfig`` + seed yields the identical trace without the
reference installed; ``token_path`` is left empty because the scheduling-
memory path re-serialises from the aligned skeleton (engine.py:202).

``micro_paths`` builds the SURVEY.md section 8(d) "mu1M" micro-benchmark workload
(k segments of ``chunk`` tokens after a shared system prefix, private suffix).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from functools import lru_cache
from typing import IO

import numpy as np

from paper_2605_08581_b200.types import Request, SegmentCatalog, Trace


@dataclass(frozen=True)
class WorkloadConfig:
    """workload.py:53-74"""

    qps: float
    num_requests: int
    k: int
    r_hot: float
    zipf_alpha: float
    suffix_tokens: int = 100
    reorderable: bool = True
    seed: int = 0


@lru_cache(maxsize=128)
def _zipf_cdf(n: int, alpha: float) -> np.ndarray:
    ranks = np.arange(1, n + 1, dtype=np.float64)
    weights = ranks ** (-alpha)
    return np.cumsum(weights / weights.sum())


def _zipf_sample(rng: np.random.Generator, n: int, alpha: float) -> int:
    cdf = _zipf_cdf(n, float(alpha))
    return min(int(np.searchsorted(cdf, rng.random(), side="right")), n - 1)


def _sample_skeleton(rng, catalog: SegmentCatalog, config: WorkloadConfig) -> list[int]:
    """Same draw sequence as sample_request (workload.py:167-202)."""
    hot_set = catalog.hot_set
    n = catalog.num_segments
    if rng.random() < config.r_hot:
        first = hot_set[_zipf_sample(rng, len(hot_set), config.zipf_alpha)]
        skeleton = [first]
        seen = {first}
        while len(skeleton) < config.k:
            c = int(rng.integers(n))
            if c not in seen:
                seen.add(c)
                skeleton.append(c)
    else:
        hot = set(hot_set)
        skeleton = []
        seen: set[int] = set()
        while len(skeleton) < config.k:
            c = int(rng.integers(n))
            if c in hot or c in seen:
                continue
            seen.add(c)
            skeleton.append(c)
    return skeleton


def generate_trace(config: WorkloadConfig, catalog: SegmentCatalog) -> Trace:
    """Poisson arrivals + Zipf-hot skeletons (workload.py:216-229)."""
    if config.k > catalog.num_segments:
        raise ValueError("k exceeds catalog size")
    rng = np.random.default_rng(config.seed)
    gaps = rng.exponential(1.0 / config.qps, size=config.num_requests)
    arrivals = np.cumsum(gaps)
    reqs = []
    for i in range(config.num_requests):
        sk = _sample_skeleton(rng, catalog, config)
        reqs.append(
            Request(
                id=i,
                arrival_time=float(arrivals[i]),
                skeleton=sk,
                reorderable=config.reorderable,
                token_path=[],
                sys_len=catalog.sys_prefix_tokens,
                reuse_len=len(sk) * catalog.chunk_tokens,
                suffix_len=config.suffix_tokens,
            )
        )
    return Trace(catalog=catalog, requests=reqs, config=config)


def save_trace(trace: Trace, stream: IO[str]) -> None:
    """JSON lines: catalog header, then one request per line (workload.py:232-255)."""
    cat = trace.catalog
    header = {
        "catalog": {
            "num_segments": cat.num_segments,
            "chunk_tokens": cat.chunk_tokens,
            "hot_set": list(cat.hot_set),
            "sys_prefix_tokens": cat.sys_prefix_tokens,
        }
    }
    stream.write(json.dumps(header) + "\n")
    for req in trace.requests:
        rec = {
            "id": req.id,
            "arrival_time": req.arrival_time,
            "skeleton": req.skeleton,
            "suffix_tokens": req.suffix_len,
            "reorderable": req.reorderable,
        }
        stream.write(json.dumps(rec) + "\n")


def load_trace(stream: IO[str]) -> Trace:
    """Parse the JSON-lines trace format (workload.py:258-313); token_path left empty."""
    lines = iter(stream)
    header = json.loads(next(lines))
    c = header["catalog"]
    catalog = SegmentCatalog(
        num_segments=c["num_segments"],
        chunk_tokens=c["chunk_tokens"],
        hot_set=tuple(c["hot_set"]),
        sys_prefix_tokens=c["sys_prefix_tokens"],
    )
    reqs = []
    seen: set[int] = set()
    last = float("-inf")
    for line in lines:
        if not line.strip():
            continue
        rec = json.loads(line)
        rid = rec["id"]
        if rid in seen:
            raise ValueError(f"duplicate request id {rid}")
        seen.add(rid)
        arrival = float(rec["arrival_time"])
        if arrival < last:
            raise ValueError("arrival_time decreases")
        last = arrival
        sk = list(rec["skeleton"])
        if any(s < 0 or s >= catalog.num_segments for s in sk):
            raise ValueError("skeleton references unknown segment")
        reqs.append(
            Request(
                id=rid,
                arrival_time=arrival,
                skeleton=sk,
                reorderable=bool(rec["reorderable"]),
                token_path=[],
                sys_len=catalog.sys_prefix_tokens,
                reuse_len=len(sk) * catalog.chunk_tokens,
                suffix_len=int(rec["suffix_tokens"]),
            )
        )
    return Trace(catalog=catalog, requests=reqs, config=None)


# ------------------------------------------------------------------ micro


@dataclass(frozen=True)
class MicroSpec:
    """125K paths -> ~1M nodes, ~16M tokens."""

    paths: int = 125_000
    sys_len: int = 28
    k: int = 8
    chunk: int = 16
    suffix: int = 16
    slot0_choices: int = 50
    other_choices: int = 2_000_000
    seed: int = 0


def micro_skeletons(spec: MicroSpec, n: int, rng: np.random.Generator) -> np.ndarray:
    """[n, k] int64 skeletons: slot 0 uniform over slot0_choices, others uniform."""
    sk = np.empty((n, spec.k), dtype=np.int64)
    sk[:, 0] = rng.integers(0, spec.slot0_choices, size=n)
    if spec.k > 1:
        sk[:, 1:] = spec.slot0_choices + rng.integers(0, spec.other_choices, size=(n, spec.k - 1))
    return sk
