"""Synthetic pending pools for the benchmark configurations (INPUT PREPARATION,
not product).  Each pool is a pending-request CSR of numpy arrays

    ids int64[P], arrival float64[P], sk_off int64[P+1], sk int32 (dense
    segment ids), reorderable uint8[P], suffix int32[P]

in the reference's request model (workload.py:77-90; token layout
workload.py:18-22, 136-154: system prefix, ``chunk`` tokens per segment,
a private suffix keyed by request id).  Deterministic per seed.

Workloads:
  mu1M -- 8 segments x 16 tokens after a 28-token system prefix, 16-token
          suffix; slot 0 uniform over 50, the others uniform over 2M.
  C3   -- agent / tool-output trace: catalog 2^20 segments, chunk 32,
          system prefix 1024, suffix 128, k = 40, reorderable = false.
          Slot 0 Zipf(1.1) over 1024 hot segments; slot d < 24 is
          child(slot d-1, r) with r a Zipf(1.1) rank over 8 children,
          child(p, r) = splitmix64(8p + r) mod 2^20 (deep shared chains);
          slots 24..39 uniform.  Segments are distinct within a request
          (a collision moves to the next id), as the reference generator's
          are (workload.py:183-199).
  C4   -- the reference RAG generator's shape (workload.py:167-202) at
          catalog 100,000 / 1,000 hot / chunk 128 / sys 28 / suffix 100 /
          k 5 / r_hot 0.7 / Zipf(1.1), vectorised (not draw-for-draw).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    z = (np.asarray(x).astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def zipf_ranks(rng: np.random.Generator, n: int, alpha: float, size) -> np.ndarray:
    """0-based ranks with P(r) proportional to (r+1)^-alpha."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
    cdf = np.cumsum(w / w.sum())
    return np.minimum(np.searchsorted(cdf, rng.random(size), side="right"), n - 1)


@dataclass(frozen=True)
class Spec:
    name: str
    nseg: int
    sys_len: int
    chunk: int
    k: int
    suffix: int
    reorderable: bool

    @property
    def path_len(self) -> int:
        return self.sys_len + self.k * self.chunk + self.suffix


MU1M = Spec("mu1M", 50 + 2_000_000, 28, 16, 8, 16, True)
C3 = Spec("C3", 1 << 20, 1024, 32, 40, 128, False)
C4 = Spec("C4", 100_000, 28, 128, 5, 100, True)
C5 = Spec("C5", 100_000, 28, 128, 5, 100, True)  # the C4 shape (bench: 10% KV budget + global demand)
SPECS = {"mu1m": MU1M, "c3": C3, "c4": C4, "c5": C5}


def _pool(ids: np.ndarray, sk: np.ndarray, spec: Spec) -> dict:
    n, k = sk.shape
    return {
        "ids": ids,
        "arrival": ids.astype(np.float64) * 1e-3,
        "sk_off": np.arange(n + 1, dtype=np.int64) * k,
        "sk": np.ascontiguousarray(sk, dtype=np.int32).reshape(-1),
        "reorderable": np.full(n, 1 if spec.reorderable else 0, dtype=np.uint8),
        "suffix": np.full(n, spec.suffix, dtype=np.int32),
    }


def mu1m_skeletons(n: int, rng: np.random.Generator) -> np.ndarray:
    sk = np.empty((n, MU1M.k), dtype=np.int64)
    sk[:, 0] = rng.integers(0, 50, size=n)
    sk[:, 1:] = 50 + rng.integers(0, 2_000_000, size=(n, MU1M.k - 1))
    return sk


def _distinct_rows(sk: np.ndarray, nseg: int, chain: np.ndarray | None = None) -> None:
    """Make segments distinct within each row (in place): a repeated id moves
    to the next free id; for chain columns the children are re-derived."""
    s = np.sort(sk, axis=1)
    bad = np.flatnonzero((s[:, 1:] == s[:, :-1]).any(axis=1))
    for i in bad.tolist():
        seen: set[int] = set()
        row = sk[i]
        for d in range(row.shape[0]):
            c = int(row[d])
            if chain is not None and 0 < d < chain.shape[1] + 1:
                c = int(splitmix64(np.uint64(8 * int(row[d - 1]) + int(chain[i, d - 1]))) % np.uint64(nseg))
            while c in seen:
                c = (c + 1) % nseg
            seen.add(c)
            row[d] = c


def c3_skeletons(n: int, rng: np.random.Generator) -> np.ndarray:
    NS, k, depth = C3.nseg, C3.k, 24
    sk = np.empty((n, k), dtype=np.int64)
    sk[:, 0] = zipf_ranks(rng, 1024, 1.1, n)
    ranks = zipf_ranks(rng, 8, 1.1, (n, depth - 1))
    for d in range(1, depth):
        sk[:, d] = (splitmix64(8 * sk[:, d - 1].astype(np.uint64) + ranks[:, d - 1].astype(np.uint64))
                    % np.uint64(NS)).astype(np.int64)
    sk[:, depth:] = rng.integers(0, NS, size=(n, k - depth))
    _distinct_rows(sk, NS, ranks)
    return sk


def c4_skeletons(n: int, rng: np.random.Generator, hot: int = 1000, r_hot: float = 0.7,
                 alpha: float = 1.1) -> np.ndarray:
    NS, k = C4.nseg, C4.k
    sk = np.empty((n, k), dtype=np.int64)
    is_hot = rng.random(n) < r_hot
    first_hot = zipf_ranks(rng, hot, alpha, n)
    first_cold = hot + rng.integers(0, NS - hot, size=n)
    sk[:, 0] = np.where(is_hot, first_hot, first_cold)
    rest = rng.integers(0, NS, size=(n, k - 1))
    # cold requests avoid the hot set (workload.py:194-199): shift into the cold range
    cold_rows = ~is_hot
    rest[cold_rows] = hot + rest[cold_rows] % (NS - hot)
    sk[:, 1:] = rest
    _distinct_rows(sk, NS)
    return sk


SKELETONS = {"mu1m": mu1m_skeletons, "c3": c3_skeletons, "c4": c4_skeletons, "c5": c4_skeletons}


def make_pool(workload: str, first_id: int, n: int, rng: np.random.Generator) -> dict:
    spec = SPECS[workload]
    sk = SKELETONS[workload](n, rng)
    return _pool(np.arange(first_id, first_id + n, dtype=np.int64), sk, spec)


def pool_bytes(pool: dict) -> int:
    return int(sum(v.nbytes for v in pool.values()))


def route(pool: dict, world: int) -> np.ndarray:
    """Shard of each request: splitmix64(skeleton[0]) mod world."""
    first = pool["sk"][pool["sk_off"][:-1]].astype(np.uint64)
    return (splitmix64(first) % np.uint64(world)).astype(np.int64)


def select(pool: dict, idx: np.ndarray) -> dict:
    """Sub-pool of the given request indices (order kept)."""
    idx = np.asarray(idx, dtype=np.int64)
    lens = np.diff(pool["sk_off"])[idx]
    off = np.zeros(len(idx) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    if len(idx) and np.all(lens == lens[0]):
        k = int(lens[0])
        sk = pool["sk"].reshape(-1, k)[idx].reshape(-1) if len(pool["sk"]) else pool["sk"]
    else:
        sk = np.concatenate([pool["sk"][pool["sk_off"][i]:pool["sk_off"][i + 1]] for i in idx.tolist()] or
                            [np.zeros(0, np.int32)])
    return {"ids": pool["ids"][idx], "arrival": pool["arrival"][idx], "sk_off": off,
            "sk": np.ascontiguousarray(sk, dtype=np.int32), "reorderable": pool["reorderable"][idx],
            "suffix": pool["suffix"][idx]}


class ShardStream:
    """This rank's sub-trace of one global request stream: requests are drawn
    globally (ids in draw order) and routed by segment hash; ``take(n)``
    returns the next n requests of this shard."""

    def __init__(self, workload: str, seed: int, world: int, rank: int, chunk: int = 1 << 15):
        self.workload, self.world, self.rank = workload, world, rank
        self.rng = np.random.default_rng(seed)
        self.next_id = 0
        self.chunk = chunk
        self.buf: dict | None = None

    def _refill(self) -> None:
        g = make_pool(self.workload, self.next_id, self.chunk, self.rng)
        self.next_id += self.chunk
        mine = g if self.world == 1 else select(g, np.flatnonzero(route(g, self.world) == self.rank))
        self.buf = mine if self.buf is None else _cat(self.buf, mine)

    def take(self, n: int) -> dict:
        while self.buf is None or len(self.buf["ids"]) < n:
            self._refill()
        out = select(self.buf, np.arange(n))
        self.buf = select(self.buf, np.arange(n, len(self.buf["ids"])))
        return out


def _cat(a: dict, b: dict) -> dict:
    return {"ids": np.concatenate([a["ids"], b["ids"]]), "arrival": np.concatenate([a["arrival"], b["arrival"]]),
            "sk_off": np.concatenate([a["sk_off"], a["sk_off"][-1] + b["sk_off"][1:]]),
            "sk": np.concatenate([a["sk"], b["sk"]]), "reorderable": np.concatenate([a["reorderable"],
                                                                                    b["reorderable"]]),
            "suffix": np.concatenate([a["suffix"], b["suffix"]])}


def serve_trace(workload: str, n: int, qps: float, seed: int):
    """A whole trace for the serving loop (paper_2605_08581_b200.serve): ``n``
    requests of ``workload``'s shape with Poisson arrivals at ``qps``
    (exponential gaps, workload.py:219-223), ids in arrival order."""
    from paper_2605_08581_b200.serve import TraceCSR

    spec = SPECS[workload]
    rng = np.random.default_rng(seed)
    arrival = np.cumsum(rng.exponential(1.0 / qps, size=n))
    sk = SKELETONS[workload](n, rng)
    k = sk.shape[1]
    return TraceCSR(np.arange(n, dtype=np.int64), arrival, np.arange(n + 1, dtype=np.int64) * k,
                    np.ascontiguousarray(sk, dtype=np.int32).reshape(-1),
                    np.full(n, 1 if spec.reorderable else 0, np.uint8), np.full(n, spec.suffix, np.int32),
                    spec.nseg, spec.chunk, spec.sys_len, tuple(range(1000)) if workload == "c4" else ())


def shard_trace(tr, world: int, rank: int):
    """This replica's sub-trace: splitmix64(skeleton[0]) mod world."""
    from paper_2605_08581_b200.serve import TraceCSR

    if world == 1:
        return tr
    first = tr.sk[tr.sk_off[:-1]].astype(np.uint64)
    idx = np.flatnonzero((splitmix64(first) % np.uint64(world)).astype(np.int64) == rank)
    k = np.diff(tr.sk_off)
    off = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(k[idx], out=off[1:])
    if len(idx) and np.all(k == k[0]):
        sk = tr.sk.reshape(-1, int(k[0]))[idx].reshape(-1)
    else:
        sk = np.concatenate([tr.sk[tr.sk_off[i]:tr.sk_off[i + 1]] for i in idx.tolist()] or [np.zeros(0, np.int32)])
    return TraceCSR(tr.ids[idx], tr.arrival[idx], off, np.ascontiguousarray(sk, np.int32), tr.reorderable[idx],
                    tr.suffix[idx], tr.num_segments, tr.chunk_tokens, tr.sys_prefix_tokens, tr.hot_set)


def prefix_trace(tr, n: int):
    from paper_2605_08581_b200.serve import TraceCSR

    n = min(n, tr.n)
    return TraceCSR(tr.ids[:n], tr.arrival[:n], tr.sk_off[:n + 1].copy(), tr.sk[:tr.sk_off[n]], tr.reorderable[:n],
                    tr.suffix[:n], tr.num_segments, tr.chunk_tokens, tr.sys_prefix_tokens, tr.hot_set)
