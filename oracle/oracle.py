"""ctypes front-end of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()``
and bench.py's CPU-baseline legs -- never by the product package.

``OracleRadixCache`` exposes the reference's ``RadixCache`` API
(kvcache.py:117-524) over the C restatement in dart_oracle.c;
``oracle_schedule_round`` exposes ``schedule_round`` (scheduler.py:192-273)
over qas_oracle.c.  Both are pinned to the reference by tests/golden/.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Iterable, Mapping, Sequence

import numpy as np

from paper_2605_08581_b200.qas_host import RoundOutputs, build_batch, marshal_round
from paper_2605_08581_b200.types import (
    KIND_CODE,
    KIND_OF_CODE,
    POLICY_CODE,
    Anchor,
    CacheConfig,
    CachePolicy,
    CapacityError,
    NodeKind,
    ReleaseError,
    kind_of,
    policy_of,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SEG_NONE = -(2**63)

_i64 = C.c_int64
_p = C.c_void_p


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        build()
    lib = C.CDLL(LIB_PATH)
    lib.ot_create.restype = _p
    lib.ot_create.argtypes = [_i64, C.c_int, _i64]
    lib.ot_destroy.argtypes = [_p]
    lib.ot_match.restype = _i64
    lib.ot_match.argtypes = [_p, _p, _i64, _p, _p]
    lib.ot_insert.restype = C.c_int
    lib.ot_insert.argtypes = [_p, _p, _i64, _i64, _p, _p, _p, _p, _p]
    lib.ot_release.restype = C.c_int
    lib.ot_release.argtypes = [_p, _i64]
    lib.ot_evict.restype = _i64
    lib.ot_evict.argtypes = [_p, _i64]
    lib.ot_set_protection.restype = _i64
    lib.ot_set_protection.argtypes = [_p, _i64, _p, _p, _p]
    lib.ot_note_active.argtypes = [_p, _i64, _p]
    for fn in ("ot_resident", "ot_clock", "ot_num_nodes"):
        getattr(lib, fn).restype = _i64
        getattr(lib, fn).argtypes = [_p]
    lib.ot_last_evicted.restype = _i64
    lib.ot_last_evicted.argtypes = [_p, _p, _i64]
    lib.ot_victim_log.restype = _i64
    lib.ot_victim_log.argtypes = [_p, _p, _i64]
    lib.ot_node_info.argtypes = [_p, _i64, _p]
    lib.ot_edge_tokens.restype = _i64
    lib.ot_edge_tokens.argtypes = [_p, _i64, _p, _i64]
    lib.ot_evict_key.argtypes = [_p, _i64, _p, _p]
    lib.ot_dump.restype = _i64
    lib.ot_dump.argtypes = [_p, _p, _i64]
    lib.oq_round.restype = C.c_int
    lib.oq_round.argtypes = [_i64, _p, _p, _p, _p, _p, _i64, _p, _p, C.c_int32, _p] + [_p] * 16
    return lib


_LIB: C.CDLL | None = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _tokens(path: Sequence[int]) -> np.ndarray:
    arr = np.asarray(path, dtype=np.int64)
    if arr.size and (arr.min() < 0 or arr.max() >= 2**32):
        raise ValueError("tokens must fit in uint32")
    return arr.astype(np.uint32)


def encode_anchors(anchors: Sequence[Anchor]):
    n = len(anchors)
    off = np.empty(n, dtype=np.int64)
    kind = np.empty(n, dtype=np.int8)
    seg = np.empty(n, dtype=np.int64)
    snap = np.zeros(3 * n, dtype=np.int64)
    for j, a in enumerate(anchors):
        off[j] = a.offset
        kind[j] = KIND_CODE[kind_of(a.kind)]
        seg[j] = SEG_NONE if a.segment_id is None else a.segment_id
        snap[3 * j : 3 * j + 3] = a.counter_snapshot
    return off, kind, seg, snap


class OracleNode:
    """Read-only view of one oracle node (the fields tests read from RadixNode)."""

    __slots__ = ("_cache", "node_id")

    def __init__(self, cache: "OracleRadixCache", node_id: int):
        self._cache = cache
        self.node_id = node_id

    def _info(self) -> np.ndarray:
        out = np.zeros(17, dtype=np.int64)
        lib().ot_node_info(self._cache._h, self.node_id, _ptr(out))
        return out

    @property
    def kind(self) -> NodeKind:
        return KIND_OF_CODE[int(self._info()[2])]

    @property
    def segment_id(self) -> int | None:
        s = int(self._info()[3])
        return None if s == SEG_NONE else s

    @property
    def ref_count(self) -> int:
        return int(self._info()[4])

    @property
    def last_access(self) -> int:
        return int(self._info()[5])

    @property
    def access_count(self) -> int:
        return int(self._info()[6])

    @property
    def edge_tokens(self) -> list[int]:
        n = lib().ot_edge_tokens(self._cache._h, self.node_id, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.uint32)
        lib().ot_edge_tokens(self._cache._h, self.node_id, _ptr(buf), n)
        return buf[:n].astype(np.int64).tolist()

    def __eq__(self, other) -> bool:
        return isinstance(other, OracleNode) and other.node_id == self.node_id

    def __hash__(self) -> int:
        return hash(self.node_id)

    def __repr__(self) -> str:
        return f"OracleNode(id={self.node_id})"


class OracleRadixCache:
    """The reference RadixCache API (kvcache.py:117-524) over dart_oracle.c."""

    def __init__(self, config: CacheConfig):
        self.config = config
        self._policy = policy_of(config.policy)
        self._h = lib().ot_create(
            config.capacity_tokens, POLICY_CODE[self._policy], config.protect_budget
        )
        if not self._h:
            raise ValueError("invalid CacheConfig")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ot_destroy(h)
            self._h = None

    # --------------------------------------------------------------- state
    @property
    def resident_tokens(self) -> int:
        return int(lib().ot_resident(self._h))

    @property
    def clock(self) -> int:
        return int(lib().ot_clock(self._h))

    @property
    def last_evicted(self) -> list[OracleNode]:
        n = lib().ot_last_evicted(self._h, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.int64)
        lib().ot_last_evicted(self._h, _ptr(buf), n)
        return [OracleNode(self, int(i)) for i in buf[:n]]

    def victim_log(self) -> list[int]:
        """Node ids of every victim of every evict call so far, in order."""
        n = lib().ot_victim_log(self._h, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.int64)
        lib().ot_victim_log(self._h, _ptr(buf), n)
        return buf[:n].tolist()

    @property
    def root(self) -> OracleNode:
        return OracleNode(self, 0)

    # ----------------------------------------------------------------- ops
    def match_prefix(self, token_path: Sequence[int]) -> tuple[int, list[OracleNode]]:
        p = _tokens(token_path)
        vis = np.zeros(max(len(p), 1), dtype=np.int64)
        nv = np.zeros(1, dtype=np.int64)
        hit = lib().ot_match(self._h, _ptr(p), len(p), _ptr(vis), _ptr(nv))
        return int(hit), [OracleNode(self, int(i)) for i in vis[: nv[0]]]

    def insert_path(self, token_path: Sequence[int], anchors: Sequence[Anchor] = ()) -> OracleNode:
        p = _tokens(token_path)
        off, kind, seg, snap = encode_anchors(anchors)
        leaf = np.zeros(1, dtype=np.int64)
        rc = lib().ot_insert(
            self._h, _ptr(p), len(p), len(off), _ptr(off), _ptr(kind), _ptr(seg), _ptr(snap), _ptr(leaf)
        )
        if rc == 3:
            raise ValueError("invalid anchors (unsorted, beyond path, or reusable without segment)")
        if rc == 1:
            raise CapacityError("path cannot fit even after maximal eviction")
        return OracleNode(self, int(leaf[0]))

    def release_path(self, leaf: OracleNode) -> None:
        rc = lib().ot_release(self._h, leaf.node_id)
        if rc != 0:
            raise ReleaseError(f"node {leaf.node_id} has no active pin")

    def evict(self, k_free: int) -> int:
        if k_free < 0:
            raise ValueError("k_free must be >= 0")
        return int(lib().ot_evict(self._h, k_free))

    def set_protection(self, dispatch_priorities: Mapping[int, float]) -> set[int]:
        segs = np.fromiter(dispatch_priorities.keys(), dtype=np.int64, count=len(dispatch_priorities))
        vals = np.fromiter(dispatch_priorities.values(), dtype=np.float64, count=len(dispatch_priorities))
        out = np.zeros(max(self.config.protect_budget, 1), dtype=np.int64)
        n = lib().ot_set_protection(self._h, len(segs), _ptr(segs), _ptr(vals), _ptr(out))
        return {int(i) for i in out[:n]}

    def note_active_segments(self, active_segments: Iterable[int]) -> None:
        segs = np.fromiter(active_segments, dtype=np.int64)
        lib().ot_note_active(self._h, len(segs), _ptr(segs))

    def evict_key(self, node: OracleNode) -> tuple:
        ints = np.zeros(3, dtype=np.int64)
        pri = np.zeros(1, dtype=np.float64)
        lib().ot_evict_key(self._h, node.node_id, _ptr(ints), _ptr(pri))
        a, b, c = (int(x) for x in ints)
        if self._policy is CachePolicy.DART:
            return (a, float(pri[0]), b, c)
        if self._policy is CachePolicy.LRU:
            return (a, b)
        return (a, b, c)

    # --------------------------------------------------------------- debug
    def _records(self) -> dict[int, np.ndarray]:
        n = lib().ot_num_nodes(self._h)
        recs = {}
        buf = np.zeros(17, dtype=np.int64)
        for i in range(n):
            lib().ot_node_info(self._h, i, _ptr(buf))
            if i == 0 or buf[9]:
                recs[i] = buf.copy()
        return recs

    def _dfs(self, recs: dict[int, np.ndarray]) -> list[int]:
        children: dict[int, list[tuple[int, int]]] = {}
        for i, r in recs.items():
            if i != 0:
                children.setdefault(int(r[0]), []).append((int(r[10]), i))
        order: list[int] = []
        stack = [0]
        while stack:
            node = stack.pop()
            if node != 0:
                order.append(node)
            for _, c in sorted(children.get(node, []), reverse=True):
                stack.append(c)
        return order

    def debug_nodes(self) -> list[dict]:
        """kvcache.py:473-492 (same dict keys and DFS order)."""
        recs = self._records()
        out = []
        for i in self._dfs(recs):
            r = recs[i]
            out.append(
                {
                    "node_id": i,
                    "parent_id": int(r[0]),
                    "edge_len": int(r[1]),
                    "kind": KIND_OF_CODE[int(r[2])].value,
                    "segment_id": None if r[3] == SEG_NONE else int(r[3]),
                    "ref_count": int(r[4]),
                    "last_access": int(r[5]),
                    "access_count": int(r[6]),
                    "protected": bool(r[7]),
                    "has_anchor": bool(r[8]),
                }
            )
        return out

    def debug_dump(self) -> str:
        return "\n".join(
            f"{r['node_id']} parent={r['parent_id']} len={r['edge_len']} "
            f"kind={r['kind']} seg={r['segment_id']} ref={r['ref_count']} "
            f"last={r['last_access']} hits={r['access_count']} "
            f"prot={int(r['protected'])}"
            for r in self.debug_nodes()
        )

    def resident_full_paths(self) -> list[list[int]]:
        recs = self._records()
        children: dict[int, list[tuple[int, int]]] = {}
        for i, r in recs.items():
            if i != 0:
                children.setdefault(int(r[0]), []).append((int(r[10]), i))
        paths: list[list[int]] = []

        def walk(node: int, prefix: list[int]) -> None:
            cur = prefix + OracleNode(self, node).edge_tokens
            kids = sorted(children.get(node, []))
            if not kids:
                paths.append(cur)
                return
            for _, c in kids:
                walk(c, cur)

        for _, c in sorted(children.get(0, [])):
            walk(c, [])
        return paths

    def recompute_resident_tokens(self) -> int:
        recs = self._records()
        return int(sum(int(r[1]) for i, r in recs.items() if i != 0))


def oracle_round_arrays(m, config):
    """Run qas_oracle.c on a MarshaledRound; returns RoundOutputs."""
    P = len(m.pending)
    kappa = config.signature_size
    nseg = m.nseg
    w = config.weights

    class _Cfg(C.Structure):
        _fields_ = [
            ("dispatch_budget", _i64),
            ("cold_quota", _i64),
            ("front_width", _i64),
            ("signature_size", _i64),
            ("w_g", C.c_double),
            ("w_a", C.c_double),
            ("w_n", C.c_double),
            ("alpha_size", C.c_double),
            ("beta_util", C.c_double),
        ]

    cfg = _Cfg(
        config.dispatch_budget,
        config.cold_quota,
        config.front_width,
        config.signature_size,
        w.w_g,
        w.w_a,
        w.w_n,
        config.alpha_size,
        config.beta_util,
    )
    n1 = max(P, 1)
    hot = np.zeros(n1, dtype=np.int64)
    cold = np.zeros(n1, dtype=np.int64)
    nhot = np.zeros(1, dtype=np.int64)
    ncold = np.zeros(1, dtype=np.int64)
    aligned = np.zeros(max(len(m.sk), 1), dtype=np.int32)
    sig = np.zeros(n1 * kappa, dtype=np.int32)
    siglen = np.zeros(n1, dtype=np.int32)
    rank = np.zeros(n1, dtype=np.int64)
    bucket = np.zeros(n1, dtype=np.int64)
    bscore = np.zeros(n1, dtype=np.float64)
    nb = np.zeros(1, dtype=np.int64)
    s1 = max(nseg, 1)
    g = np.zeros(s1, dtype=np.int32)
    a = np.zeros(s1, dtype=np.int32)
    nd = np.zeros(s1, dtype=np.int32)
    prio = np.zeros(s1, dtype=np.float64)
    dom = np.zeros(s1, dtype=np.uint8)
    sk = m.sk if len(m.sk) else np.zeros(1, dtype=np.int32)
    ask = m.act_sk if len(m.act_sk) else np.zeros(1, dtype=np.int32)
    rc = lib().oq_round(
        P, _ptr(m.ids) if P else None, _ptr(m.arrival) if P else None, _ptr(m.sk_off), _ptr(sk),
        _ptr(m.reorderable) if P else None, len(m.act_off) - 1, _ptr(m.act_off), _ptr(ask), nseg,
        C.addressof(cfg), _ptr(hot), _ptr(nhot), _ptr(cold), _ptr(ncold), _ptr(aligned), _ptr(sig),
        _ptr(siglen), _ptr(rank), _ptr(bucket), _ptr(bscore), _ptr(nb), _ptr(g), _ptr(a), _ptr(nd),
        _ptr(prio), _ptr(dom),
    )
    if rc != 0:
        raise ValueError("invalid SchedulerConfig")
    return RoundOutputs(
        hot=hot[: nhot[0]],
        cold=cold[: ncold[0]],
        aligned=aligned[: len(m.sk)],
        sig=sig[: P * kappa].reshape(P, kappa),
        siglen=siglen[:P],
        rank=rank[:P],
        bucket=bucket[:P],
        bscore=bscore[: nb[0]],
        g=g[:nseg],
        a=a[:nseg],
        nd=nd[:nseg],
        prio=prio[:nseg],
        dom=dom[:nseg],
    )


def oracle_schedule_round(pending, active_set, config, now: float = 0.0):
    """schedule_round (scheduler.py:192-273) over qas_oracle.c."""
    m = marshal_round(pending, active_set)
    return build_batch(m, oracle_round_arrays(m, config))
