"""DeviceRadixCache: the reference ``RadixCache`` API over the B200 device tree.

Drop-in for ``prefixsim.kvcache.RadixCache`` (kvcache.py:117-524): same
constructor (a ``CacheConfig``), same methods, same return values and the
same exceptions (``CapacityError``, ``ReleaseError``, ``ValueError``).  All
tree state lives in HBM behind libprism.so; this class only marshals
arguments.  ``admit_wave`` additionally runs the engine's whole admission
loop for one wave (engine.py:200-213) as one batched device call.

Use ``install(prefixsim)`` (paper_2605_08581_b200.integrate) to inject it
into the reference's serving loop; it then raises the reference's own
exception classes.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import PRISM_CAPACITY, PRISM_INVALID, PRISM_OK, PRISM_RELEASE, SEG_NONE, check
from .types import (
    KIND_CODE,
    KIND_OF_CODE,
    POLICY_CODE,
    Anchor,
    CacheConfig,
    CachePolicy,
    kind_of,
    policy_of,
)
from . import types as _types

# exception classes raised by the cache; integrate.install() may rebind them
ERRORS = {"capacity": _types.CapacityError, "release": _types.ReleaseError}


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _tokens(path: Sequence[int]) -> np.ndarray:
    arr = np.asarray(path, dtype=np.int64)
    if arr.size and (arr.min() < 0 or arr.max() >= 2**32):
        raise ValueError("tokens must be unsigned 32-bit (SURVEY.md Appendix C item 15)")
    return np.ascontiguousarray(arr, dtype=np.uint32)


def _seg_code(s) -> int:
    if s is None:
        return SEG_NONE
    s = int(s)
    if s < 0 or s >= 2**31 - 1:
        raise ValueError("segment ids must be non-negative int32")
    return s


def encode_anchors(anchors: Sequence[Anchor]):
    n = len(anchors)
    off = np.empty(n, dtype=np.int32)
    kind = np.empty(n, dtype=np.int8)
    seg = np.empty(n, dtype=np.int32)
    snap = np.zeros(3 * n, dtype=np.int32)
    for j, a in enumerate(anchors):
        off[j] = a.offset
        kind[j] = KIND_CODE[kind_of(a.kind)]
        seg[j] = _seg_code(a.segment_id)
        snap[3 * j : 3 * j + 3] = a.counter_snapshot
    return off, kind, seg, snap


class DeviceNode:
    """Handle of one device node: (slot, node_id) plus lazily read fields."""

    __slots__ = ("_cache", "slot", "node_id", "_rec")

    def __init__(self, cache: "DeviceRadixCache", slot: int, node_id: int, rec: dict | None = None):
        self._cache = cache
        self.slot = slot
        self.node_id = node_id
        self._rec = rec

    def _fields(self) -> dict:
        if self._rec is not None:
            return self._rec
        snap = self._cache._snapshot()
        i = self.slot
        if i >= len(snap["nid"]) or snap["nid"][i] != self.node_id:
            raise KeyError(f"node {self.node_id} is no longer resident")
        return {
            "kind": int(snap["kind"][i]),
            "seg": int(snap["seg"][i]),
            "ref": int(snap["ref"][i]),
            "last": int(snap["last"][i]),
            "hits": int(snap["hits"][i]),
            "eoff": int(snap["eoff"][i]),
            "elen": int(snap["elen"][i]),
            "ftok": int(snap["ftok"][i]),
        }

    @property
    def kind(self):
        return KIND_OF_CODE[self._fields()["kind"]]

    @property
    def segment_id(self):
        s = self._fields()["seg"]
        return None if s == SEG_NONE else s

    @property
    def ref_count(self) -> int:
        return self._fields()["ref"]

    @property
    def last_access(self) -> int:
        return self._fields()["last"]

    @property
    def access_count(self) -> int:
        return self._fields()["hits"]

    @property
    def edge_tokens(self) -> list[int]:
        f = self._fields()
        if "tokens" in f:
            return f["tokens"]
        return self._cache._arena(f["eoff"], f["elen"])

    def __eq__(self, other) -> bool:
        return isinstance(other, DeviceNode) and other.node_id == self.node_id

    def __hash__(self) -> int:
        return hash(self.node_id)

    def __lt__(self, other) -> bool:  # heap tuples in the engine never compare leaves
        return self.node_id < other.node_id

    def __repr__(self) -> str:
        return f"DeviceNode(slot={self.slot}, id={self.node_id})"


class DeviceRadixCache:
    """The reference ``RadixCache`` (kvcache.py:117-524) on the B200 device tree."""

    def __init__(self, config: CacheConfig, device: int = 0, initial_slots: int = 0,
                 initial_arena_tokens: int = 0, record_victims: bool = True):
        self.config = config
        self._policy = policy_of(config.policy)
        if config.capacity_tokens <= 0:
            raise ValueError("capacity_tokens must be > 0")
        if config.protect_budget < 0:
            raise ValueError("protect_budget must be >= 0")
        _lib.require_device()
        self._L = _lib.lib()
        self._h = self._L.prism_tree_create(
            config.capacity_tokens,
            POLICY_CODE[self._policy],
            config.protect_budget,
            initial_slots,
            initial_arena_tokens,
            device,
        )
        if not self._h:
            raise _lib.PrismError(_lib.last_error())
        self.device = device
        self._record = record_victims
        self._vlog_seen = 0
        self._victim_ids: list[int] = []
        self._last: tuple[int, int] | None = (0, 0)  # victim-log range of the last evict call
        self._snap_cache = None
        self._op = np.zeros(8, dtype=np.int64)

    @classmethod
    def attach(cls, handle, config: CacheConfig, record_victims: bool = True) -> "DeviceRadixCache":
        """A non-owning view of an existing device tree (e.g. a WaveEngine's)."""
        self = cls.__new__(cls)
        self.config = config
        self._policy = policy_of(config.policy)
        self._L = _lib.lib()
        self._h = handle
        self._owner = False
        self.device = None
        self._record = record_victims
        self._vlog_seen = 0
        self._victim_ids = []
        self._last = (0, 0)
        self._snap_cache = None
        self._op = np.zeros(8, dtype=np.int64)
        return self

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owner", True):
            self._L.prism_tree_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    # ------------------------------------------------------------ helpers
    def _dirty(self) -> None:
        self._snap_cache = None

    _VLOG_DRAIN = 1 << 19  # half the device victim ring (dart.cu): drain before it wraps

    def _after_op(self) -> None:
        self._L.prism_last_op(self._h, _ptr(self._op))
        if self._op[0]:
            self._last = (int(self._op[1]), int(self._op[2]))
            if self._record and int(self._op[2]) - self._vlog_seen > self._VLOG_DRAIN:
                self._log_victims()
        self._dirty()

    TUNABLES = {"list_min_tokens": 0, "list_slack_tokens": 1, "sel_min_candidates": 2, "use_coop": 3,
                "use_sample": 4, "prebuild": 5}

    def tune(self, **kw) -> None:
        """Eviction-list prefix sizing (semantics-free; tests force tiny prefixes)."""
        for k, v in kw.items():
            check(self._L.prism_tune(self._h, self.TUNABLES[k], int(v)))

    def stats(self) -> dict:
        out = np.zeros(16, dtype=np.int64)
        check(self._L.prism_stats(self._h, _ptr(out)))
        keys = [
            "resident", "clock", "next_id", "hw", "live_nodes", "arena_used", "hash_live",
            "hash_tomb", "victims", "evict_calls", "builds", "slot_cap", "arena_cap",
            "hash_cap", "fast_members", "slow_members",
        ]
        return dict(zip(keys, out.tolist()))

    def _victims(self, first: int, count: int) -> list[dict]:
        if count <= 0:
            return []
        ids = np.zeros(count, dtype=np.int64)
        kinds = np.zeros(count, dtype=np.int8)
        segs = np.zeros(count, dtype=np.int32)
        ftok = np.zeros(count, dtype=np.uint32)
        elen = np.zeros(count, dtype=np.int32)
        eoff = np.zeros(count, dtype=np.int64)
        check(self._L.prism_victims(self._h, first, count, _ptr(ids), _ptr(kinds), _ptr(segs),
                                    _ptr(ftok), _ptr(elen), _ptr(eoff)))
        return [
            {"id": int(ids[i]), "kind": int(kinds[i]), "seg": int(segs[i]), "ftok": int(ftok[i]),
             "elen": int(elen[i]), "eoff": int(eoff[i])}
            for i in range(count)
        ]

    def _arena(self, off: int, n: int) -> list[int]:
        buf = np.zeros(max(n, 1), dtype=np.uint32)
        check(self._L.prism_arena_read(self._h, off, n, _ptr(buf)))
        return buf[:n].astype(np.int64).tolist()

    def _snapshot(self) -> dict:
        if self._snap_cache is not None:
            return self._snap_cache
        hw = np.zeros(1, dtype=np.int64)
        cap = 0
        while True:
            arrs = {
                "nid": np.zeros(cap, np.int64), "par": np.zeros(cap, np.int32),
                "elen": np.zeros(cap, np.int32), "kind": np.zeros(cap, np.int8),
                "seg": np.zeros(cap, np.int32), "ref": np.zeros(cap, np.int32),
                "last": np.zeros(cap, np.int64), "hits": np.zeros(cap, np.int32),
                "prot": np.zeros(cap, np.int8), "hasanc": np.zeros(cap, np.int8),
                "ftok": np.zeros(cap, np.uint32), "akind": np.zeros(cap, np.int8),
                "aseg": np.zeros(cap, np.int32), "aoff": np.zeros(cap, np.int32),
                "snap": np.zeros(3 * cap, np.int32), "eoff": np.zeros(cap, np.int64),
            }
            order = ["nid", "par", "elen", "kind", "seg", "ref", "last", "hits", "prot", "hasanc",
                     "ftok", "akind", "aseg", "aoff", "snap", "eoff"]
            ptrs = [(_ptr(arrs[k]) if cap else None) for k in order]
            check(self._L.prism_snapshot(self._h, cap, _ptr(hw), *ptrs))
            if cap >= hw[0]:
                break
            cap = int(hw[0])
        self._snap_cache = arrs
        return arrs

    def _log_victims(self) -> None:
        if not self._record:
            return
        total = self.stats()["victims"]
        if total > self._vlog_seen:
            self._victim_ids.extend(v["id"] for v in self._victims(self._vlog_seen, total - self._vlog_seen))
            self._vlog_seen = total

    def victim_log(self) -> list[int]:
        """Node ids of every victim of every evict call so far, in order."""
        self._log_victims()
        return list(self._victim_ids)

    # ------------------------------------------------------------ state
    @property
    def resident_tokens(self) -> int:
        return int(self.stats()["resident"])

    @property
    def last_evicted(self) -> list[DeviceNode]:
        if self._last is None:
            raise RuntimeError("last_evicted is not tracked across admit_wave (one batched call covers many "
                               "evict calls); use victim_log()")
        first, end = self._last
        out = []
        for v in self._victims(first, end - first):
            rec = {"kind": v["kind"], "seg": v["seg"], "ref": 0, "last": -1, "hits": -1,
                   "eoff": v["eoff"], "elen": v["elen"], "ftok": v["ftok"]}
            node = DeviceNode(self, -1, v["id"], rec)
            out.append(node)
        return out

    @property
    def root(self) -> DeviceNode:
        return DeviceNode(self, 0, 0)

    # ------------------------------------------------------------ ops
    def match_prefix(self, token_path: Sequence[int]) -> tuple[int, list[DeviceNode]]:
        """kvcache.py:146-171"""
        p = _tokens(token_path)
        n = len(p)
        hit = np.zeros(1, dtype=np.int64)
        nv = np.zeros(1, dtype=np.int64)
        vs = np.zeros(max(n, 1), dtype=np.int32)
        vi = np.zeros(max(n, 1), dtype=np.int64)
        check(self._L.prism_match(self._h, _ptr(p), n, _ptr(hit), _ptr(vs), _ptr(vi), _ptr(nv)))
        self._dirty()
        return int(hit[0]), [DeviceNode(self, int(vs[i]), int(vi[i])) for i in range(int(nv[0]))]

    def insert_path(self, token_path: Sequence[int], anchors: Sequence[Anchor] = ()) -> DeviceNode:
        """kvcache.py:190-241 (with _reserve/evict, 243-273)"""
        offsets = [a.offset for a in anchors]
        if offsets != sorted(offsets):
            raise ValueError("anchor offsets must be sorted")
        if offsets and offsets[-1] > len(token_path):
            raise ValueError("anchor offset beyond path length")
        for a in anchors:
            if kind_of(a.kind) is _types.NodeKind.REUSABLE and a.segment_id is None:
                raise ValueError("reusable anchor requires segment_id")
        p = _tokens(token_path)
        off, kind, seg, snap = encode_anchors(anchors)
        slot = np.zeros(1, dtype=np.int32)
        lid = np.zeros(1, dtype=np.int64)
        rc = self._L.prism_insert(self._h, _ptr(p), len(p), len(off), _ptr(off), _ptr(kind), _ptr(seg),
                                  _ptr(snap), _ptr(slot), _ptr(lid))
        self._after_op()
        if rc == PRISM_CAPACITY:
            raise ERRORS["capacity"](_lib.last_error())
        check(rc)
        return DeviceNode(self, int(slot[0]), int(lid[0]))

    def release_path(self, leaf: DeviceNode) -> None:
        """kvcache.py:350-360"""
        s = np.array([leaf.slot], dtype=np.int32)
        i = np.array([leaf.node_id], dtype=np.int64)
        rc = self._L.prism_release(self._h, 1, _ptr(s), _ptr(i))
        self._dirty()
        if rc == PRISM_RELEASE:
            raise ERRORS["release"](f"node {leaf.node_id} has no active pin")
        check(rc)

    def evict(self, k_free: int) -> int:
        """kvcache.py:425-460"""
        if k_free < 0:
            raise ValueError("k_free must be >= 0")
        freed = np.zeros(1, dtype=np.int64)
        check(self._L.prism_evict(self._h, int(k_free), _ptr(freed)))
        self._after_op()
        return int(freed[0])

    def set_protection(self, dispatch_priorities: Mapping[int, float]) -> set[int]:
        """kvcache.py:364-383"""
        n = len(dispatch_priorities)
        segs = np.fromiter((_seg_code(s) for s in dispatch_priorities.keys()), dtype=np.int32, count=n)
        vals = np.fromiter(dispatch_priorities.values(), dtype=np.float64, count=n)
        out = np.zeros(max(self.config.protect_budget, 1), dtype=np.int64)
        nout = np.zeros(1, dtype=np.int64)
        check(self._L.prism_set_protection(self._h, n, _ptr(segs), _ptr(vals), _ptr(out), _ptr(nout)))
        self._dirty()
        return {int(x) for x in out[: nout[0]]}

    def note_active_segments(self, active_segments: Iterable[int]) -> None:
        """kvcache.py:385-393"""
        segs = np.fromiter((_seg_code(s) for s in active_segments), dtype=np.int32)
        check(self._L.prism_note_active(self._h, len(segs), _ptr(segs)))
        self._dirty()

    def admit_wave(self, paths: Sequence[Sequence[int]], anchors: Sequence[Sequence[Anchor]]):
        """One wave of engine.py:200-213 in a single device call.

        Returns (hits, leaves) for the admitted prefix of the members; a
        CapacityError in member j admits members [0, j) exactly like the
        reference loop's ``break``.
        """
        B = len(paths)
        lens = np.fromiter((len(p) for p in paths), dtype=np.int64, count=B)
        poff = np.zeros(B + 1, dtype=np.int64)
        np.cumsum(lens, out=poff[1:])
        tokens = _tokens([t for p in paths for t in p]) if poff[-1] else np.zeros(1, np.uint32)
        alens = np.fromiter((len(a) for a in anchors), dtype=np.int64, count=B)
        aoffs = np.zeros(B + 1, dtype=np.int64)
        np.cumsum(alens, out=aoffs[1:])
        flat = [a for al in anchors for a in al]
        off, kind, seg, snap = encode_anchors(flat)
        if not len(off):
            off, kind, seg, snap = (np.zeros(1, np.int32), np.zeros(1, np.int8), np.zeros(1, np.int32),
                                    np.zeros(3, np.int32))
        hits = np.zeros(max(B, 1), dtype=np.int64)
        slots = np.zeros(max(B, 1), dtype=np.int32)
        ids = np.zeros(max(B, 1), dtype=np.int64)
        nadm = np.zeros(1, dtype=np.int64)
        check(self._L.prism_admit_wave(self._h, B, _ptr(poff), _ptr(tokens), _ptr(aoffs), _ptr(off),
                                       _ptr(kind), _ptr(seg), _ptr(snap), _ptr(hits), _ptr(slots),
                                       _ptr(ids), _ptr(nadm)))
        self._dirty()
        self._last = None
        if self._record and self.stats()["victims"] - self._vlog_seen > self._VLOG_DRAIN:
            self._log_victims()
        k = int(nadm[0])
        return hits[:k].tolist(), [DeviceNode(self, int(slots[i]), int(ids[i])) for i in range(k)]

    def evict_key(self, node: DeviceNode) -> tuple:
        """kvcache.py:397-414, decoded from the device's packed key."""
        k = np.zeros(3, dtype=np.uint64)
        check(self._L.prism_evict_key(self._h, node.slot, _ptr(k)))
        v = (int(k[0]) << 128) | (int(k[1]) << 64) | int(k[2])
        nid = v & ((1 << 40) - 1)
        last = (v >> 40) & ((1 << 40) - 1)
        rest = v >> 80
        if self._policy is CachePolicy.DART:
            bits = rest & ((1 << 64) - 1)
            cls = rest >> 64
            b = bits ^ (1 << 63) if bits >> 63 else ~bits & ((1 << 64) - 1)
            pri = float(np.array([b], dtype=np.uint64).view(np.float64)[0])
            return (cls, pri if cls == 1 else 0.0, last, nid)
        if self._policy is CachePolicy.LRU:
            return (last, nid)
        return (rest, last, nid)

    # ------------------------------------------------------------ debug
    def _tree(self):
        s = self._snapshot()
        live = [i for i in range(len(s["nid"])) if s["nid"][i] >= 0 and (i == 0 or s["par"][i] >= 0)]
        children: dict[int, list[tuple[int, int]]] = {}
        for i in live:
            if i != 0:
                children.setdefault(int(s["par"][i]), []).append((int(s["ftok"][i]), i))
        return s, children

    def _dfs(self, children) -> list[int]:
        order, stack = [], [0]
        while stack:
            node = stack.pop()
            if node != 0:
                order.append(node)
            for _, c in sorted(children.get(node, []), reverse=True):
                stack.append(c)
        return order

    def debug_nodes(self) -> list[dict]:
        """kvcache.py:473-492"""
        s, children = self._tree()
        out = []
        for i in self._dfs(children):
            out.append(
                {
                    "node_id": int(s["nid"][i]),
                    "parent_id": int(s["nid"][s["par"][i]]),
                    "edge_len": int(s["elen"][i]),
                    "kind": KIND_OF_CODE[int(s["kind"][i])].value,
                    "segment_id": None if s["seg"][i] == SEG_NONE else int(s["seg"][i]),
                    "ref_count": int(s["ref"][i]),
                    "last_access": int(s["last"][i]),
                    "access_count": int(s["hits"][i]),
                    "protected": bool(s["prot"][i]),
                    "has_anchor": bool(s["hasanc"][i]),
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
        """kvcache.py:505-521"""
        s, children = self._tree()
        paths: list[list[int]] = []

        def walk(i: int, prefix: list[int]) -> None:
            cur = prefix + self._arena(int(s["eoff"][i]), int(s["elen"][i]))
            kids = sorted(children.get(i, []))
            if not kids:
                paths.append(cur)
                return
            for _, c in kids:
                walk(c, cur)

        for _, c in sorted(children.get(0, [])):
            walk(c, [])
        return paths

    def recompute_resident_tokens(self) -> int:
        s, children = self._tree()
        return int(sum(int(s["elen"][i]) for i in self._dfs(children)))
