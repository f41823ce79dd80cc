"""Host-side mirror of the reference's data types for the QAS + DART path.

Pure Python, no device code.  Names, fields, defaults and validation follow
the reference one for one so that code written against ``prefixsim`` reads
the same against this package:

* ``CachePolicy``, ``NodeKind``, ``CacheError``/``CapacityError``/
  ``ReleaseError``, ``Anchor``, ``CacheConfig``  -- kvcache.py:19-76
* ``PriorityWeights``, ``SchedulerConfig``, ``SegmentCounters``, ``Bucket``,
  ``DispatchHint``, ``DispatchBatch``, ``export_anchor_offsets``,
  ``count_segments``                             -- scheduler.py:19-189
* ``Request``, ``SegmentCatalog``, ``Trace``, token layout constants and
  ``serialize_skeleton``/``serialize_tokens``     -- workload.py:18-164

The enums are ``str`` enums with the reference's values, so they compare
equal to the reference's own enum members (``NodeKind.PRIVATE ==
prefixsim.kvcache.NodeKind.PRIVATE``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Sequence

# ---------------------------------------------------------------- kvcache.py


class CachePolicy(str, Enum):
    """kvcache.py:19-23"""

    DART = "DART"
    LRU = "LRU"
    LRU_ACTIVE = "LRU_ACTIVE"
    LFU = "LFU"


class NodeKind(str, Enum):
    """kvcache.py:26-29"""

    SYSTEM = "system"
    REUSABLE = "reusable"
    PRIVATE = "private"


POLICY_CODE = {CachePolicy.DART: 0, CachePolicy.LRU: 1, CachePolicy.LRU_ACTIVE: 2, CachePolicy.LFU: 3}
KIND_CODE = {NodeKind.SYSTEM: 0, NodeKind.REUSABLE: 1, NodeKind.PRIVATE: 2}
KIND_OF_CODE = {0: NodeKind.SYSTEM, 1: NodeKind.REUSABLE, 2: NodeKind.PRIVATE}


def policy_of(p) -> CachePolicy:
    """Accept this package's or the reference's CachePolicy (or its value)."""
    return CachePolicy(getattr(p, "value", p))


def kind_of(k) -> NodeKind:
    """Accept this package's or the reference's NodeKind (or its value)."""
    return NodeKind(getattr(k, "value", k))


class CacheError(RuntimeError):
    """kvcache.py:32-33"""


class CapacityError(CacheError):
    """Path cannot be made resident even after maximal eviction (kvcache.py:36-37)."""


class ReleaseError(CacheError):
    """Release of a path that is not currently pinned (kvcache.py:40-41)."""


class SimulationError(RuntimeError):
    """The serving loop cannot make progress, or a path exceeds the capacity (engine.py:31-32)."""


class TraceFormatError(ValueError):
    """A trace file fails to parse or validate (workload.py:29-30)."""


@dataclass(frozen=True)
class Anchor:
    """Boundary to materialize during insert (kvcache.py:56-63)."""

    offset: int
    kind: NodeKind
    segment_id: int | None = None
    counter_snapshot: tuple[int, int, int] = (0, 0, 0)


@dataclass(frozen=True)
class CacheConfig:
    """kvcache.py:66-76"""

    capacity_tokens: int
    policy: CachePolicy = CachePolicy.DART
    protect_budget: int = 0

    def __post_init__(self) -> None:
        if self.capacity_tokens <= 0:
            raise ValueError("capacity_tokens must be > 0")
        if self.protect_budget < 0:
            raise ValueError("protect_budget must be >= 0")


# -------------------------------------------------------------- scheduler.py


@dataclass(frozen=True)
class PriorityWeights:
    """scheduler.py:19-23"""

    w_g: float = 1.0
    w_a: float = 1e6
    w_n: float = 1e5


@dataclass(frozen=True)
class SchedulerConfig:
    """scheduler.py:26-43"""

    window_s: float = 0.05
    dispatch_budget: int = 64
    cold_quota: int = 2
    front_width: int = 3
    signature_size: int = 1
    weights: PriorityWeights = field(default_factory=PriorityWeights)
    alpha_size: float = 1.0
    beta_util: float = 0.5

    def __post_init__(self) -> None:
        if self.cold_quota > self.dispatch_budget:
            raise ValueError("cold_quota must be <= dispatch_budget")
        if self.signature_size < 1:
            raise ValueError("signature_size must be >= 1")
        if self.front_width < self.signature_size:
            raise ValueError("front_width must be >= signature_size")


@dataclass
class SegmentCounters:
    """scheduler.py:46-50"""

    g: dict[int, int]
    a: dict[int, int]
    n: dict[int, int]


@dataclass
class Bucket:
    """scheduler.py:53-57"""

    signature: tuple[int, ...]
    members: list
    creation_order: int


@dataclass
class DispatchHint:
    """scheduler.py:60-66"""

    signature: tuple[int, ...]
    rank: int
    counter_snapshot: dict[int, tuple[int, int, int]]
    anchor_offsets: list[int]
    aligned_skeleton: list[int]


@dataclass
class DispatchBatch:
    """scheduler.py:69-80"""

    hot: list
    cold: list
    hints: dict[int, DispatchHint]
    priorities: dict[int, float]
    counters: SegmentCounters
    bucket_scores: dict[tuple[int, ...], float] = field(default_factory=dict)

    @property
    def members(self) -> list:
        return self.hot + self.cold


def count_segments(requests: Iterable) -> dict[int, int]:
    """Per-segment request counts, once per distinct segment (scheduler.py:83-89)."""
    counts: dict[int, int] = {}
    for req in requests:
        for r in set(req.skeleton):
            counts[r] = counts.get(r, 0) + 1
    return counts


def export_anchor_offsets(request) -> list[int]:
    """Offsets at end-of-system, each segment end, suffix end (scheduler.py:174-189)."""
    m = len(request.skeleton)
    chunk = request.reuse_len // m if m else 0
    offsets = [request.sys_len]
    for j in range(1, m + 1):
        offsets.append(request.sys_len + j * chunk)
    offsets.append(request.sys_len + request.reuse_len + request.suffix_len)
    out: list[int] = []
    for off in offsets:
        if off > 0 and (not out or off > out[-1]):
            out.append(off)
    return out


# --------------------------------------------------------------- workload.py

# Disjoint token-ID ranges (workload.py:18-22).
SEGMENT_TOKEN_BASE = 1_000_000
SUFFIX_TOKEN_BASE = 2_000_000_000


@dataclass(frozen=True)
class SegmentCatalog:
    """workload.py:33-50"""

    num_segments: int
    chunk_tokens: int
    hot_set: tuple[int, ...]
    sys_prefix_tokens: int = 0

    def __post_init__(self) -> None:
        if self.chunk_tokens < 1:
            raise ValueError("chunk_tokens must be >= 1")
        if self.sys_prefix_tokens < 0:
            raise ValueError("sys_prefix_tokens must be >= 0")
        hot = tuple(self.hot_set)
        if len(set(hot)) != len(hot):
            raise ValueError("hot_set IDs must be distinct")
        if any(h < 0 or h >= self.num_segments for h in hot):
            raise ValueError("hot_set IDs must be < num_segments")
        object.__setattr__(self, "hot_set", hot)


@dataclass
class Request:
    """workload.py:77-90 (``token_path`` may be empty: the path never reads it)."""

    id: int
    arrival_time: float
    skeleton: list[int]
    reorderable: bool
    token_path: list[int]
    sys_len: int
    reuse_len: int
    suffix_len: int

    @property
    def path_len(self) -> int:
        return self.sys_len + self.reuse_len + self.suffix_len


@dataclass
class Trace:
    """workload.py:93-97"""

    catalog: SegmentCatalog
    requests: list
    config: object | None = None


def serialize_skeleton(
    skeleton: Sequence[int], catalog, request_id: int, suffix_tokens: int
) -> list[int]:
    """Exact token path: sys prefix, segment chunks, private suffix (workload.py:136-154)."""
    chunk = catalog.chunk_tokens
    path = list(range(catalog.sys_prefix_tokens))
    for r in skeleton:
        base = SEGMENT_TOKEN_BASE + r * chunk
        path.extend(range(base, base + chunk))
    base = SUFFIX_TOKEN_BASE + request_id * suffix_tokens
    path.extend(range(base, base + suffix_tokens))
    return path


def serialize_tokens(request, catalog, skeleton: Sequence[int] | None = None) -> list[int]:
    """workload.py:157-164"""
    order = request.skeleton if skeleton is None else skeleton
    return serialize_skeleton(order, catalog, request.id, request.suffix_len)


# ----------------------------------------------------------------- engine.py


def build_anchors(request, aligned_skeleton: Sequence[int], snapshots: dict) -> list[Anchor]:
    """The hint hand-off glue, engine.py:269-292: SYSTEM@sys_len, REUSABLE@each segment end, PRIVATE@path_len."""
    anchors: list[Anchor] = []
    if request.sys_len > 0:
        anchors.append(Anchor(offset=request.sys_len, kind=NodeKind.SYSTEM))
    m = len(aligned_skeleton)
    chunk = request.reuse_len // m if m else 0
    depth = request.sys_len
    for seg in aligned_skeleton:
        depth += chunk
        anchors.append(
            Anchor(
                offset=depth,
                kind=NodeKind.REUSABLE,
                segment_id=seg,
                counter_snapshot=snapshots.get(seg, (0, 0, 0)),
            )
        )
    if request.suffix_len > 0:
        anchors.append(Anchor(offset=request.path_len, kind=NodeKind.PRIVATE))
    return anchors
