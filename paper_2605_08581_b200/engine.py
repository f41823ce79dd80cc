"""Serving loop that drives QAS + DART: the caller side of the hot path.

Mirrors ``prefixsim.engine.run_simulation`` (engine.py:141-266) and its
hint hand-off glue (engine.py:189-213, ``_build_anchors`` 269-292) so the
parity tests can replay the reference's own experiments without the
reference installed.  The wave cost model (engine.py:221-230) and metrics
(engine.py:295-318) are reproduced unchanged so derived TTFT is comparable
with the reference's.

Backends are injectable: ``cache_factory(CacheConfig)`` builds the radix
cache and ``schedule_fn(pending, active, SchedulerConfig, t)`` runs one QAS
round.  With ``admit="wave"`` the whole admission loop of a wave runs as one
batched ``cache.admit_wave`` call (device fused path) instead of per-member
``match_prefix``/``insert_path`` calls; results are identical.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Callable, Sequence

from .types import (
    Anchor,
    CacheConfig,
    CachePolicy,
    CapacityError,
    NodeKind,
    SchedulerConfig,
    count_segments,
    policy_of,
    serialize_tokens,
)


class SimulationError(RuntimeError):
    pass


@dataclass(frozen=True)
class SimConfig:
    """engine.py:35-48"""

    prefill_rate: float
    decode_rate: float
    cache: CacheConfig
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    output_tokens: int = 32
    decode_attenuation_enabled: bool = False

    def __post_init__(self) -> None:
        if self.prefill_rate <= 0 or self.decode_rate <= 0:
            raise ValueError("prefill_rate and decode_rate must be > 0")
        if self.output_tokens < 1:
            raise ValueError("output_tokens must be >= 1")


@dataclass
class RequestMetrics:
    """engine.py:51-80"""

    request_id: int
    arrival: float
    admit: float
    prefill_end: float
    first_token: float
    completion: float
    hit_tokens: int
    eff_tokens: int
    path_tokens: int
    reuse_hit_tokens: int
    sys_len: int
    reuse_len: int

    @property
    def ttft(self) -> float:
        return self.first_token - self.arrival


@dataclass
class WaveRecord:
    """engine.py:83-90"""

    wave_index: int
    members: list[int]
    launch_time: float
    duration: float
    uncached_tokens: int
    cached_tokens: int


@dataclass
class RunMetrics:
    """engine.py:93-106"""

    p50: float
    p90: float
    p95: float
    p99: float
    throughput: float
    hit_rate: float
    reuse_hit_rate: float
    mean_wave_size: float
    completed: int
    mean_extend_tokens: float
    mean_prompt_tokens: float
    makespan: float


@dataclass
class SimResult:
    run: RunMetrics
    requests: list[RequestMetrics]
    waves: list[WaveRecord]


def percentile(samples: Sequence[float], p: float) -> float:
    """Nearest-rank percentile (engine.py:116-124)."""
    if not samples:
        raise ValueError("percentile of empty sample set")
    if not 0 < p <= 100:
        raise ValueError("p must be in (0, 100]")
    ordered = sorted(samples)
    return ordered[math.ceil(p / 100 * len(ordered)) - 1]


def effective_prefill_rate(config: SimConfig, throughput_estimate: float) -> float:
    """engine.py:127-133"""
    if not config.decode_attenuation_enabled:
        return config.prefill_rate
    alpha = throughput_estimate * config.output_tokens / config.decode_rate
    alpha = min(max(alpha, 0.0), 0.95)
    return config.prefill_rate * (1.0 - alpha)


def build_anchors(request, aligned_skeleton: Sequence[int], snapshots: dict) -> list[Anchor]:
    """engine.py:269-292: SYSTEM@sys_len, REUSABLE@each segment end, PRIVATE@path_len."""
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


_MAX_WINDOWS = 50_000_000


def _default_cache_factory(cfg: CacheConfig):
    from .dart import DeviceRadixCache

    return DeviceRadixCache(cfg)


def _default_schedule(pending, active, cfg, t):
    from .qas import schedule_round

    return schedule_round(pending, active, cfg, t)


def run_simulation(
    trace,
    config: SimConfig,
    admit_probe: Callable | None = None,
    cache_factory: Callable | None = None,
    schedule_fn: Callable | None = None,
    admit: str = "call",
    cache_hook: Callable | None = None,
) -> SimResult:
    """Replay a trace (engine.py:141-266).  ``admit`` is "call" or "wave"."""
    capacity = config.cache.capacity_tokens
    for req in trace.requests:
        if req.path_len > capacity:
            raise SimulationError(
                f"request {req.id} path ({req.path_len} tokens) exceeds cache capacity ({capacity})"
            )
    cache = (cache_factory or _default_cache_factory)(config.cache)
    if cache_hook is not None:
        cache_hook(cache)
    schedule = schedule_fn or _default_schedule
    policy = policy_of(config.cache.policy)
    window = config.scheduler.window_s
    arrivals = sorted(trace.requests, key=lambda r: (r.arrival_time, r.id))
    next_arrival = 0
    pending: list = []
    active: dict[int, object] = {}
    completions: list = []
    metrics: dict[int, RequestMetrics] = {}
    waves: list[WaveRecord] = []
    completed = 0
    busy_until = 0.0
    total = len(trace.requests)
    k = 0
    while completed < total:
        k += 1
        if k > _MAX_WINDOWS:
            raise SimulationError("simulation failed to make progress")
        t = k * window
        while completions and completions[0][0] <= t + 1e-12:
            _, rid, leaf = heapq.heappop(completions)
            cache.release_path(leaf)
            del active[rid]
            completed += 1
        while next_arrival < total and arrivals[next_arrival].arrival_time <= t + 1e-12:
            pending.append(arrivals[next_arrival])
            next_arrival += 1
        if not pending or t + 1e-12 < busy_until:
            continue

        batch = schedule(pending, active.values(), config.scheduler, t)
        if not batch.members:
            continue
        if policy is CachePolicy.DART:
            cache.set_protection(batch.priorities)
        elif policy is CachePolicy.LRU_ACTIVE:
            counts = count_segments(list(active.values()) + batch.members)
            cache.note_active_segments(r for r, c in counts.items() if c > 0)

        admitted: list = []
        if admit == "wave":
            paths, anchors = [], []
            for req in batch.members:
                hint = batch.hints[req.id]
                paths.append(serialize_tokens(req, trace.catalog, hint.aligned_skeleton))
                anchors.append(build_anchors(req, hint.aligned_skeleton, hint.counter_snapshot))
            hits, leaves = cache.admit_wave(paths, anchors)
            for req, path, hit, leaf in zip(batch.members, paths, hits, leaves):
                admitted.append((req, hit, len(path) - hit, leaf))
        else:
            for req in batch.members:
                hint = batch.hints[req.id]
                path = serialize_tokens(req, trace.catalog, hint.aligned_skeleton)
                hit, _ = cache.match_prefix(path)
                if admit_probe is not None:
                    admit_probe(req, path, hit, cache)
                anchors = build_anchors(req, hint.aligned_skeleton, hint.counter_snapshot)
                try:
                    leaf = cache.insert_path(path, anchors)
                except CapacityError:
                    break
                admitted.append((req, hit, len(path) - hit, leaf))
        if not admitted:
            continue

        admitted_ids = {req.id for req, _, _, _ in admitted}
        pending = [r for r in pending if r.id not in admitted_ids]
        uncached = sum(eff for _, _, eff, _ in admitted)
        cached = sum(hit for _, hit, _, _ in admitted)
        throughput_estimate = completed / t if t > 0 else 0.0
        rate = effective_prefill_rate(config, throughput_estimate)
        duration = uncached / rate
        wave_size = len(admitted)
        prefill_end = t + duration
        first_token = prefill_end + wave_size / config.decode_rate
        completion = first_token + (config.output_tokens - 1) * wave_size / config.decode_rate
        busy_until = prefill_end
        waves.append(
            WaveRecord(
                wave_index=len(waves),
                members=[req.id for req, _, _, _ in admitted],
                launch_time=t,
                duration=duration,
                uncached_tokens=uncached,
                cached_tokens=cached,
            )
        )
        for req, hit, eff, leaf in admitted:
            metrics[req.id] = RequestMetrics(
                request_id=req.id,
                arrival=req.arrival_time,
                admit=t,
                prefill_end=prefill_end,
                first_token=first_token,
                completion=completion,
                hit_tokens=hit,
                eff_tokens=eff,
                path_tokens=req.path_len,
                reuse_hit_tokens=min(max(hit - req.sys_len, 0), req.reuse_len),
                sys_len=req.sys_len,
                reuse_len=req.reuse_len,
            )
            active[req.id] = req
            heapq.heappush(completions, (completion, req.id, leaf))
    per_request = [metrics[r.id] for r in trace.requests]
    return SimResult(run=_summarize(per_request, waves), requests=per_request, waves=waves)


def _summarize(per_request: list[RequestMetrics], waves: list[WaveRecord]) -> RunMetrics:
    """engine.py:295-318"""
    ttfts = [m.ttft for m in per_request]
    total_hit = sum(m.hit_tokens for m in per_request)
    total_len = sum(m.path_tokens for m in per_request)
    total_reuse_hit = sum(m.reuse_hit_tokens for m in per_request)
    total_reuse = sum(m.reuse_len for m in per_request)
    makespan = max((m.completion for m in per_request), default=0.0)
    n = len(per_request)
    return RunMetrics(
        p50=percentile(ttfts, 50),
        p90=percentile(ttfts, 90),
        p95=percentile(ttfts, 95),
        p99=percentile(ttfts, 99),
        throughput=n / makespan if makespan > 0 else 0.0,
        hit_rate=total_hit / total_len if total_len else 0.0,
        reuse_hit_rate=total_reuse_hit / total_reuse if total_reuse else 0.0,
        mean_wave_size=n / len(waves) if waves else 0.0,
        completed=n,
        mean_extend_tokens=(sum(w.uncached_tokens for w in waves) / len(waves) if waves else 0.0),
        mean_prompt_tokens=total_len / n if n else 0.0,
        makespan=makespan,
    )
