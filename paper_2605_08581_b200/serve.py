"""The serving loop on the device: ``run_simulation`` (engine.py:141-266) with
the trace, pending queue, in-flight set, admission log and per-request metrics
resident in HBM (csrc/serve.cu), plus native trace ingestion (csrc/trace_io.cu,
workload.py:258-313).

``TraceCSR`` is the skeleton CSR the device consumes: ``from_trace`` converts a
reference ``Trace`` (catalog + requests), ``load_jsonl`` reads a ``save_trace``
file natively (multi-threaded; no Python object per request).
``DeviceServingLoop(config, trace).run()`` replays it; ``run_simulation`` is the
one-call form.  ``config`` is the reference's ``SimConfig`` (or any object with
its fields: prefill_rate, decode_rate, cache, scheduler, output_tokens,
decode_attenuation_enabled).  Results are arrays in trace order
(``ServeResult``), with the reference's RunMetrics summary (engine.py:295-318).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check
from .qas import _cfg
from .types import POLICY_CODE, SimulationError, TraceFormatError, policy_of


@dataclass
class TraceCSR:
    """A trace as arrays: requests in (arrival_time, id) order (engine.py:158)."""

    ids: np.ndarray  # int64 [n]
    arrival: np.ndarray  # float64 [n]
    sk_off: np.ndarray  # int64 [n+1]
    sk: np.ndarray  # int32 (segment ids)
    reorderable: np.ndarray  # uint8 [n]
    suffix: np.ndarray  # int32 [n]
    num_segments: int
    chunk_tokens: int
    sys_prefix_tokens: int
    hot_set: tuple = field(default_factory=tuple)

    @property
    def n(self) -> int:
        return int(self.ids.shape[0])

    def path_len(self) -> np.ndarray:
        k = np.diff(self.sk_off)
        return self.sys_prefix_tokens + k * self.chunk_tokens + self.suffix.astype(np.int64)

    def sorted(self) -> "TraceCSR":
        """The same trace in (arrival_time, id) order."""
        order = np.lexsort((self.ids, self.arrival))
        if np.all(order == np.arange(self.n)):
            return self
        k = np.diff(self.sk_off)
        off = np.zeros(self.n + 1, np.int64)
        np.cumsum(k[order], out=off[1:])
        sk = np.concatenate([self.sk[self.sk_off[i]:self.sk_off[i + 1]] for i in order]) if self.n else self.sk
        return TraceCSR(self.ids[order], self.arrival[order], off, sk.astype(np.int32), self.reorderable[order],
                        self.suffix[order], self.num_segments, self.chunk_tokens, self.sys_prefix_tokens,
                        self.hot_set)

    @staticmethod
    def from_trace(trace) -> "TraceCSR":
        """From a reference ``Trace`` (workload.py:93-97).  The device serializes
        paths from the skeleton (workload.py:136-164), so every request must have
        the catalog's layout: sys_len = sys_prefix_tokens, reuse_len =
        len(skeleton) * chunk_tokens (what generate_trace / load_trace produce)."""
        cat = trace.catalog
        reqs = trace.requests
        for r in reqs:
            if r.sys_len != cat.sys_prefix_tokens or r.reuse_len != len(r.skeleton) * cat.chunk_tokens:
                raise ValueError(f"request {r.id}: sys_len / reuse_len do not follow the catalog layout")
        off = np.zeros(len(reqs) + 1, np.int64)
        np.cumsum([len(r.skeleton) for r in reqs], out=off[1:])
        return TraceCSR(np.array([r.id for r in reqs], np.int64), np.array([r.arrival_time for r in reqs], np.float64),
                        off, np.array([s for r in reqs for s in r.skeleton], np.int32),
                        np.array([1 if r.reorderable else 0 for r in reqs], np.uint8),
                        np.array([r.suffix_len for r in reqs], np.int32), cat.num_segments, cat.chunk_tokens,
                        cat.sys_prefix_tokens, tuple(cat.hot_set))

    @staticmethod
    def load_jsonl(path: str, threads: int = 0) -> "TraceCSR":
        """workload.load_trace natively (csrc/trace_io.cu); raises TraceFormatError."""
        L = _lib.lib()
        h = L.prism_trace_load_jsonl(str(path).encode(), int(threads))
        if not h:
            msg = _lib.last_error()
            if msg.startswith("TraceFormatError: "):
                raise TraceFormatError(msg[len("TraceFormatError: "):])
            raise OSError(msg)
        try:
            info = np.zeros(6, np.int64)
            check(L.prism_trace_info(h, info.ctypes.data))
            n, nsk, nseg, chunk, sys_len, nhot = (int(x) for x in info)
            ids, arr = np.empty(n, np.int64), np.empty(n, np.float64)
            off, sk = np.empty(n + 1, np.int64), np.empty(nsk, np.int32)
            reo, sfx, hot = np.empty(n, np.uint8), np.empty(n, np.int32), np.empty(nhot, np.int64)
            check(L.prism_trace_copy(h, ids.ctypes.data, arr.ctypes.data, off.ctypes.data, sk.ctypes.data,
                                     reo.ctypes.data, sfx.ctypes.data, hot.ctypes.data))
        finally:
            L.prism_trace_free(h)
        return TraceCSR(ids, arr, off, sk, reo, sfx, nseg, chunk, sys_len, tuple(int(x) for x in hot))


def percentile(samples: np.ndarray, p: float) -> float:
    """Nearest rank: the element at 1-based index ceil(p/100 * n) (engine.py:113-122)."""
    if samples.size == 0:
        raise ValueError("percentile of empty sample set")
    if not 0 < p <= 100:
        raise ValueError("p must be in (0, 100]")
    return float(np.sort(samples)[math.ceil(p / 100 * samples.size) - 1])


@dataclass
class ServeResult:
    """Per-request metrics in trace order and per-wave records."""

    trace: TraceCSR
    admit: np.ndarray
    prefill_end: np.ndarray
    first_token: np.ndarray
    completion: np.ndarray
    hit_tokens: np.ndarray
    eff_tokens: np.ndarray
    wave_launch: np.ndarray
    wave_duration: np.ndarray
    wave_uncached: np.ndarray
    wave_cached: np.ndarray
    wave_off: np.ndarray  # [W+1] into wave_members
    wave_members: np.ndarray  # trace indices, admission order
    windows: int = 0

    @property
    def ttft(self) -> np.ndarray:  # RequestMetrics.ttft (engine.py:67-69)
        return self.first_token - self.trace.arrival

    def admission(self) -> list[list[int]]:
        """[w.members for w in result.waves] -- request ids per wave."""
        ids = self.trace.ids[self.wave_members]
        return [ids[self.wave_off[w]:self.wave_off[w + 1]].tolist() for w in range(len(self.wave_launch))]

    def summary(self) -> dict:
        """RunMetrics (engine.py:295-318)."""
        tr = self.trace
        ttft = self.ttft
        n = tr.n
        plen = tr.path_len()
        reuse_len = np.diff(tr.sk_off) * tr.chunk_tokens
        reuse_hit = np.minimum(np.maximum(self.hit_tokens - tr.sys_prefix_tokens, 0), reuse_len)
        makespan = float(self.completion.max()) if n else 0.0
        W = len(self.wave_launch)
        return {
            "p50": percentile(ttft, 50), "p90": percentile(ttft, 90), "p95": percentile(ttft, 95),
            "p99": percentile(ttft, 99),
            "throughput": n / makespan if makespan > 0 else 0.0,
            "hit_rate": int(self.hit_tokens.sum()) / int(plen.sum()) if plen.sum() else 0.0,
            "reuse_hit_rate": int(reuse_hit.sum()) / int(reuse_len.sum()) if reuse_len.sum() else 0.0,
            "mean_wave_size": n / W if W else 0.0,
            "completed": n,
            "mean_extend_tokens": int(self.wave_uncached.sum()) / W if W else 0.0,
            "mean_prompt_tokens": int(plen.sum()) / n if n else 0.0,
            "makespan": makespan,
        }


class DeviceServingLoop:
    """One replica's serving loop over a trace (engine.py:141-266) on the device."""

    def __init__(self, config, trace: TraceCSR, device: int = 0, initial_slots: int = 0,
                 initial_arena_tokens: int = 0):
        _lib.require_device()
        self.L = _lib.lib()
        self.config = config
        self.trace = trace = trace.sorted()
        cache, sched = config.cache, config.scheduler
        # sized up front (no growth / compaction mid-run): slots <= resident tokens, arena 32x the capacity
        initial_slots = initial_slots or max(1 << 12, min(cache.capacity_tokens + 2, 1 << 22))
        initial_arena_tokens = initial_arena_tokens or max(1 << 20, 32 * cache.capacity_tokens)
        self.t = self.L.prism_tree_create(cache.capacity_tokens, POLICY_CODE[policy_of(cache.policy)],
                                          cache.protect_budget, initial_slots, initial_arena_tokens, device)
        if not self.t:
            raise _lib.PrismError(_lib.last_error())
        self.q = self.L.prism_qas_create(device)
        if not self.q:
            raise _lib.PrismError(_lib.last_error())
        self._cfg = _cfg(sched)
        self._keep = [np.ascontiguousarray(a) for a in (trace.ids, trace.arrival, trace.sk_off, trace.sk,
                                                         trace.reorderable, trace.suffix)]
        ids, arr, off, sk, reo, sfx = self._keep
        self.s = self.L.prism_serve_create(
            self.t, self.q, trace.n, ids.ctypes.data, arr.ctypes.data, off.ctypes.data, sk.ctypes.data,
            reo.ctypes.data, sfx.ctypes.data, trace.num_segments, trace.sys_prefix_tokens, trace.chunk_tokens,
            cache.capacity_tokens, C.addressof(self._cfg), float(sched.window_s), float(config.prefill_rate),
            float(config.decode_rate), int(config.output_tokens), 1 if config.decode_attenuation_enabled else 0)
        if not self.s:
            msg = _lib.last_error()
            self.close()
            if "exceeds cache capacity" in msg:
                raise SimulationError(msg)
            raise ValueError(msg)

    def close(self) -> None:
        if getattr(self, "s", None):
            self.L.prism_serve_destroy(self.s)
            self.s = None
        if getattr(self, "q", None):
            self.L.prism_qas_destroy(self.q)
            self.q = None
        if getattr(self, "t", None):
            self.L.prism_tree_destroy(self.t)
            self.t = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    def run(self, max_waves: int = 0) -> bool:
        """Advance by up to max_waves waves (0: to the end); True when finished."""
        ran, fin = C.c_int64(0), C.c_int32(0)
        check(self.L.prism_serve_run(self.s, int(max_waves), C.byref(ran), C.byref(fin)))
        return bool(fin.value)

    def counts(self) -> dict:
        out = np.zeros(5, np.int64)
        check(self.L.prism_serve_counts(self.s, out.ctypes.data))
        return dict(zip(("waves", "admitted", "windows", "completed", "pending"), out.tolist()))

    def result(self) -> ServeResult:
        n = self.trace.n
        c = self.counts()
        adm, pe, ft, comp = (np.empty(n, np.float64) for _ in range(4))
        hit, eff = np.empty(n, np.int64), np.empty(n, np.int64)
        check(self.L.prism_serve_requests(self.s, adm.ctypes.data, pe.ctypes.data, ft.ctypes.data, comp.ctypes.data,
                                          hit.ctypes.data, eff.ctypes.data))
        W = c["waves"]
        wl, wd = np.empty(W, np.float64), np.empty(W, np.float64)
        wu, wc, wo = np.empty(W, np.int64), np.empty(W, np.int64), np.empty(W + 1, np.int64)
        wm = np.empty(c["admitted"], np.int32)
        check(self.L.prism_serve_waves(self.s, wl.ctypes.data, wd.ctypes.data, wu.ctypes.data, wc.ctypes.data,
                                       wo.ctypes.data, wm.ctypes.data))
        return ServeResult(self.trace, adm, pe, ft, comp, hit, eff, wl, wd, wu, wc, wo, wm, c["windows"])

    def cache_view(self):
        """The reference RadixCache API over this replica's tree (tests / debug)."""
        from .dart import DeviceRadixCache

        return DeviceRadixCache.attach(self.t, self.config.cache)


def run_simulation(trace, config, device: int = 0) -> ServeResult:
    """``engine.run_simulation(trace, config)`` on the device; ``trace`` is a
    reference ``Trace`` or a ``TraceCSR``."""
    csr = trace if isinstance(trace, TraceCSR) else TraceCSR.from_trace(trace)
    loop = DeviceServingLoop(config, csr, device=device)
    try:
        loop.run()
        return loop.result()
    finally:
        loop.close()
