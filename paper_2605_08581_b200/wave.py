"""Fused device wave: one serving-loop wave of QAS + DART without host round trips.

``WaveEngine.step(pending)`` runs engine.py:189-213 for a DEVICE-resident
pending set (``DevicePending``, torch tensors used purely as device buffers):
the QAS round, the protection / active-set hand-off, serialisation of every
member's token path from its aligned skeleton, and ordered
match+insert+evict, all inside libprism.so.  ``release`` drops the pins of
a completed wave (engine.py:177-181).  This is the path bench.py measures.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check
from .qas import _cfg
from .types import CacheConfig, POLICY_CODE, SchedulerConfig, policy_of

_p = C.c_void_p
_i64 = C.c_int64


def _bind(lib):
    sig = {
        "prism_wave_step": (C.c_int, [_p, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _p, _p, C.c_int32, _p,
                                      _i64, _i64, _p, _p, _p, _p, _p, _p]),
        "prism_wave_step_host": (C.c_int, [_p, _p, _i64, _p, _p, _p, _p, _p, _p, _i64, _p, _p, C.c_int32, _p, _i64,
                                           _i64, _i64,
                                           _p, _p, _p, _p, _p, _p, _p, _p, _p]),
        "prism_qas_stream": (_p, [_p]),
        "prism_qas_counters": (C.c_int, [_p, _p, C.c_int32]),
        "prism_qas_demand": (C.c_int, [_p, _i64, _p, _p, C.c_int32, _p]),
        "prism_qas_set_global_demand": (C.c_int, [_p, _p, C.c_int32]),
        "prism_qas_defer_release": (C.c_int, [_p, _i64, _p]),
        "prism_set_protection_device": (C.c_int, [_p, _p, C.c_int32, _p, _p]),
        "prism_profile": (C.c_int, [_p, C.c_int32]),
        "prism_profile_read": (C.c_int, [_p, _p]),
        "prism_qas_counts": (C.c_int, [_p, _p]),
        "prism_qas_profile": (C.c_int, [_p, C.c_int32]),
        "prism_qas_set_commit_mode": (C.c_int, [_p, C.c_int32]),
        "prism_wave_stats": (C.c_int, [_p, _p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


@dataclass
class DevicePending:
    """A pending snapshot as device CSR (ids, arrival, skeleton offsets/ids,
    reorderable flags, suffix lengths); segment ids dense in [0, nseg)."""

    ids: torch.Tensor  # int64 [P]
    arrival: torch.Tensor  # float64 [P]
    sk_off: torch.Tensor  # int64 [P+1]
    sk: torch.Tensor  # int32
    reorderable: torch.Tensor  # uint8 [P]
    suffix: torch.Tensor  # int32 [P]

    @property
    def P(self) -> int:
        return int(self.ids.shape[0])

    @staticmethod
    def from_host(ids, arrival, sk_off, sk, reorderable, suffix, device) -> "DevicePending":
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)  # noqa: E731
        return DevicePending(t(ids, torch.int64), t(arrival, torch.float64), t(sk_off, torch.int64),
                             t(sk, torch.int32), t(reorderable, torch.uint8), t(suffix, torch.int32))

    def nbytes(self) -> int:
        return sum(x.numel() * x.element_size() for x in
                   (self.ids, self.arrival, self.sk_off, self.sk, self.reorderable, self.suffix))


class WaveEngine:
    """One replica: a device tree (DART) + a device scheduler (QAS)."""

    def __init__(self, cache: CacheConfig, sched: SchedulerConfig, nseg: int, sys_len: int, chunk: int,
                 device: int = 0, initial_slots: int = 0, initial_arena_tokens: int = 0):
        _lib.require_device()
        self.L = _bind(_lib.lib())
        self.device = device
        self.cache_cfg, self.sched = cache, sched
        self.nseg, self.sys_len, self.chunk = nseg, sys_len, chunk
        self.t = self.L.prism_tree_create(cache.capacity_tokens, POLICY_CODE[policy_of(cache.policy)],
                                          cache.protect_budget, initial_slots, initial_arena_tokens, device)
        if not self.t:
            raise _lib.PrismError(_lib.last_error())
        self.q = self.L.prism_qas_create(device)
        if not self.q:
            raise _lib.PrismError(_lib.last_error())
        self._cfg = _cfg(sched)
        dev = torch.device("cuda", device)
        cap = max(sched.dispatch_budget, 1)
        self.members = torch.empty(cap, dtype=torch.int64, device=dev)
        self.hits = torch.empty(cap, dtype=torch.int64, device=dev)
        self.leaf_slots = torch.empty(cap, dtype=torch.int32, device=dev)
        self.leaf_ids = torch.empty(cap, dtype=torch.int64, device=dev)
        self._nm = np.zeros(1, np.int64)
        self._na = np.zeros(1, np.int64)
        self.stream = torch.cuda.ExternalStream(self.L.prism_qas_stream(self.q), device=dev)

    def close(self) -> None:
        if getattr(self, "t", None):
            self.L.prism_tree_destroy(self.t)
            self.t = None
        if getattr(self, "q", None):
            self.L.prism_qas_destroy(self.q)
            self.q = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    def step(self, pend: DevicePending, active: DevicePending | None = None, release_n: int = 0,
             release_slots: torch.Tensor | None = None) -> tuple[int, int]:
        """One wave; returns (members dispatched, members admitted).

        ``active``: the requests in flight (engine.py:189 ``active.values()``),
        whose skeletons (``sk_off`` / ``sk``) feed the round's a-counters
        (w_a, scheduler.py:203) and, under LRU_ACTIVE, the active-segment flags
        (engine.py:195-197).  None: no request in flight."""
        P = pend.P
        A, aoff, ask = self._active(active)
        if release_n > 0:  # completions dropped by the wave itself, beside its QAS round
            slots = self.leaf_slots if release_slots is None else release_slots
            if release_slots is None and P > self.members.shape[0]:
                raise ValueError("release_n refers to leaf_slots, which a larger pending set would reallocate")
            check(self.L.prism_qas_defer_release(self.q, int(release_n), slots.data_ptr()))
        self._ensure(P)
        check(self.L.prism_wave_step(
            self.t, self.q, P, pend.ids.data_ptr(), pend.arrival.data_ptr(), pend.sk_off.data_ptr(),
            pend.sk.data_ptr(), pend.reorderable.data_ptr(), pend.suffix.data_ptr(), A, aoff, ask,
            self.nseg, C.addressof(self._cfg),
            self.sys_len, self.chunk, self.members.data_ptr(), self.hits.data_ptr(), self.leaf_slots.data_ptr(),
            self.leaf_ids.data_ptr(), self._nm.ctypes.data, self._na.ctypes.data,
        ))
        return int(self._nm[0]), int(self._na[0])

    def _ensure(self, P: int) -> None:
        """Per-member device outputs for a pending set of P (dispatch <= P)."""
        if P > self.members.shape[0]:
            dev = self.members.device
            self.members = torch.empty(P, dtype=torch.int64, device=dev)
            self.hits = torch.empty(P, dtype=torch.int64, device=dev)
            self.leaf_slots = torch.empty(P, dtype=torch.int32, device=dev)
            self.leaf_ids = torch.empty(P, dtype=torch.int64, device=dev)

    @staticmethod
    def _active(active) -> tuple[int, int, int]:
        if active is None:
            return 0, 0, 0
        if isinstance(active, dict):
            off, sk = active["sk_off"], active["sk"]
        else:
            off, sk = active.sk_off, active.sk
        A = int(off.shape[0]) - 1
        if A <= 0:
            return 0, 0, 0
        return A, off.data_ptr(), sk.data_ptr()

    def step_host(self, pool: dict, out_members: np.ndarray, out_hits: np.ndarray, release_n: int = 0,
                  active: dict | None = None) -> tuple[int, int]:
        """One wave from host memory to host memory (the end-to-end entry point).

        ``pool`` maps ids / arrival / sk_off / sk / reorderable / suffix to
        pinned host tensors (read in place by the device); the previous wave's
        ``release_n`` pins (``self.leaf_slots``) are dropped first; the dispatch
        order and the hits come back in ``out_members`` / ``out_hits`` (int64).
        ``active``: the in-flight requests' skeleton CSR (``sk_off`` / ``sk``,
        pinned host tensors), as in ``step``."""
        P = int(pool["ids"].shape[0])
        A, aoff, ask = self._active(active)
        if release_n > 0 and P > self.members.shape[0]:
            raise ValueError("release_n refers to leaf_slots, which a larger pending set would reallocate")
        self._ensure(P)
        if out_members.shape[0] < min(P, self.sched.dispatch_budget) or out_hits.shape[0] < min(
                P, self.sched.dispatch_budget):
            raise ValueError("out_members / out_hits smaller than the wave")
        check(self.L.prism_wave_step_host(
            self.t, self.q, P, pool["ids"].data_ptr(), pool["arrival"].data_ptr(), pool["sk_off"].data_ptr(),
            pool["sk"].data_ptr(), pool["reorderable"].data_ptr(), pool["suffix"].data_ptr(), A, aoff, ask, self.nseg,
            C.addressof(self._cfg), self.sys_len, self.chunk, release_n, self.leaf_slots.data_ptr(),
            self.members.data_ptr(), self.hits.data_ptr(), self.leaf_slots.data_ptr(), self.leaf_ids.data_ptr(),
            out_members.ctypes.data, out_hits.ctypes.data, self._nm.ctypes.data, self._na.ctypes.data,
        ))
        return int(self._nm[0]), int(self._na[0])

    def release(self, slots: torch.Tensor, n: int) -> None:
        """Drop the pins of n admitted leaves (completions, engine.py:177-181)."""
        if n > 0:
            check(self.L.prism_release_device(self.t, n, slots.data_ptr(), None,
                                              self.L.prism_qas_stream(self.q)))

    def demand_counters(self, dst: torch.Tensor) -> None:
        """Last round's pending demand counters g (int32 [nseg]) into dst."""
        check(self.L.prism_qas_counters(self.q, dst.data_ptr(), self.nseg))

    def demand(self, pend, dst: torch.Tensor) -> None:
        """count_segments(pending) (scheduler.py:83-89) into dst (int32 [nseg],
        device): this replica's per-window demand counters.  ``pend``: a
        DevicePending or a pool of pinned host tensors (read in place)."""
        off, sk = (pend["sk_off"], pend["sk"]) if isinstance(pend, dict) else (pend.sk_off, pend.sk)
        check(self.L.prism_qas_demand(self.q, int(off.shape[0]) - 1, off.data_ptr(), sk.data_ptr(), self.nseg,
                                      dst.data_ptr()))

    def set_global_demand(self, G: torch.Tensor | None) -> None:
        """Global-demand knob (multi-GPU): the protection hand-off uses P-hat
        from G (the replicas' all-reduced demand, read at every wave) instead
        of the local round's g.  None: the reference behaviour."""
        self._gdem = G
        check(self.L.prism_qas_set_global_demand(self.q, G.data_ptr() if G is not None else None,
                                                 self.nseg if G is not None else 0))

    def set_graph(self, enable: bool) -> None:
        """Replay the wave's tail (protection, serialization, commit) as a CUDA graph."""
        self.L.prism_qas_tune.argtypes = [_p, C.c_int32, _i64, _p]
        check(self.L.prism_qas_tune(self.q, 4, 1 if enable else 0, None))

    def graph_stats(self) -> dict:
        self.L.prism_qas_tune.argtypes = [_p, C.c_int32, _i64, _p]
        out = np.zeros(3, dtype=np.int64)
        check(self.L.prism_qas_tune(self.q, 5, 3, out.ctypes.data))
        return {"captures": int(out[0]), "replays": int(out[1]), "pdl_edges": int(out[2])}

    def set_commit_mode(self, mode: int) -> None:
        """0: exact parallel wave commit with ordered fallback; 1: ordered only."""
        check(self.L.prism_qas_set_commit_mode(self.q, mode))

    def wave_stats(self) -> dict:
        out = np.zeros(4, dtype=np.int64)
        check(self.L.prism_wave_stats(self.t, out.ctypes.data))
        return {"parallel_waves": int(out[0]), "ordered_waves": int(out[1]), "last_fallback": int(out[2]),
                "capacity_stops": int(out[3])}

    def tune(self, **kw) -> None:
        """Eviction-list prefix sizing (see DeviceRadixCache.tune)."""
        from .dart import DeviceRadixCache

        for k, v in kw.items():
            check(self.L.prism_tune(self.t, DeviceRadixCache.TUNABLES[k], int(v)))

    def build_timeline(self) -> dict:
        """Phase durations (us) of the last cooperative eviction-list build."""
        self.L.prism_coop_timeline.argtypes = [_p, _p, _p]
        out = np.zeros(40, dtype=np.uint64)
        n = np.zeros(1, dtype=np.int32)
        check(self.L.prism_coop_timeline(self.t, out.ctypes.data, n.ctypes.data))
        ts = out[: n[0]].astype(np.int64)
        return {"phases_us": (np.diff(ts) / 1e3).round(1).tolist(), "selected": int(out[39]),
                "sampled": int(out[38]), "samples": int(out[33]), "splitters": int(out[34]),
                "fallback_reason": int(out[35]), "kept_mass": int(out[36]), "W": int(out[37]),
                "dbg": out[21:33].astype(np.int64).tolist()}

    def cache_view(self):
        """The reference RadixCache API over this engine's tree (tests/debug)."""
        from .dart import DeviceRadixCache

        return DeviceRadixCache.attach(self.t, self.cache_cfg)

    def reusable_anchors(self) -> int:
        """Live nodes carrying a REUSABLE anchor: the A of the protection scan's
        16-A algorithmic bytes (kvcache.py:374-376)."""
        s = self.cache_view()._snapshot()
        live = (s["nid"] >= 0) & (s["par"] >= 0)
        return int(np.count_nonzero(live & (s["hasanc"] != 0) & (s["akind"] == 1)))

    def profile(self, enable: bool) -> None:
        check(self.L.prism_profile(self.t, 1 if enable else 0))
        check(self.L.prism_qas_profile(self.q, 1 if enable else 0))

    PHASES = ("commit", "build", "protect", "prematch", "release", "note", "maint")

    def profile_read(self) -> dict:
        """Cumulative live profile: device ms / calls / launches per phase."""
        out = np.zeros(27, dtype=np.float64)
        check(self.L.prism_profile_read(self.t, out.ctypes.data))
        qc = np.zeros(4, dtype=np.int64)
        check(self.L.prism_qas_counts(self.q, qc.ctypes.data))
        prof = {p: {"ms": float(out[i]), "calls": int(out[8 + i]), "launches": int(out[16 + i])}
                for i, p in enumerate(self.PHASES)}
        prof["qas"] = {"ms": qc[3] / 1000.0, "calls": int(qc[2]), "launches": int(qc[0])}
        prof["lib_calls"] = int(out[24]) + int(qc[1])
        prof["chain_nodes"] = int(out[25])
        prof["inserted_tokens"] = int(out[26])
        return prof

    def compactions(self) -> int:
        """Token-arena compactions so far (maintenance between waves)."""
        self.L.prism_compactions.restype = C.c_int64
        self.L.prism_compactions.argtypes = [_p]
        return int(self.L.prism_compactions(self.t))

    def stats(self) -> dict:
        out = np.zeros(16, dtype=np.int64)
        check(self.L.prism_stats(self.t, out.ctypes.data))
        keys = ["resident", "clock", "next_id", "hw", "live_nodes", "arena_used", "hash_live", "hash_tomb",
                "victims", "evict_calls", "builds", "slot_cap", "arena_cap", "hash_cap", "fast_members",
                "slow_members"]
        return dict(zip(keys, out.tolist()))
