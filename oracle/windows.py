"""Windowed parity driver: the CPU oracle run through the SAME serving-loop
windows as the device's fused wave (``WaveEngine.step``), plus whole-tree
comparison tables.

TEST INFRASTRUCTURE ONLY (imported by tests/ and by bench.py's cpu_baseline
leg, which both times the oracle and checks the device against it).

One window (engine.py:171-213 as the device wave runs it):
  1. release the previous window's admitted leaves (engine.py:177-181);
  2. ``schedule_round(pending, active=[], ...)`` (scheduler.py:192-273);
  3. ``set_protection(P-hat)`` for DART (engine.py:193-194) or
     ``note_active_segments`` for LRU_ACTIVE (engine.py:195-197);
  4. for every member in dispatch order: ``serialize_tokens`` of the aligned
     skeleton (workload.py:136-164), ``match_prefix``, ``_build_anchors``
     (engine.py:269-292), ``insert_path``; stop at the first CapacityError
     (engine.py:209-212).
Pending requests that were not admitted stay pending, in arrival order.
"""

from __future__ import annotations

import time

import numpy as np

from oracle.oracle import OracleRadixCache, _ptr, lib as olib, oracle_round_arrays
from paper_2605_08581_b200.qas_host import MarshaledRound
from paper_2605_08581_b200.types import (
    SEGMENT_TOKEN_BASE,
    SUFFIX_TOKEN_BASE,
    CacheConfig,
    CachePolicy,
    SchedulerConfig,
)

SEG_NONE64 = -(2**63)
FIELDS = ("id", "parent", "edge_len", "kind", "seg", "ref", "last", "hits", "prot", "has_anchor", "first_tok")
POOL_KEYS = ("ids", "arrival", "sk_off", "sk", "reorderable", "suffix")


def concat_pools(a: dict | None, b: dict) -> dict:
    """Pending CSR ``a`` followed by ``b``."""
    if a is None or len(a["ids"]) == 0:
        return {k: np.ascontiguousarray(v) for k, v in b.items()}
    out = {}
    for k in ("ids", "arrival", "reorderable", "suffix", "sk"):
        out[k] = np.concatenate([a[k], b[k]])
    out["sk_off"] = np.concatenate([a["sk_off"], a["sk_off"][-1] + b["sk_off"][1:]])
    return out


def drop_members(pool: dict, taken: np.ndarray) -> dict:
    """The pending CSR without the (admitted) indices ``taken``, order kept."""
    P = len(pool["ids"])
    keep = np.ones(P, dtype=bool)
    keep[np.asarray(taken, dtype=np.int64)] = False
    idx = np.flatnonzero(keep)
    lens = np.diff(pool["sk_off"])[idx]
    off = np.zeros(len(idx) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    rows = [pool["sk"][pool["sk_off"][i]:pool["sk_off"][i + 1]] for i in idx.tolist()]
    sk = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    return {"ids": pool["ids"][idx], "arrival": pool["arrival"][idx], "sk_off": off, "sk": sk,
            "reorderable": pool["reorderable"][idx], "suffix": pool["suffix"][idx]}


class OracleReplica:
    """One replica (tree + scheduler) on the CPU oracle, stepped window by window."""

    def __init__(self, cache: CacheConfig, sched: SchedulerConfig, nseg: int, sys_len: int, chunk: int):
        self.cache = OracleRadixCache(cache)
        self.sched = sched
        self.policy = cache.policy
        self.nseg, self.sys_len, self.chunk = nseg, sys_len, chunk
        self.L = olib()
        self.prev: list[int] = []
        self.segs = np.arange(nseg, dtype=np.int64)
        self._leaf = np.zeros(1, np.int64)
        self._nv = np.zeros(1, np.int64)
        self.decision_seconds = 0.0
        self.decisions = 0

    def _path(self, rid: int, segs: np.ndarray, suffix: int) -> np.ndarray:
        s, c = self.sys_len, self.chunk
        p = np.empty(s + len(segs) * c + suffix, dtype=np.uint32)
        p[:s] = np.arange(s)
        p[s:s + len(segs) * c] = (SEGMENT_TOKEN_BASE + segs[:, None].astype(np.int64) * c + np.arange(c)).reshape(-1)
        p[s + len(segs) * c:] = SUFFIX_TOKEN_BASE + rid * suffix + np.arange(suffix)
        return p

    def step(self, pool: dict, deadline: float | None = None, active: tuple | None = None,
             release_prev: bool = True, global_g: np.ndarray | None = None) -> dict:
        """One window over the pending CSR ``pool``; returns dispatch order
        (pending indices), hits, leaf ids and the admitted count.  ``active``:
        the in-flight set's skeleton CSR (act_off, act_sk); ``release_prev``:
        drop the previous window's pins first (the fixed-lag windows)."""
        L, h = self.L, self.cache._h
        if release_prev:
            for leaf in self.prev:
                L.ot_release(h, leaf)
            self.prev = []
        P = len(pool["ids"])
        aoff, ask = active if active is not None else (np.zeros(1, np.int64), np.zeros(0, np.int32))
        m = MarshaledRound(list(range(P)), self.segs, pool["ids"], pool["arrival"], pool["sk_off"],
                           pool["sk"].astype(np.int32), pool["reorderable"], np.asarray(aoff, np.int64),
                           np.asarray(ask, np.int32))
        t0 = time.perf_counter()
        out = oracle_round_arrays(m, self.sched)
        if self.policy is CachePolicy.DART and global_g is not None:
            # the global-demand knob: scheduler.py:247-251 with g := the replicas' summed demand
            w = self.sched.weights
            G = np.asarray(global_g, np.int64)
            dom = np.flatnonzero((G > 0) | (out.a > 0) | (out.nd > 0))
            self.cache.set_protection({int(r): (w.w_g * int(G[r]) + w.w_a * int(out.a[r])) + w.w_n * int(out.nd[r])
                                       for r in dom.tolist()})
        elif self.policy is CachePolicy.DART:
            dom = np.flatnonzero(out.dom)
            self.cache.set_protection(dict(zip(dom.tolist(), out.prio[dom].tolist())))
        elif self.policy is CachePolicy.LRU_ACTIVE:
            self.cache.note_active_segments(np.flatnonzero((out.a > 0) | (out.nd > 0)).tolist())
        members = np.concatenate([out.hot, out.cold]).astype(np.int64)
        hits, leaves = [], []
        for i in members.tolist():
            lo, hi = int(pool["sk_off"][i]), int(pool["sk_off"][i + 1])
            al = out.aligned[lo:hi].astype(np.int64)
            rid, sfx = int(pool["ids"][i]), int(pool["suffix"][i])
            p = self._path(rid, al, sfx)
            k = len(al)
            na = (1 if self.sys_len > 0 else 0) + k + (1 if sfx > 0 else 0)
            a_off = np.empty(na, np.int64)
            a_kind = np.empty(na, np.int8)
            a_seg = np.full(na, SEG_NONE64, np.int64)
            snaps = np.zeros(3 * na, np.int64)
            j = 0
            if self.sys_len > 0:
                a_off[0], a_kind[0] = self.sys_len, 0
                j = 1
            a_off[j:j + k] = self.sys_len + self.chunk * np.arange(1, k + 1)
            a_kind[j:j + k] = 1
            a_seg[j:j + k] = al
            snaps[3 * j:3 * (j + k)] = np.stack([out.g[al], out.a[al], out.nd[al]], axis=1).reshape(-1)
            if sfx > 0:
                a_off[na - 1], a_kind[na - 1] = len(p), 2
            hit = L.ot_match(h, _ptr(p), len(p), None, _ptr(self._nv))
            rc = L.ot_insert(h, _ptr(p), len(p), na, _ptr(a_off), _ptr(a_kind), _ptr(a_seg), _ptr(snaps),
                             _ptr(self._leaf))
            if rc == 1:  # CapacityError: the wave stops (engine.py:209-212)
                break
            if rc != 0:
                raise ValueError(f"oracle insert failed ({rc})")
            hits.append(int(hit))
            leaves.append(int(self._leaf[0]))
            if deadline is not None and time.perf_counter() > deadline:
                break
        el = time.perf_counter() - t0
        self.decision_seconds += el
        self.decisions += len(leaves)
        self.prev = leaves
        return {"members": members, "hits": np.array(hits, np.int64), "leaf_ids": np.array(leaves, np.int64),
                "n_admitted": len(leaves), "seconds": el}

    def table(self) -> np.ndarray:
        n = int(self.L.ot_dump(self.cache._h, None, 0))
        out = np.zeros((max(n, 1), 11), dtype=np.int64)
        self.L.ot_dump(self.cache._h, _ptr(out), n)
        out = out[:n]
        out[out[:, 4] == SEG_NONE64, 4] = -1
        return out

    def victims(self) -> np.ndarray:
        n = int(self.L.ot_victim_log(self.cache._h, None, 0))
        out = np.zeros(max(n, 1), dtype=np.int64)
        self.L.ot_victim_log(self.cache._h, _ptr(out), n)
        return out[:n]

    @property
    def resident(self) -> int:
        return int(self.L.ot_resident(self.cache._h))


def device_table(view) -> np.ndarray:
    """The same 11-column table from a device tree (``DeviceRadixCache`` view)."""
    s = view._snapshot()
    nid, par = s["nid"], s["par"]
    n = len(nid)
    live = np.flatnonzero((nid >= 0) & (par >= 0) & (np.arange(n) != 0))
    seg = s["seg"][live].astype(np.int64)
    seg[seg == -(2**31)] = -1
    ftok = np.where(s["elen"][live] > 0, s["ftok"][live].astype(np.int64), -1)
    t = np.stack([nid[live], nid[par[live]], s["elen"][live], s["kind"][live], seg, s["ref"][live],
                  s["last"][live], s["hits"][live], s["prot"][live], s["hasanc"][live], ftok], axis=1)
    t = t.astype(np.int64)
    return t[np.argsort(t[:, 0], kind="stable")]


def device_victims(view) -> np.ndarray:
    total = view.stats()["victims"]
    ids = np.zeros(max(total, 1), dtype=np.int64)
    z8 = np.zeros(max(total, 1), dtype=np.int8)
    z32 = np.zeros(max(total, 1), dtype=np.int32)
    zu = np.zeros(max(total, 1), dtype=np.uint32)
    z64 = np.zeros(max(total, 1), dtype=np.int64)
    if total:
        first = max(0, total - (1 << 20))  # the device ring keeps the last 2^20 records
        cnt = total - first
        from paper_2605_08581_b200._lib import check

        check(view._L.prism_victims(view._h, first, cnt, _ptr(ids), _ptr(z8), _ptr(z32), _ptr(zu), _ptr(z32),
                                    _ptr(z64)))
        return ids[:cnt], first
    return ids[:0], 0


def compare_tables(a: np.ndarray, b: np.ndarray) -> str | None:
    """None when identical, else a one-line description of the first difference."""
    if a.shape != b.shape:
        return f"node count {a.shape[0]} vs {b.shape[0]}"
    diff = np.argwhere(a != b)
    if len(diff) == 0:
        return None
    r, c = diff[0]
    return f"node {a[r, 0]} field {FIELDS[c]}: {a[r, c]} vs {b[r, c]} ({len(np.unique(diff[:, 0]))} nodes differ)"


def oracle_windows(rep: OracleReplica, windows: list, record_from: int = 0) -> dict:
    """Drive the oracle replica through ``windows`` (arrival pools; requests
    not admitted stay pending).  Records dispatch order / hits / leaf ids of
    the windows from ``record_from`` on, the victim log and the final tree."""
    pend, res = None, {}
    for i, pool in enumerate(windows):
        pend = concat_pools(pend, pool)
        if i == record_from:
            rep.decisions, rep.decision_seconds = 0, 0.0
        r = rep.step(pend)
        if i >= record_from:
            j = i - record_from
            res[f"m{j}"], res[f"h{j}"], res[f"l{j}"] = r["members"], r["hits"], r["leaf_ids"]
        pend = drop_members(pend, r["members"][: r["n_admitted"]])
    res["table"] = rep.table()
    res["victims"] = rep.victims()
    res["resident"] = np.array([rep.resident])
    res["timing"] = np.array([rep.decisions, rep.decision_seconds])
    return res


def device_windows(eng, windows: list, device, record_from: int = 0, reduce_demand=None) -> dict:
    """The same windows through a device replica (``WaveEngine.step``).
    ``reduce_demand(G)``: the global-demand knob -- each window's pending
    demand is computed on the device and reduced over the replicas in place."""
    import torch

    from paper_2605_08581_b200.wave import DevicePending

    G = None
    if reduce_demand is not None:
        G = torch.zeros(eng.nseg, dtype=torch.int32, device=device)
        eng.set_global_demand(G)
    pend, prev, out = None, 0, {}
    for i, pool in enumerate(windows):
        pend = concat_pools(pend, pool)
        eng.release(eng.leaf_slots, prev)
        dp = DevicePending.from_host(pend["ids"], pend["arrival"], pend["sk_off"], pend["sk"], pend["reorderable"],
                                     pend["suffix"], device)
        if G is not None:
            with torch.cuda.stream(eng.stream):
                eng.demand(dp, G)
                reduce_demand(G)
        nm, na = eng.step(dp)
        members = eng.members[:nm].cpu().numpy()
        if i >= record_from:
            j = i - record_from
            out[f"m{j}"], out[f"h{j}"] = members, eng.hits[:na].cpu().numpy()
            out[f"l{j}"] = eng.leaf_ids[:na].cpu().numpy()
        prev = na
        pend = drop_members(pend, members[:na])
    view = eng.cache_view()
    out["table"] = device_table(view)
    out["victims"], out["vfirst"] = device_victims(view)
    out["resident"] = view.resident_tokens
    out["stats"] = eng.wave_stats()
    return out


def compare_windows(d: dict, o, waves: int, path_len: int | None = None) -> dict:
    """Parity verdict of device outputs ``d`` against oracle outputs ``o``."""
    diffs = []
    for j in range(waves):
        for key, name in (("m", "dispatch order"), ("h", "hits"), ("l", "leaf ids")):
            if not np.array_equal(np.asarray(d[f"{key}{j}"]), np.asarray(o[f"{key}{j}"])):
                diffs.append(f"window {j}: {name}")
    ov = np.asarray(o["victims"])
    dv = d["victims"]
    if d["vfirst"] + len(dv) != len(ov) or not np.array_equal(dv, ov[d["vfirst"]:]):
        diffs.append(f"victims ({len(ov)} oracle, {d['vfirst'] + len(dv)} device)")
    t = compare_tables(d["table"], np.asarray(o["table"]))
    if t:
        diffs.append("tree: " + t)
    if int(d["resident"]) != int(np.asarray(o["resident"]).reshape(-1)[0]):
        diffs.append("resident tokens")
    adm = sum(len(o[f"l{j}"]) for j in range(waves))
    hit = sum(int(np.asarray(o[f"h{j}"]).sum()) for j in range(waves))
    out = {"waves_checked": waves, "identical": not diffs, "differences": diffs[:5], "decisions_checked": adm,
           "victims_checked": int(len(ov)), "tree_nodes_checked": int(len(o["table"])),
           "device_commit": d["stats"]}
    if path_len:
        out["hit_rate"] = hit / max(adm * path_len, 1)
    return out


def pool_demand(pool: dict, nseg: int) -> np.ndarray:
    """count_segments (scheduler.py:83-89) of a pending CSR, dense int64 [nseg]."""
    G = np.zeros(nseg, np.int64)
    off, sk = pool["sk_off"], pool["sk"]
    for i in range(len(off) - 1):
        G[np.unique(sk[off[i]:off[i + 1]])] += 1
    return G


def oracle_windows_global(reps: list, windows: list, record_rank: int, record_from: int = 0) -> dict:
    """The replicas of every shard in lockstep (``windows[r]`` = rank r's
    arrival pools): each window, every replica's pending demand is summed (the
    per-window all-reduce) and fed to all of them as P-hat (the global-demand
    knob); records rank ``record_rank`` like ``oracle_windows``."""
    world = len(reps)
    pends = [None] * world
    res = {}
    for i in range(len(windows[0])):
        for r in range(world):
            pends[r] = concat_pools(pends[r], windows[r][i])
        G = sum(pool_demand(pends[r], reps[r].nseg) for r in range(world))
        for r in range(world):
            if i == record_from:
                reps[r].decisions, reps[r].decision_seconds = 0, 0.0
            out = reps[r].step(pends[r], global_g=G)
            if r == record_rank and i >= record_from:
                j = i - record_from
                res[f"m{j}"], res[f"h{j}"], res[f"l{j}"] = out["members"], out["hits"], out["leaf_ids"]
            pends[r] = drop_members(pends[r], out["members"][: out["n_admitted"]])
    rep = reps[record_rank]
    res["table"] = rep.table()
    res["victims"] = rep.victims()
    res["resident"] = np.array([rep.resident])
    res["timing"] = np.array([rep.decisions, rep.decision_seconds])
    return res
