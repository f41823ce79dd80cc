"""The windowed parity driver (oracle/windows.py) that bench.py and the
at-scale GPU parity tests use, pinned on CPU against the serving-loop
semantics it claims (engine.py:171-213): the same windows driven through the
reference's OWN RadixCache and schedule_round (baseline/_ref, when installed)
and through the Python API of the pinned oracle."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from oracle.oracle import OracleRadixCache, oracle_schedule_round
from oracle.windows import OracleReplica, concat_pools, drop_members
from paper_2605_08581_b200.types import (
    CacheConfig,
    CachePolicy,
    CapacityError,
    Request,
    SchedulerConfig,
    SegmentCatalog,
    build_anchors,
    serialize_tokens,
)
from traces import synth as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

CASES = {
    # (workload, spec override): small trees, capacity stops carry requests over
    "c3_small": dict(workload="c3", sys_len=64, chunk=4, cap=4000, wave=40, windows=6, policy=CachePolicy.DART),
    "mu_small": dict(workload="mu1m", sys_len=28, chunk=16, cap=4000, wave=48, windows=6, policy=CachePolicy.DART),
    "c4_lru": dict(workload="c4", sys_len=28, chunk=8, cap=1000, wave=32, windows=6, policy=CachePolicy.LRU),
    "c4_lru_active": dict(workload="c4", sys_len=28, chunk=8, cap=1000, wave=32, windows=6,
                          policy=CachePolicy.LRU_ACTIVE),
    "c3_lfu": dict(workload="c3", sys_len=16, chunk=2, cap=1500, wave=24, windows=6, policy=CachePolicy.LFU),
}


def _pools(case, seed=1):
    rng = np.random.default_rng(seed)
    out, nid = [], 0
    for _ in range(case["windows"]):
        p = S.make_pool(case["workload"], nid, case["wave"], rng)
        p["suffix"] = (p["suffix"] // 16).astype(np.int32)  # short suffixes keep the trees small
        nid += case["wave"]
        out.append(p)
    return out


def _requests(pend, case):
    reqs = []
    for i in range(len(pend["ids"])):
        sk = pend["sk"][pend["sk_off"][i]:pend["sk_off"][i + 1]].astype(int).tolist()
        reqs.append(Request(int(pend["ids"][i]), float(pend["arrival"][i]), sk, bool(pend["reorderable"][i]), [],
                            case["sys_len"], len(sk) * case["chunk"], int(pend["suffix"][i])))
    return reqs


def _api_loop(case, cache, schedule, kv_capacity_error, anchors_of=build_anchors, sched=None):
    """The windows through the Python API (the reference's call sequence)."""
    nseg = S.SPECS[case["workload"]].nseg
    cat = SegmentCatalog(num_segments=nseg, chunk_tokens=case["chunk"], hot_set=(), sys_prefix_tokens=case["sys_len"])
    pend, prev, out = None, [], []
    for pool in _pools(case):
        pend = concat_pools(pend, pool)
        for leaf in prev:
            cache.release_path(leaf)
        reqs = _requests(pend, case)
        b = schedule(reqs, [], sched, 0.0)
        if case["policy"] is CachePolicy.DART:
            cache.set_protection(b.priorities)
        elif case["policy"] is CachePolicy.LRU_ACTIVE:
            from paper_2605_08581_b200.types import count_segments

            cache.note_active_segments(r for r, c in count_segments(b.members).items() if c > 0)
        idx = {r.id: i for i, r in enumerate(reqs)}
        hits, leaves = [], []
        for r in b.members:
            h = b.hints[r.id]
            path = serialize_tokens(r, cat, h.aligned_skeleton)
            hit = cache.match_prefix(path)[0]
            try:
                leaves.append(cache.insert_path(path, anchors_of(r, h.aligned_skeleton, h.counter_snapshot)))
            except kv_capacity_error:
                break
            hits.append(hit)
        members = [idx[r.id] for r in b.members]
        out.append((members, hits, [x.node_id for x in leaves]))
        prev = leaves
        pend = drop_members(pend, np.array(members[: len(leaves)], dtype=np.int64))
    return out


def _replica_loop(case):
    cfg = CacheConfig(capacity_tokens=case["cap"], policy=case["policy"], protect_budget=5)
    sched = SchedulerConfig(dispatch_budget=case["wave"], cold_quota=4)
    rep = OracleReplica(cfg, sched, S.SPECS[case["workload"]].nseg, case["sys_len"], case["chunk"])
    pend, out = None, []
    for pool in _pools(case):
        pend = concat_pools(pend, pool)
        r = rep.step(pend)
        out.append((r["members"].tolist(), r["hits"].tolist(), r["leaf_ids"].tolist()))
        pend = drop_members(pend, r["members"][: r["n_admitted"]])
    return out, rep


@pytest.mark.parametrize("name", sorted(CASES))
def test_replica_matches_oracle_api_loop(name):
    case = CASES[name]
    got, rep = _replica_loop(case)
    cfg = CacheConfig(capacity_tokens=case["cap"], policy=case["policy"], protect_budget=5)
    sched = SchedulerConfig(dispatch_budget=case["wave"], cold_quota=4)
    ora = OracleRadixCache(cfg)
    want = _api_loop(case, ora, oracle_schedule_round, CapacityError, sched=sched)
    assert got == want
    assert sum(len(w[2]) for w in want) > 0
    assert any(len(w[2]) < len(w[0]) for w in want), "the case should hit capacity stops"
    assert rep.victims().tolist() == ora.victim_log()
    t = rep.table()
    assert [int(x) for x in t[:, 0]] == sorted(n["node_id"] for n in ora.debug_nodes())


@pytest.fixture(scope="module")
def prefixsim():
    if not os.path.isdir(os.path.join(REF, "prefixsim")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import prefixsim.engine  # noqa: F401
        import prefixsim.kvcache  # noqa: F401
        import prefixsim.scheduler  # noqa: F401
    finally:
        sys.path.remove(REF)
    return sys.modules["prefixsim"]


@pytest.mark.parametrize("name", ["c3_small", "mu_small", "c4_lru_active"])
def test_replica_matches_reference_itself(prefixsim, name):
    """The same windows through the UNMODIFIED reference classes."""
    K, Sch, E = prefixsim.kvcache, prefixsim.scheduler, prefixsim.engine
    case = CASES[name]
    got, rep = _replica_loop(case)
    cfg = K.CacheConfig(capacity_tokens=case["cap"], policy=K.CachePolicy(case["policy"].value), protect_budget=5)
    cache = K.RadixCache(cfg)
    victims = []
    orig = cache.evict

    def evict(k):
        f = orig(k)
        victims.extend(n.node_id for n in cache.last_evicted)
        return f

    cache.evict = evict
    sched = Sch.SchedulerConfig(dispatch_budget=case["wave"], cold_quota=4)
    want = _api_loop(case, cache, Sch.schedule_round, K.CapacityError, anchors_of=E._build_anchors, sched=sched)
    assert got == want
    assert rep.victims().tolist() == victims
