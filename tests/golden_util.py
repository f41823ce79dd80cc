"""Loaders and replayers for the reference-generated fixtures in tests/golden/.

The same replayers drive the CPU oracle (CPU tests) and the device cache
(GPU tests), so both are compared against the identical reference record.
"""

from __future__ import annotations

import gzip
import hashlib
import io
import json
import os
from functools import lru_cache

from sim_harness import SimConfig, run_simulation
from paper_2605_08581_b200.types import (
    Anchor,
    CacheConfig,
    CachePolicy,
    CapacityError,
    NodeKind,
    PriorityWeights,
    ReleaseError,
    Request,
    SchedulerConfig,
)
from traces.refgen import load_trace

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def load(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


def H(x) -> str:
    return hashlib.sha256(json.dumps(x).encode()).hexdigest()[:16]


# ------------------------------------------------------------------ engine


def engine_case(i: int):
    doc = load("engine_runs.json.gz")
    run = doc["runs"][i]
    trace = load_trace(io.StringIO(doc["traces"][run["trace"]]))
    s = run["sim"]
    cfg = SimConfig(
        prefill_rate=s["prefill_rate"],
        decode_rate=s["decode_rate"],
        output_tokens=s["output_tokens"],
        cache=CacheConfig(
            capacity_tokens=run["capacity"],
            policy=CachePolicy(run["policy"]),
            protect_budget=s["protect_budget"],
        ),
        scheduler=SchedulerConfig(
            window_s=s["window_s"],
            dispatch_budget=s["dispatch_budget"],
            cold_quota=s["cold_quota"],
            front_width=s["front_width"],
            signature_size=s["signature_size"],
            weights=PriorityWeights(),
        ),
    )
    return run, trace, cfg


def run_engine_case(i: int, cache_factory, schedule_fn, admit: str = "call"):
    """Run golden engine case i; returns (observed dict, expected run record)."""
    run, trace, cfg = engine_case(i)
    holder = {}
    res = run_simulation(
        trace,
        cfg,
        cache_factory=cache_factory,
        schedule_fn=schedule_fn,
        admit=admit,
        cache_hook=lambda c: holder.setdefault("cache", c),
    )
    cache = holder["cache"]
    obs = {
        "hit_rate": res.run.hit_rate,
        "hits": [m.hit_tokens for m in res.requests],
        "admission": [w.members for w in res.waves],
        "victims": cache.victim_log(),
        "ttft": [m.ttft for m in res.requests],
    }
    return obs, run


def assert_engine_parity(obs, run, ttft_rel=1e-6):
    assert obs["hits"] == run["hits"], "per-request hit tokens differ"
    assert obs["admission"] == run["admission"], "admission order differs"
    assert obs["victims"] == run["victims"], "eviction victims differ"
    assert obs["hit_rate"] == run["hit_rate"]
    for a, b in zip(obs["ttft"], run["ttft"]):
        assert abs(a - b) <= ttft_rel * max(abs(b), 1e-12)
    # SURVEY.md Appendix A digests
    d = run["digest"]
    assert H(obs["hits"]) == d[1] and H(obs["admission"]) == d[2] and H(obs["victims"]) == d[3]
    assert len(obs["victims"]) == d[4]


# ------------------------------------------------------------------ DART ops


def _anchors(js) -> list[Anchor]:
    return [Anchor(o, NodeKind(k), s, tuple(snap)) for o, k, s, snap in js]


def replay_dart_case(case: dict, cache_factory) -> None:
    """Replay one recorded op sequence and assert every recorded result."""
    cache = cache_factory(
        CacheConfig(
            capacity_tokens=case["capacity"],
            policy=CachePolicy(case["policy"]),
            protect_budget=case["protect_budget"],
        )
    )
    leaves: dict[int, object] = {}
    for step, op in enumerate(case["ops"]):
        ctx = f"step {step} op {op['op']}"
        kind = op["op"]
        if kind == "match":
            hit, visited = cache.match_prefix(op["path"])
            assert hit == op["hit"], ctx
            assert [n.node_id for n in visited] == op["visited"], ctx
        elif kind == "insert":
            try:
                leaf = cache.insert_path(op["path"], _anchors(op["anchors"]))
                assert op["leaf"] == leaf.node_id, ctx
                leaves[leaf.node_id] = leaf
            except CapacityError:
                assert op["leaf"] is None, ctx
            assert cache.resident_tokens == op["resident"], ctx
        elif kind == "release":
            try:
                cache.release_path(leaves[op["leaf"]])
                ok = True
            except ReleaseError:
                ok = False
            assert ok == op["ok"], ctx
        elif kind == "protect":
            prot = cache.set_protection({int(k): v for k, v in op["prio"]})
            assert sorted(prot) == op["protected"], ctx
        elif kind == "active":
            cache.note_active_segments(op["segs"])
        elif kind == "evict":
            freed = cache.evict(op["k"])
            assert freed == op["freed"], ctx
            assert [n.node_id for n in cache.last_evicted] == op["victims"], ctx
            assert cache.resident_tokens == op["resident"], ctx
    assert cache.debug_nodes() == case["final_nodes"]
    assert cache.resident_tokens == case["resident"]


# ------------------------------------------------------------------ QAS


def qas_case(case: dict):
    def req(js):
        rid, arr, sk, reo, sys_len, reuse, suffix = js
        return Request(rid, arr, list(sk), reo, [], sys_len, reuse, suffix)

    pending = [req(r) for r in case["pending"]]
    active = [req(r) for r in case["active"]]
    b, c, f, s = case["config"]
    cfg = SchedulerConfig(dispatch_budget=b, cold_quota=c, front_width=f, signature_size=s)
    return pending, active, cfg


def assert_qas_case(case: dict, batch) -> None:
    assert [r.id for r in batch.hot] == case["hot"]
    assert [r.id for r in batch.cold] == case["cold"]
    assert set(batch.hints) == {int(k) for k in case["hints"]}
    for rid, (sig, rank, snap, offs, aligned) in case["hints"].items():
        h = batch.hints[int(rid)]
        assert list(h.signature) == sig
        assert h.rank == rank
        assert {int(k): list(v) for k, v in snap.items()} == {k: list(v) for k, v in h.counter_snapshot.items()}
        assert h.anchor_offsets == offs
        assert h.aligned_skeleton == aligned
    assert [[k, v] for k, v in sorted(batch.priorities.items())] == sorted(case["priorities"])
    assert sorted(batch.counters.g.items()) == sorted((k, v) for k, v in case["g"])
    assert sorted(batch.counters.a.items()) == sorted((k, v) for k, v in case["a"])
    assert sorted(batch.counters.n.items()) == sorted((k, v) for k, v in case["n"])
    assert [[list(k), v] for k, v in batch.bucket_scores.items()] == case["bucket_scores"]
