"""Generate tests/golden/ fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Writes (gzip JSON, small):
  engine_runs.json.gz   SURVEY.md Appendix A configurations: trace (JSONL
                        text), per-request hit tokens, admission waves,
                        every eviction victim (node id, in order), TTFTs,
                        hit rate -- from prefixsim.engine.run_simulation.
  dart_ops.json.gz      random op sequences on prefixsim.kvcache.RadixCache
                        with every result and the final debug_nodes().
  qas_rounds.json.gz    random rounds of prefixsim.scheduler.schedule_round
                        with the full DispatchBatch.
The fixtures are the pins for oracle/ (tests/test_oracle_golden.py) and,
through the oracle and directly, for the device path.
"""

from __future__ import annotations

import gzip
import hashlib
import io
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import prefixsim.engine as E  # noqa: E402
import prefixsim.kvcache as K  # noqa: E402
from prefixsim.experiment import SimSpec, WorkloadSpec  # noqa: E402
from prefixsim.kvcache import Anchor, CacheConfig, CachePolicy, NodeKind, RadixCache  # noqa: E402
from prefixsim.scheduler import SchedulerConfig, schedule_round  # noqa: E402
from prefixsim.workload import Request, generate_trace, save_trace  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# SURVEY.md Appendix A (cap, qps, policy, seed)
ENGINE_CONFIGS = [
    (32000, 40.0, "DART", 1),
    (32000, 40.0, "LRU", 1),
    (32000, 40.0, "LRU_ACTIVE", 1),
    (32000, 40.0, "LFU", 1),
    (5760, 20.0, "DART", 1),
    (12557, 40.0, "DART", 1),
    (32000, 10.0, "DART", 2),
]


def H(x) -> str:
    return hashlib.sha256(json.dumps(x).encode()).hexdigest()[:16]


def engine_runs() -> dict:
    victims: list[int] = []
    orig = K.RadixCache.evict

    def _evict(self, k):
        f = orig(self, k)
        victims.extend(n.node_id for n in self.last_evicted)
        return f

    K.RadixCache.evict = _evict
    wl = WorkloadSpec()
    traces: dict[str, str] = {}
    runs = []
    try:
        for cap, qps, pol, seed in ENGINE_CONFIGS:
            victims.clear()
            tr = generate_trace(wl.config(qps, seed), wl.catalog())
            tkey = f"q{qps:g}_s{seed}"
            if tkey not in traces:
                buf = io.StringIO()
                save_trace(tr, buf)
                traces[tkey] = buf.getvalue()
            sim = SimSpec(capacity_tokens=cap)
            r = E.run_simulation(tr, sim.config(CachePolicy(pol), 2))
            hits = [m.hit_tokens for m in r.requests]
            adm = [w.members for w in r.waves]
            ttft = [m.ttft for m in r.requests]
            runs.append(
                {
                    "capacity": cap,
                    "qps": qps,
                    "policy": pol,
                    "seed": seed,
                    "trace": tkey,
                    "sim": {
                        "prefill_rate": sim.prefill_rate,
                        "decode_rate": sim.decode_rate,
                        "output_tokens": sim.output_tokens,
                        "protect_budget": sim.protect_budget,
                        "window_s": sim.window_s,
                        "dispatch_budget": sim.dispatch_budget,
                        "cold_quota": 2,
                        "front_width": sim.front_width,
                        "signature_size": sim.signature_size,
                    },
                    "hit_rate": r.run.hit_rate,
                    "p99": r.run.p99,
                    "hits": hits,
                    "admission": adm,
                    "victims": list(victims),
                    "ttft": ttft,
                    "digest": [
                        r.run.hit_rate,
                        H(hits),
                        H(adm),
                        H(victims),
                        len(victims),
                        H(ttft),
                    ],
                }
            )
            print(f"engine {cap} {qps} {pol} {seed}: hit_rate={r.run.hit_rate} victims={len(victims)}")
    finally:
        K.RadixCache.evict = orig
    return {"traces": traces, "runs": runs}


# ------------------------------------------------------------------ DART ops


def _anchor_json(a: Anchor) -> list:
    return [a.offset, a.kind.value, a.segment_id, list(a.counter_snapshot)]


def dart_ops(n_instances: int = 160) -> list:
    """Random op sequences (mirrors test_kvcache.py:285-317 and widens it:
    tight capacities so inserts evict and raise CapacityError, repeated
    protection/active updates, direct evicts, double releases)."""
    out = []
    policies = list(CachePolicy)
    for inst in range(n_instances):
        rng = np.random.default_rng(10_000 + inst)
        policy = policies[inst % 4]
        cap = int(rng.choice([12, 24, 40, 64, 100_000]))
        prot = int(rng.integers(0, 4))
        cache = RadixCache(CacheConfig(capacity_tokens=cap, policy=policy, protect_budget=prot))
        alphabet = int(rng.integers(2, 6))
        leaves: dict[int, object] = {}
        ops = []
        for step in range(int(rng.integers(5, 60))):
            r = rng.random()
            if r < 0.45:
                length = int(rng.integers(0, min(cap, 20) + 1))
                path = [int(t) for t in rng.integers(0, alphabet, size=length)]
                anchors = []
                if length >= 2 and rng.random() < 0.8:
                    mid = int(rng.integers(1, length))
                    if rng.random() < 0.5 and mid > 1:
                        anchors.append(Anchor(int(rng.integers(1, mid)), NodeKind.SYSTEM))
                    anchors.append(
                        Anchor(mid, NodeKind.REUSABLE, segment_id=int(rng.integers(0, 8)),
                               counter_snapshot=(int(rng.integers(0, 5)), int(rng.integers(0, 2)), int(rng.integers(0, 3))))
                    )
                    anchors.append(Anchor(length, NodeKind.PRIVATE))
                hit, visited = cache.match_prefix(path)
                rec = {"op": "match", "path": path, "hit": hit, "visited": [n.node_id for n in visited]}
                ops.append(rec)
                try:
                    leaf = cache.insert_path(path, anchors)
                    leaves[leaf.node_id] = leaf
                    ops.append({"op": "insert", "path": path, "anchors": [_anchor_json(a) for a in anchors],
                                "leaf": leaf.node_id, "resident": cache.resident_tokens})
                except K.CapacityError:
                    ops.append({"op": "insert", "path": path, "anchors": [_anchor_json(a) for a in anchors],
                                "leaf": None, "resident": cache.resident_tokens})
            elif r < 0.65 and leaves:
                lid = int(rng.choice(sorted(leaves)))
                try:
                    cache.release_path(leaves[lid])
                    ok = True
                except K.ReleaseError:
                    ok = False
                if rng.random() < 0.7:
                    leaves.pop(lid)
                ops.append({"op": "release", "leaf": lid, "ok": ok})
            elif r < 0.75:
                pr = {int(s): float(np.round(rng.random() * 10, 3)) for s in range(8) if rng.random() < 0.7}
                protected = cache.set_protection(pr)
                ops.append({"op": "protect", "prio": [[k, v] for k, v in pr.items()],
                            "protected": sorted(protected)})
            elif r < 0.82:
                act = [int(s) for s in range(8) if rng.random() < 0.3]
                cache.note_active_segments(act)
                ops.append({"op": "active", "segs": act})
            elif r < 0.92:
                k = int(rng.integers(0, max(cache.resident_tokens, 1) + 1))
                freed = cache.evict(k)
                ops.append({"op": "evict", "k": k, "freed": freed,
                            "victims": [n.node_id for n in cache.last_evicted],
                            "resident": cache.resident_tokens})
            else:
                length = int(rng.integers(0, 20))
                path = [int(t) for t in rng.integers(0, alphabet, size=length)]
                hit, visited = cache.match_prefix(path)
                ops.append({"op": "match", "path": path, "hit": hit, "visited": [n.node_id for n in visited]})
        out.append({"policy": policy.value, "capacity": cap, "protect_budget": prot, "ops": ops,
                    "final_nodes": cache.debug_nodes(), "resident": cache.resident_tokens})
    return out


# ------------------------------------------------------------------ QAS


def _req(rid, skel, arrival, reorderable, sys_len, chunk, suffix):
    return Request(id=rid, arrival_time=arrival, skeleton=list(skel), reorderable=reorderable,
                   token_path=[], sys_len=sys_len, reuse_len=len(skel) * chunk, suffix_len=suffix)


def _req_json(r: Request) -> list:
    return [r.id, r.arrival_time, r.skeleton, r.reorderable, r.sys_len, r.reuse_len, r.suffix_len]


def qas_rounds(n_rounds: int = 300) -> list:
    """Random rounds (mirrors test_scheduler.py:289-328, widened: duplicate
    segments inside a skeleton, kappa > 1, larger pendings)."""
    rng = np.random.default_rng(4242)
    out = []
    for trial in range(n_rounds):
        n_seg = int(rng.integers(1, 14))
        n_req = int(rng.integers(0, 60)) if trial % 10 else int(rng.integers(100, 400))
        pending = []
        for i in range(n_req):
            k = int(rng.integers(0, min(n_seg, 6) + 1))
            if rng.random() < 0.1:
                skel = [int(s) for s in rng.integers(0, n_seg, size=k)]  # duplicates allowed
            else:
                skel = [int(s) for s in rng.choice(n_seg, size=k, replace=False)]
            arr = float(np.round(rng.random(), 2))  # ties on arrival exercise the id tie-break
            pending.append(_req(i * 3 + 1, skel, arr, bool(rng.random() < 0.8), 10, 8, 4))
        active = [_req(1000 + j, [int(s) for s in rng.choice(n_seg, size=int(rng.integers(1, 3)))], 0.0, True, 10, 8, 4)
                  for j in range(int(rng.integers(0, 6)))]
        sig = int(rng.integers(1, 3))
        cfg = SchedulerConfig(dispatch_budget=int(rng.integers(2, 16)), cold_quota=int(rng.integers(0, 3)),
                              front_width=int(rng.integers(sig, 5)), signature_size=sig)
        b = schedule_round(pending, active, cfg, now=0.0)
        out.append(
            {
                "pending": [_req_json(r) for r in pending],
                "active": [_req_json(r) for r in active],
                "config": [cfg.dispatch_budget, cfg.cold_quota, cfg.front_width, cfg.signature_size],
                "hot": [r.id for r in b.hot],
                "cold": [r.id for r in b.cold],
                "hints": {
                    str(rid): [list(h.signature), h.rank, {str(s): list(v) for s, v in h.counter_snapshot.items()},
                               h.anchor_offsets, h.aligned_skeleton]
                    for rid, h in b.hints.items()
                },
                "priorities": [[s, v] for s, v in b.priorities.items()],
                "g": [[s, v] for s, v in b.counters.g.items()],
                "a": [[s, v] for s, v in b.counters.a.items()],
                "n": [[s, v] for s, v in b.counters.n.items()],
                "bucket_scores": [[list(s), v] for s, v in b.bucket_scores.items()],
            }
        )
    return out


def _write(name: str, obj) -> None:
    path = os.path.join(OUT, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    _write("qas_rounds.json.gz", qas_rounds())
    _write("dart_ops.json.gz", dart_ops())
    _write("engine_runs.json.gz", engine_runs())
