"""The fused device wave (prism_wave_step) against the CPU oracle.

Each wave: QAS round -> protection / active-set hand-off -> serialization ->
admission, on the device (exact parallel commit with ordered fallback, and
the ordered commit alone) and on the oracle driven exactly like
engine.py:189-213.  Compared per wave: dispatch order, hit lengths, leaf
node ids; at the end: the whole tree (debug_nodes) and every eviction victim.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import OracleRadixCache, oracle_schedule_round
from paper_2605_08581_b200.types import build_anchors
from paper_2605_08581_b200.types import (
    CacheConfig,
    CachePolicy,
    CapacityError,
    Request,
    SchedulerConfig,
    SegmentCatalog,
    count_segments,
    serialize_tokens,
)

pytestmark = pytest.mark.gpu


def _requests(rng, first_id, n, nseg, hot, kmin, kmax, suffixes, sys, chunk, zipf=1.3, reo=1.0):
    reqs = []
    for i in range(n):
        k = int(rng.integers(kmin, kmax + 1))
        sk = []
        if rng.random() < 0.7 and hot:
            sk.append(int(min(rng.zipf(zipf), hot) - 1))
        while len(sk) < k:
            c = int(rng.integers(0, nseg))
            if c not in sk:
                sk.append(c)
        sfx = int(rng.choice(suffixes))
        reqs.append(Request(first_id + i, float(first_id + i) * 0.01, sk, bool(rng.random() < reo), [], sys, k * chunk,
                            sfx))
    return reqs


def _pending_arrays(reqs):
    P = len(reqs)
    off = np.zeros(P + 1, np.int64)
    np.cumsum([len(r.skeleton) for r in reqs], out=off[1:])
    return (np.array([r.id for r in reqs], np.int64), np.array([r.arrival_time for r in reqs], np.float64), off,
            np.array([s for r in reqs for s in r.skeleton], np.int32),
            np.array([1 if r.reorderable else 0 for r in reqs], np.uint8),
            np.array([r.suffix_len for r in reqs], np.int32))


def run_case(seed, policy, mode, nseg=40, hot=6, kmin=2, kmax=5, suffixes=(2, 4), sys=8, chunk=4, cap=600,
             wave=24, nwaves=8, protect=3, cold=2, tiny=False, coop=1, sample=1, reo=1.0, prebuild=1,
             split_waves=()):
    import torch

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    rng = np.random.default_rng(seed)
    cfg = CacheConfig(capacity_tokens=cap, policy=policy, protect_budget=protect)
    scfg = SchedulerConfig(dispatch_budget=wave, cold_quota=cold)
    eng = WaveEngine(cfg, scfg, nseg, sys, chunk, device=0)
    eng.set_commit_mode(mode)
    eng.tune(use_coop=coop, use_sample=sample, prebuild=prebuild)
    if tiny:  # minimal selected prefixes of the eviction order
        eng.tune(list_min_tokens=1, list_slack_tokens=0, sel_min_candidates=0)
    ora = OracleRadixCache(cfg)
    cat = SegmentCatalog(num_segments=nseg, chunk_tokens=chunk, hot_set=tuple(range(min(hot, nseg))),
                         sys_prefix_tokens=sys)
    dev_prev = 0
    ora_prev = []
    next_id = 0
    for w in range(nwaves):
        reqs = _requests(rng, next_id, wave + int(rng.integers(0, 6)), nseg, hot, kmin, kmax, suffixes, sys, chunk,
                         reo=reo)
        next_id += len(reqs)
        pend = DevicePending.from_host(*_pending_arrays(reqs), torch.device("cuda", 0))
        eng.release(eng.leaf_slots, dev_prev)
        nm, na = eng.step(pend)
        dev_prev = na
        members = eng.members[:nm].cpu().tolist()
        hits = eng.hits[:na].cpu().tolist()
        leaf_ids = eng.leaf_ids[:na].cpu().tolist()
        # oracle, the engine's own order of operations
        for leaf in ora_prev:
            ora.release_path(leaf)
        ora_prev = []
        b = oracle_schedule_round(reqs, [], scfg, 0.0)
        idx = {r.id: i for i, r in enumerate(reqs)}
        assert members == [idx[r.id] for r in b.members], f"wave {w}: dispatch order"
        if policy is CachePolicy.DART:
            ora.set_protection(b.priorities)
        elif policy is CachePolicy.LRU_ACTIVE:
            counts = count_segments(b.members)
            ora.note_active_segments(r for r, c in counts.items() if c > 0)
        ohits, oleaves = [], []
        for r in b.members:
            h = b.hints[r.id]
            path = serialize_tokens(r, cat, h.aligned_skeleton)
            hit = ora.match_prefix(path)[0]
            try:
                oleaves.append(ora.insert_path(path, build_anchors(r, h.aligned_skeleton, h.counter_snapshot)))
            except CapacityError:
                break
            ohits.append(hit)
        ora_prev = oleaves
        assert hits == ohits, f"wave {w}: hits"
        assert leaf_ids == [x.node_id for x in oleaves], f"wave {w}: leaf ids"
        if w in split_waves and b.members:
            # a per-call insert that splits a node on the pinned root path of
            # this wave's first member (mid-way into its first segment piece),
            # released at once: the next wave's release must not trust the
            # root paths the parallel commit recorded (k_release_par)
            r = b.members[0]
            path = serialize_tokens(r, cat, b.hints[r.id].aligned_skeleton)
            cut = sys + max(chunk // 2, 1)
            probe = list(path[:cut]) + [10_000_000 + 7 * w + q for q in range(3)]
            view = eng.cache_view()
            view.release_path(view.insert_path(probe))
            ora.release_path(ora.insert_path(probe))
            assert view.debug_nodes() == ora.debug_nodes(), f"wave {w}: split probe"
    view = eng.cache_view()
    assert view.debug_nodes() == ora.debug_nodes()
    assert view.victim_log() == ora.victim_log()
    assert view.resident_tokens == ora.resident_tokens
    return eng.wave_stats()


@pytest.mark.parametrize("policy", list(CachePolicy))
@pytest.mark.parametrize("seed", range(3))
def test_parallel_commit_matches_oracle(policy, seed):
    st = run_case(seed, policy, mode=0)
    assert st["parallel_waves"] > 0, st


@pytest.mark.parametrize("policy", [CachePolicy.DART, CachePolicy.LRU])
def test_release_after_split(policy):
    """Releases of a parallel wave's members after a split on their pinned
    paths (the recorded root paths are stale: every leaf climbs), and the
    recorded-path release of the waves without one."""
    st = run_case(5, policy, mode=0, split_waves=(1, 4, 5), nwaves=9)
    assert st["parallel_waves"] > 0, st


@pytest.mark.parametrize("policy", [CachePolicy.DART, CachePolicy.LRU])
def test_ordered_commit_matches_oracle(policy):
    st = run_case(11, policy, mode=1)
    assert st["parallel_waves"] == 0


@pytest.mark.parametrize("variant", [
    dict(suffixes=(0,), kmin=1, kmax=3),               # shared whole paths, prefix paths
    dict(sys=0, suffixes=(0, 3)),                      # no system prompt
    dict(cap=120, wave=16, nwaves=10),                 # capacity stops (ordered fallback)
    dict(nseg=8, hot=4, kmin=3, kmax=6, wave=48),      # heavy intra-wave sharing
    dict(chunk=1, sys=3, kmax=8, suffixes=(1, 2)),     # one-token segments
    dict(cap=100_000, nwaves=4),                       # no eviction at all
    dict(tiny=True),                                   # minimal eviction-order prefixes
    dict(tiny=True, cap=150, wave=32, nwaves=10),      # ... with capacity stops
    dict(coop=0),                                      # multi-kernel build / protection
    dict(coop=0, tiny=True),
    dict(sample=0),                                    # materialising radix selection only
    dict(sample=0, tiny=True),
    dict(prebuild=0),                                  # whole build on the tree stream
    dict(prebuild=0, tiny=True),
    dict(cap=100_000, nwaves=4, tiny=True),            # sample taken ahead, no eviction demand
    dict(reo=0.0),                                     # non-reorderable skeletons (no front-alignment)
    dict(reo=0.5, kmin=1, kmax=6),                     # mixed
    dict(nseg=300, hot=8, kmin=20, kmax=40, suffixes=(0, 8), wave=16, nwaves=6, cap=6000),  # agent-like deep paths
    dict(nseg=300, hot=8, kmin=20, kmax=40, suffixes=(8,), wave=24, nwaves=8, cap=900, reo=0.0),  # ... evicting
    dict(cap=260, wave=48, nwaves=12, protect=8),      # eviction stress: most of the tree turns over per wave
    dict(protect=30, nseg=12, hot=3, kmin=1, kmax=2),  # fewer positive-P-hat anchors than the budget (fallback top-f)
    dict(protect=60, nseg=40, cap=2000, wave=32),      # ... and a budget near the small top-f's limit
])
def test_parallel_commit_variants(variant):
    run_case(5, CachePolicy.DART, mode=0, **variant)


def _mu_pool(rng, first, n, k=6, chunk=8, slot0=20, others=200_000, suffix=8):
    sk = np.empty((n, k), dtype=np.int32)
    sk[:, 0] = rng.integers(0, slot0, size=n)
    sk[:, 1:] = slot0 + rng.integers(0, others, size=(n, k - 1))
    ids = np.arange(first, first + n, dtype=np.int64)
    return (ids, ids.astype(np.float64) * 1e-3, np.arange(n + 1, dtype=np.int64) * k, sk.reshape(-1),
            np.ones(n, np.uint8), np.full(n, suffix, np.int32))


@pytest.mark.parametrize("protect", [20, 3000])
def test_sampled_selection_at_scale(protect):
    """~150K-node tree, every wave evicts: the sampled eviction-prefix / top-f
    selection (coop.cuh) commits exactly what the materialising radix selection
    commits -- hits, leaf ids, the whole victim log and the final tree."""
    import torch

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    dev = torch.device("cuda", 0)
    runs = []
    for sample, pre in ((1, 1), (0, 0), (1, 0)):
        rng = np.random.default_rng(5)
        cfg = CacheConfig(capacity_tokens=1_000_000, policy=CachePolicy.DART, protect_budget=protect)
        eng = WaveEngine(cfg, SchedulerConfig(dispatch_budget=2048, cold_quota=16), 20 + 200_000, 12, 8, device=0)
        eng.tune(use_sample=sample, prebuild=pre)
        nid, prev, out, sampled = 0, 0, [], 0
        for w in range(30):
            pend = DevicePending.from_host(*_mu_pool(rng, nid, 2048), dev)
            nid += 2048
            eng.release(eng.leaf_slots, prev)
            nm, prev = eng.step(pend)
            out.append((eng.members[:nm].cpu().tolist(), eng.hits[:prev].cpu().tolist(),
                        eng.leaf_ids[:prev].cpu().tolist()))
            sampled += eng.build_timeline()["sampled"]
        view = eng.cache_view()
        runs.append((out, view.victim_log(), view.debug_nodes(), eng.stats()["live_nodes"], sampled))
        eng.close()
    (o1, v1, d1, n1, s1), (o0, v0, d0, n0, s0), (o2, v2, d2, n2, s2) = runs
    assert n1 > 100_000 and len(v1) > 10_000
    assert s1 > 0 and s2 > 0 and s0 == 0  # the sampled path ran (and only where enabled)
    assert o1 == o0 == o2
    assert v1 == v0 == v2
    assert d1 == d0 == d2


def test_graph_replay_matches_plain_launches():
    """The wave tail replayed as a CUDA graph (fixed wave shape: captured on the
    second wave, replayed after) commits exactly what plain launches commit."""
    import torch

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    dev = torch.device("cuda", 0)
    runs = []
    for graph in (True, False):
        rng = np.random.default_rng(9)
        cfg = CacheConfig(capacity_tokens=400_000, policy=CachePolicy.DART, protect_budget=20)
        eng = WaveEngine(cfg, SchedulerConfig(dispatch_budget=1024, cold_quota=16), 20 + 200_000, 12, 8, device=0)
        eng.set_graph(graph)
        nid, prev, out = 0, 0, []
        for w in range(40):
            pend = DevicePending.from_host(*_mu_pool(rng, nid, 1024), dev)
            nid += 1024
            eng.release(eng.leaf_slots, prev)
            nm, prev = eng.step(pend)
            out.append((eng.members[:nm].cpu().tolist(), eng.hits[:prev].cpu().tolist(),
                        eng.leaf_ids[:prev].cpu().tolist()))
        view = eng.cache_view()
        runs.append((out, view.victim_log(), view.debug_nodes(), eng.graph_stats()))
        eng.close()
    (o1, v1, d1, g1), (o0, v0, d0, g0) = runs
    assert g1["replays"] > 10 and g0["replays"] == 0, (g1, g0)
    assert o1 == o0
    assert v1 == v0
    assert d1 == d0


def test_step_host_matches_device_step():
    """prism_wave_step_host (pinned host inputs read in place, results copied
    to host inside the wave, release folded in) == prism_wave_step."""
    import torch

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    dev = torch.device("cuda", 0)
    outs = []
    for host in (True, False):
        rng = np.random.default_rng(13)
        cfg = CacheConfig(capacity_tokens=200_000, policy=CachePolicy.DART, protect_budget=10)
        eng = WaveEngine(cfg, SchedulerConfig(dispatch_budget=512, cold_quota=8), 20 + 200_000, 12, 8, device=0)
        nid, prev, out = 0, 0, []
        om, oh = np.empty(512, np.int64), np.empty(512, np.int64)
        for w in range(30):
            arrs = _mu_pool(rng, nid, 512)
            nid += 512
            if host:
                names = ("ids", "arrival", "sk_off", "sk", "reorderable", "suffix")
                pool = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for k, a in zip(names, arrs)}
                nm, na = eng.step_host(pool, om, oh, release_n=prev)
                out.append((om[:nm].tolist(), oh[:na].tolist(), eng.leaf_ids[:na].cpu().tolist()))
            else:
                eng.release(eng.leaf_slots, prev)
                nm, na = eng.step(DevicePending.from_host(*arrs, dev))
                out.append((eng.members[:nm].cpu().tolist(), eng.hits[:na].cpu().tolist(),
                            eng.leaf_ids[:na].cpu().tolist()))
            prev = na
        outs.append((out, eng.cache_view().victim_log()))
        eng.close()
    assert outs[0] == outs[1]


def _csr_active(reqs):
    off = np.zeros(len(reqs) + 1, np.int64)
    np.cumsum([len(r.skeleton) for r in reqs], out=off[1:])
    return off, np.array([s for r in reqs for s in r.skeleton], np.int32)


def run_inflight(seed, policy, lag=3, host=False, wave=24, pend=30, nwaves=10, cap=700, nseg=40, hot=6,
                 kmin=2, kmax=5, protect=3, cold=2, mode=0):
    """Waves with requests in flight (engine.py:171-189): each wave's members
    stay pinned for ``lag`` waves and form the next rounds' active set, which
    feeds the a-counters (w_a = 1e6) and, under LRU_ACTIVE, the active-segment
    flags.  Device (step / step_host with the active CSR) vs the oracle."""
    import torch

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(seed)
    cfg = CacheConfig(capacity_tokens=cap, policy=policy, protect_budget=protect)
    scfg = SchedulerConfig(dispatch_budget=wave, cold_quota=cold)
    eng = WaveEngine(cfg, scfg, nseg, 8, 4, device=0)
    eng.set_commit_mode(mode)
    ora = OracleRadixCache(cfg)
    cat = SegmentCatalog(num_segments=nseg, chunk_tokens=4, hot_set=tuple(range(min(hot, nseg))), sys_prefix_tokens=8)
    inflight = []  # (wave, admitted requests, device leaf slots, oracle leaves)
    om, oh = np.empty(max(pend + 6, wave), np.int64), np.empty(max(pend + 6, wave), np.int64)
    next_id = 0
    for w in range(nwaves):
        for f in [x for x in inflight if x[0] <= w - lag]:  # completions
            eng.release(f[2], f[2].shape[0])
            for leaf in f[3]:
                ora.release_path(leaf)
        inflight = [x for x in inflight if x[0] > w - lag]
        active = [r for x in inflight for r in x[1]]
        reqs = _requests(rng, next_id, pend + int(rng.integers(0, 6)), nseg, hot, kmin, kmax, (2, 4), 8, 4)
        next_id += len(reqs)
        aoff, ask = _csr_active(active)
        if host:
            names = ("ids", "arrival", "sk_off", "sk", "reorderable", "suffix")
            pool = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                    for k, a in zip(names, _pending_arrays(reqs))}
            act = {"sk_off": torch.from_numpy(aoff).pin_memory(), "sk": torch.from_numpy(ask).pin_memory()}
            nm, na = eng.step_host(pool, om, oh, release_n=0, active=act)
            members, hits = om[:nm].tolist(), oh[:na].tolist()
        else:
            act = DevicePending(torch.zeros(len(active), dtype=torch.int64, device=dev),
                                torch.zeros(len(active), dtype=torch.float64, device=dev),
                                torch.from_numpy(aoff).to(dev), torch.from_numpy(ask).to(dev),
                                torch.zeros(len(active), dtype=torch.uint8, device=dev),
                                torch.zeros(len(active), dtype=torch.int32, device=dev))
            nm, na = eng.step(DevicePending.from_host(*_pending_arrays(reqs), dev), act)
            members, hits = eng.members[:nm].cpu().tolist(), eng.hits[:na].cpu().tolist()
        leaf_ids = eng.leaf_ids[:na].cpu().tolist()
        b = oracle_schedule_round(reqs, active, scfg, 0.0)
        idx = {r.id: i for i, r in enumerate(reqs)}
        assert members == [idx[r.id] for r in b.members], f"wave {w}: dispatch order"
        if policy is CachePolicy.DART:
            ora.set_protection(b.priorities)
        elif policy is CachePolicy.LRU_ACTIVE:
            counts = count_segments(list(active) + list(b.members))
            ora.note_active_segments(r for r, c in counts.items() if c > 0)
        ohits, oleaves = [], []
        for r in b.members:
            h = b.hints[r.id]
            path = serialize_tokens(r, cat, h.aligned_skeleton)
            hit = ora.match_prefix(path)[0]
            try:
                oleaves.append(ora.insert_path(path, build_anchors(r, h.aligned_skeleton, h.counter_snapshot)))
            except CapacityError:
                break
            ohits.append(hit)
        assert hits == ohits, f"wave {w}: hits"
        assert leaf_ids == [x.node_id for x in oleaves], f"wave {w}: leaf ids"
        inflight.append((w, b.members[:na], eng.leaf_slots[:na].clone(), oleaves))
    view = eng.cache_view()
    assert view.debug_nodes() == ora.debug_nodes()
    assert view.victim_log() == ora.victim_log()
    eng.close()


@pytest.mark.parametrize("policy", list(CachePolicy))
@pytest.mark.parametrize("host", [False, True])
def test_inflight_active_set(policy, host):
    run_inflight(3, policy, host=host)


@pytest.mark.parametrize("variant", [
    dict(lag=1),                                   # nothing in flight at the round (A = 0)
    dict(lag=5, cap=2000, nwaves=12),              # deep in-flight set
    dict(mode=1),                                  # ordered commit
    dict(pend=9000, wave=4096, cold=64, nwaves=4, cap=200_000, nseg=3000, hot=40),  # P > 4096: multi-kernel round
])
def test_inflight_variants(variant):
    run_inflight(7, CachePolicy.DART, **variant)


@pytest.mark.parametrize("variant", [
    dict(cap=300, wave=24, nwaves=8, nseg=100_000, hot=0),            # no sharing: no chain conflicts
    dict(cap=250, wave=32, nwaves=12, suffixes=(0, 2)),
    dict(cap=500, wave=48, nwaves=8, nseg=50_000, hot=1, kmin=3, kmax=6),
])
def test_capacity_stop_commits_in_parallel(variant):
    """A wave whose demand exceeds the evictable tokens stops at the first member
    the whole eviction order cannot satisfy (CapacityError, engine.py:209-212):
    the members before it commit in parallel, the stopping member's match and
    evict sweep are applied, and everything equals the oracle."""
    st = run_case(21, CachePolicy.DART, mode=0, protect=2, **variant)
    assert st["capacity_stops"] > 0, st
