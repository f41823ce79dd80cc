"""Device QAS parity against the reference record (golden rounds), the
reference's own scheduler scenarios (test_scheduler.py), and the oracle on
large randomized rounds."""

from __future__ import annotations

import numpy as np
import pytest

import golden_util as G
from oracle.oracle import oracle_schedule_round
from paper_2605_08581_b200.types import Request, SchedulerConfig

pytestmark = pytest.mark.gpu


def sched(pending, active, cfg, now=0.0):
    from paper_2605_08581_b200.qas import schedule_round

    return schedule_round(pending, active, cfg, now)


def make_request(rid, skeleton, arrival=0.0, reorderable=True, sys_len=10, chunk=8, suffix=4):
    return Request(rid, arrival, list(skeleton), reorderable, [], sys_len, len(skeleton) * chunk, suffix)


@pytest.mark.parametrize("small", [4096, True, False])
def test_golden_rounds(small):
    from paper_2605_08581_b200.qas import DeviceScheduler

    ds = DeviceScheduler()
    ds.set_small(small)  # one-CTA rounds vs the multi-kernel round
    for i, case in enumerate(G.load("qas_rounds.json.gz")):
        pending, active, cfg = G.qas_case(case)
        try:
            G.assert_qas_case(case, ds.schedule_round(pending, active, cfg, 0.0))
        except AssertionError as e:
            raise AssertionError(f"round {i}: {e}") from e


@pytest.mark.parametrize("small", [4096, True])
def test_mixed_round_sizes_one_scheduler(small):
    """Small (one-launch) and large (multi-kernel) rounds interleaved on one
    scheduler: the per-round counter reset (touched lists / full resets) must
    never leak state between rounds.  small=True: one-launch rounds up to 8192
    pending (only P=8000+ ... none here above it: every round one launch)."""
    from paper_2605_08581_b200.qas import DeviceScheduler

    ds = DeviceScheduler()
    ds.set_small(small)
    rng = np.random.default_rng(31)
    for P in (100, 5000, 200, 300, 8000, 50, 4096, 1):
        nseg = int(rng.integers(20, 3000))
        pend = [Request(i, float(rng.random()), [int(x) for x in rng.choice(nseg, size=int(rng.integers(1, 7)),
                                                                          replace=False)], True, [], 8, 32, 4)
                for i in range(P)]
        act = [Request(10**6 + j, 0.0, [int(rng.integers(0, nseg))], True, [], 8, 8, 4) for j in range(3)]
        cfg = SchedulerConfig(dispatch_budget=min(P, 512) or 1, cold_quota=min(2, min(P, 512) or 1))
        bd = ds.schedule_round(pend, act, cfg, 0.0)
        bo = oracle_schedule_round(pend, act, cfg)
        assert [r.id for r in bd.members] == [r.id for r in bo.members], P
        assert bd.priorities == bo.priorities, P
        assert bd.bucket_scores == bo.bucket_scores, P
        assert bd.counters.g == bo.counters.g and bd.counters.n == bo.counters.n, P


@pytest.mark.parametrize("small", [4096, False])
def test_long_skeletons(small):
    """Skeletons longer than the per-thread limit (64) are aligned by a whole
    block (rank counting); a round whose skeleton entries exceed the one-CTA
    buffers is redone by the multi-kernel path.  Duplicated segments, fronts
    wider than kappa and non-reorderable requests included; the next round
    must see clean counters."""
    from paper_2605_08581_b200.qas import DeviceScheduler

    ds = DeviceScheduler()
    ds.set_small(small)
    rng = np.random.default_rng(5)
    for r in range(8):
        P = [40, 2, 300, 3, 40, 5000, 7, 64][r]
        nseg = [200, 50, 1000, 30, 200, 3000, 400, 90][r]

        def skel(i):
            k = int(rng.choice([3, 70, 150, 700])) if i % 5 == r % 5 else int(rng.integers(1, 6))
            return [int(x) for x in rng.integers(0, nseg, size=k)]  # duplicates allowed

        pend = [Request(i, float(rng.integers(0, 50)), skel(i), bool(rng.random() < 0.8), [], 8, 32, 4)
                for i in range(P)]
        act = [Request(10**6 + j, 0.0, [int(x) for x in rng.integers(0, nseg, size=80)], True, [], 8, 8, 4)
               for j in range(2)]
        cfg = SchedulerConfig(dispatch_budget=min(P, 16), cold_quota=min(P, 2), front_width=[3, 90, 5][r % 3],
                              signature_size=[2, 1, 4][r % 3])
        bd = ds.schedule_round(pend, act, cfg, 0.0)
        bo = oracle_schedule_round(pend, act, cfg)
        assert [r_.id for r_ in bd.members] == [r_.id for r_ in bo.members], r
        assert bd.priorities == bo.priorities and bd.bucket_scores == bo.bucket_scores, r
        assert bd.counters.g == bo.counters.g and bd.counters.a == bo.counters.a, r
        for rid, h in bo.hints.items():
            d = bd.hints[rid]
            assert (d.signature, d.rank, d.aligned_skeleton, d.counter_snapshot) == (
                h.signature, h.rank, h.aligned_skeleton, h.counter_snapshot), (r, rid)


@pytest.mark.parametrize("case", range(6))
def test_warp_aligned_skeletons(case):
    """Skeletons of 17..64 segments (the agent / C3 regime, k=40) are aligned
    by one warp per request with selection rounds: duplicates, equal
    priorities (seg / index tie-breaks), fronts and signatures from 1 to wider
    than k, reorderable and not, mixed with short (16-lane) and long (block)
    skeletons in one round."""
    from paper_2605_08581_b200.qas import DeviceScheduler

    ds = DeviceScheduler()
    ds.set_small(4096)
    rng = np.random.default_rng(100 + case)
    P = [64, 500, 4096, 1000, 3, 2000][case]
    nseg = [40, 300, 5000, 64, 20, 100000][case]
    front, kappa = [(3, 1), (40, 4), (70, 64), (2, 2), (64, 64), (3, 1)][case]

    def skel(i):
        k = int(rng.choice([17, 31, 32, 33, 40, 63, 64])) if i % 7 else int(rng.choice([1, 5, 16, 65, 90]))
        if case % 2:  # duplicates allowed
            return [int(x) for x in rng.integers(0, nseg, size=k)]
        return [int(x) for x in rng.choice(max(nseg, k), size=k, replace=False)]

    pend = [Request(i, float(rng.integers(0, 50)), skel(i), bool(rng.random() < [0.0, 0.5, 1.0][case % 3]), [],
                    8, 32, 4) for i in range(P)]
    act = [Request(10**6 + j, 0.0, [int(x) for x in rng.integers(0, nseg, size=40)], True, [], 8, 8, 4)
           for j in range(case)]
    cfg = SchedulerConfig(dispatch_budget=min(P, 1024), cold_quota=min(P, 16), front_width=front,
                          signature_size=kappa)
    bd = ds.schedule_round(pend, act, cfg, 0.0)
    bo = oracle_schedule_round(pend, act, cfg)
    assert [r_.id for r_ in bd.members] == [r_.id for r_ in bo.members]
    assert bd.priorities == bo.priorities and bd.bucket_scores == bo.bucket_scores
    assert bd.counters.g == bo.counters.g and bd.counters.a == bo.counters.a and bd.counters.n == bo.counters.n
    for rid, h in bo.hints.items():
        d = bd.hints[rid]
        assert (d.signature, d.rank, d.aligned_skeleton, d.counter_snapshot) == (
            h.signature, h.rank, h.aligned_skeleton, h.counter_snapshot), rid


class TestScheduleRound:
    def test_single_request(self):
        b = sched([make_request(0, [3, 1])], [], SchedulerConfig(dispatch_budget=4, cold_quota=1))
        assert [r.id for r in b.members] == [0] and b.hints[0].aligned_skeleton[0] in (1, 3)

    def test_empty_pending(self):
        assert sched([], [], SchedulerConfig()).members == []

    def test_cold_lane_takes_oldest(self):
        cfg = SchedulerConfig(dispatch_budget=3, cold_quota=1, front_width=1, signature_size=1)
        reqs = [make_request(0, [1], 0.0), make_request(1, [1], 0.1), make_request(2, [2], 0.2),
                make_request(3, [3], 0.3)]
        b = sched(reqs, [], cfg, 1.0)
        assert [r.id for r in b.hot] == [0, 1] and [r.id for r in b.cold] == [2]

    def test_starvation_guard_progress(self):
        cfg = SchedulerConfig(dispatch_budget=4, cold_quota=1, front_width=1)
        hot = [make_request(i, [1], 0.01 * i) for i in range(20)]
        loner = make_request(99, [9], 0.0)
        assert loner.id in {r.id for r in sched(hot + [loner], [], cfg, 1.0).cold}

    def test_priorities_cover_dispatch_segments(self):
        b = sched([make_request(0, [1, 2]), make_request(1, [2, 3])], [], SchedulerConfig(dispatch_budget=4, cold_quota=0))
        assert set(b.priorities) >= {1, 2, 3}
        assert b.priorities[2] == 2 * 1.0 + 2 * 1e5

    def test_purity(self):
        cfg = SchedulerConfig(dispatch_budget=4, cold_quota=1)
        reqs = [make_request(i, [i % 3, 3 + i % 2]) for i in range(6)]
        before = [(r.id, list(r.skeleton)) for r in reqs]
        b1 = sched(reqs, [], cfg)
        b2 = sched(reqs, [], cfg)
        assert before == [(r.id, list(r.skeleton)) for r in reqs]
        assert [r.id for r in b1.members] == [r.id for r in b2.members]


@pytest.mark.parametrize("seed", range(4))
def test_large_rounds_vs_oracle(seed):
    """Deep queues (the post-knee regime) with Zipf-skewed segments."""
    rng = np.random.default_rng(seed)
    P = [1000, 5000, 20000, 50000][seed]
    nseg = [50, 981, 5000, 100000][seed]
    pend = []
    for i in range(P):
        k = int(rng.integers(1, 9))
        sk = [int(min(rng.zipf(1.2), nseg) - 1)] + [int(x) for x in rng.integers(0, nseg, size=k - 1)]
        pend.append(Request(i, float(rng.random() * 10), sk, bool(rng.random() < 0.9), [], 28, 128 * k, 100))
    active = [Request(10**6 + j, 0.0, [int(x) for x in rng.integers(0, nseg, size=3)], True, [], 28, 384, 100)
              for j in range(int(rng.integers(0, 50)))]
    cfg = SchedulerConfig(dispatch_budget=[64, 512, 2048, 4096][seed], cold_quota=[2, 8, 32, 64][seed],
                          front_width=3, signature_size=1 + seed % 2)
    bd = sched(pend, active, cfg)
    bo = oracle_schedule_round(pend, active, cfg)
    assert [r.id for r in bd.hot] == [r.id for r in bo.hot]
    assert [r.id for r in bd.cold] == [r.id for r in bo.cold]
    assert bd.priorities == bo.priorities
    assert bd.bucket_scores == bo.bucket_scores
    for rid, h in bo.hints.items():
        d = bd.hints[rid]
        assert (d.signature, d.rank, d.aligned_skeleton, d.counter_snapshot, d.anchor_offsets) == (
            h.signature, h.rank, h.aligned_skeleton, h.counter_snapshot, h.anchor_offsets)


@pytest.mark.parametrize("case", range(len(G.load("engine_runs.json.gz")["runs"])))
def test_engine_runs_full_device(case):
    """Both halves of the hot path on the device: QAS + DART (wave admission)."""
    from paper_2605_08581_b200.dart import DeviceRadixCache

    obs, run = G.run_engine_case(case, DeviceRadixCache, sched, admit="wave")
    G.assert_engine_parity(obs, run)
