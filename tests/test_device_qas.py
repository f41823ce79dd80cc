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


def test_golden_rounds():
    for i, case in enumerate(G.load("qas_rounds.json.gz")):
        pending, active, cfg = G.qas_case(case)
        try:
            G.assert_qas_case(case, sched(pending, active, cfg))
        except AssertionError as e:
            raise AssertionError(f"round {i}: {e}") from e


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
