"""Windowed oracle parity of the fused device wave at benchmark shapes.

The device replica (``WaveEngine.step``: QAS round -> protection ->
serialization -> match/insert/evict, CUDA graph, exact parallel commit) and
the CPU oracle replica (oracle/windows.py, pinned to the reference on CPU by
tests/test_oracle_windows.py) run the same arrival windows; requests that a
CapacityError stops stay pending.  Compared: dispatch order, hits and leaf
ids of every recorded window, every eviction victim, the whole final tree
(node ids, parents, edge lengths, kinds, segments, ref counts, recency, hit
counts, protection, anchors, first tokens) and the resident token count.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle.windows import OracleReplica, compare_windows, device_windows, oracle_windows
from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig
from traces import synth as S

pytestmark = pytest.mark.gpu


def _windows(workload, seed, sizes, suffix_div=1):
    st = S.ShardStream(workload, seed, 1, 0)
    out = []
    for n in sizes:
        p = st.take(n)
        if suffix_div > 1:
            p["suffix"] = (p["suffix"] // suffix_div).astype(np.int32)
        out.append(p)
    return out


def _run(workload, windows, record_from, capacity, wave, policy=CachePolicy.DART, protect=20, cold=64,
         tune=None, graph=True):
    import torch

    from paper_2605_08581_b200.wave import WaveEngine

    spec = S.SPECS[workload]
    cfg = CacheConfig(capacity_tokens=capacity, policy=policy, protect_budget=protect)
    sched = SchedulerConfig(dispatch_budget=wave, cold_quota=cold)
    eng = WaveEngine(cfg, sched, spec.nseg, spec.sys_len, spec.chunk, device=0)
    if tune:
        eng.tune(**tune)
    eng.set_graph(graph)
    d = device_windows(eng, windows, torch.device("cuda", 0), record_from)
    eng.close()
    o = oracle_windows(OracleReplica(cfg, sched, spec.nseg, spec.sys_len, spec.chunk), windows, record_from)
    v = compare_windows(d, o, len(windows) - record_from, spec.path_len)
    assert v["identical"], v
    return v, d


def test_c3_1_64_scale_wave_4096():
    """C3 at 1/64 of the benchmark capacity with M = 4096: every window
    stops on a CapacityError, the rest stays pending (P grows past 4096)."""
    wins = _windows("c3", 5, [4096] * 6)
    v, d = _run("c3", wins, 0, 36_000_000 // 64, 4096)
    assert v["decisions_checked"] > 1000 and v["victims_checked"] > 10_000
    assert any(len(d[f"l{j}"]) < len(d[f"m{j}"]) for j in range(6))


def test_c3_steady_state_windows():
    """C3 at 1/8 scale: warm start to capacity, then evicting windows of 1024."""
    wins = _windows("c3", 6, [1024] * 6 + [1024] * 3)
    v, _ = _run("c3", wins, 6, 36_000_000 // 8, 1024)
    assert v["tree_nodes_checked"] > 50_000 and v["decisions_checked"] == 3 * 1024


def test_mu1m_eighth_scale_wave_4096():
    """mu1M at 1/8 scale (125K/8 warm paths, capacity 2M) with waves of 4096."""
    wins = _windows("mu1m", 7, [4096] * 4 + [4096] * 2)
    v, _ = _run("mu1m", wins, 4, 2_000_000, 4096)
    assert v["decisions_checked"] == 2 * 4096 and v["victims_checked"] > 5000


@pytest.mark.parametrize("policy", [CachePolicy.LRU, CachePolicy.LFU, CachePolicy.LRU_ACTIVE])
def test_c4_policies(policy):
    wins = _windows("c4", 8, [1024] * 6, suffix_div=4)
    _run("c4", wins, 0, 400_000, 1024, policy=policy, cold=16)


def test_c3_plain_launches_and_tiny_prefixes():
    """The same windows without the CUDA graph and with minimal eviction-order prefixes."""
    wins = _windows("c3", 9, [512] * 8)
    _run("c3", wins, 0, 36_000_000 // 128, 512, graph=False,
         tune=dict(list_min_tokens=1, list_slack_tokens=0, sel_min_candidates=0))
