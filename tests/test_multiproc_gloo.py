"""N>1 host-side logic on CPU: world-size-2 gloo process groups.

Covers the replica routing (segment-hash shards partition the trace, stable
per request), the per-window demand-counter all-reduce that bench.py issues
over NCCL on GPUs, and max-over-ranks timing.  The replicas' trees are
independent, so the sharded oracle runs must equal running the oracle on each
sub-trace alone.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08581_b200.shard import max_over_ranks, route, shard_requests
from paper_2605_08581_b200.types import SegmentCatalog
from traces.refgen import WorkloadConfig, generate_trace


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _trace():
    cat = SegmentCatalog(num_segments=200, chunk_tokens=8, hot_set=tuple(range(10)), sys_prefix_tokens=4)
    return generate_trace(WorkloadConfig(qps=40.0, num_requests=300, k=3, r_hot=0.7, zipf_alpha=1.2,
                                         suffix_tokens=4, seed=9), cat)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = _trace()
    mine = shard_requests(tr.requests, world, rank)
    # per-window demand counters of this replica, all-reduced
    counts = torch.zeros(200, dtype=torch.int32)
    for r in mine:
        for s in set(r.skeleton):
            counts[s] += 1
    local = counts.clone()
    dist.all_reduce(counts)
    t = max_over_ranks(float(rank + 1))
    # sharded oracle run on this replica's sub-trace
    from oracle.oracle import OracleRadixCache, oracle_schedule_round
    from sim_harness import SimConfig, run_simulation
    from paper_2605_08581_b200.types import CacheConfig, SchedulerConfig, Trace

    cfg = SimConfig(prefill_rate=5000.0, decode_rate=20000.0, cache=CacheConfig(capacity_tokens=600, protect_budget=4),
                    scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=8, cold_quota=2))
    res = run_simulation(Trace(tr.catalog, mine), cfg, cache_factory=OracleRadixCache,
                         schedule_fn=oracle_schedule_round)
    out[rank] = {"ids": [r.id for r in mine], "local": local.tolist(), "sum": counts.tolist(), "max": t,
                 "hits": [m.hit_tokens for m in res.requests]}
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    tr = _trace()
    ids0, ids1 = res[0]["ids"], res[1]["ids"]
    assert sorted(ids0 + ids1) == [r.id for r in tr.requests]  # a partition
    assert not set(ids0) & set(ids1)
    exp = np.array(res[0]["local"]) + np.array(res[1]["local"])
    assert res[0]["sum"] == exp.tolist() == res[1]["sum"]
    assert res[0]["max"] == res[1]["max"] == 2.0
    # each replica equals the oracle run on its own sub-trace alone
    from oracle.oracle import OracleRadixCache, oracle_schedule_round
    from sim_harness import SimConfig, run_simulation
    from paper_2605_08581_b200.types import CacheConfig, SchedulerConfig, Trace

    cfg = SimConfig(prefill_rate=5000.0, decode_rate=20000.0, cache=CacheConfig(capacity_tokens=600, protect_budget=4),
                    scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=8, cold_quota=2))
    for rank in range(world):
        sub = shard_requests(tr.requests, world, rank)
        alone = run_simulation(Trace(tr.catalog, sub), cfg, cache_factory=OracleRadixCache,
                               schedule_fn=oracle_schedule_round)
        assert [m.hit_tokens for m in alone.requests] == res[rank]["hits"]


def test_route_is_stable_and_balanced():
    segs = np.arange(100_000)
    for world in (2, 4, 8):
        sh = route(segs, world)
        assert sh.min() == 0 and sh.max() == world - 1
        frac = np.bincount(sh, minlength=world) / len(segs)
        assert np.all(np.abs(frac - 1 / world) < 0.01)
        assert np.array_equal(sh, route(segs, world))
