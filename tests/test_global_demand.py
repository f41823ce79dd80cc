"""C5: eviction stress with the per-window all-reduce of the replicas' demand
counters feeding P-hat (the global-demand knob).

Two replicas (world size 2, gloo for the collective, both on cuda:0) each run
their shard of one C4-shaped stream through the fused device wave at a KV
budget far below the working set; every window the pending demand is counted
on the device and all-reduced, and the protection hand-off uses the summed
counters.  The oracle runs both shards' replicas in lockstep with the same
summed counters (oracle/windows.py oracle_windows_global); each device replica
must match its oracle replica exactly: dispatch order, hits, leaf ids, every
victim and the final tree.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from traces import synth as S

pytestmark = pytest.mark.gpu

WORLD, WAVES, POOL, CAP = 2, 8, 192, 60_000


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _configs():
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig

    return (CacheConfig(capacity_tokens=CAP, policy=CachePolicy.DART, protect_budget=16),
            SchedulerConfig(dispatch_budget=POOL, cold_quota=8))


def _windows(rank):
    st = S.ShardStream("c4", 17, WORLD, rank, chunk=4096)
    return [st.take(POOL) for _ in range(WAVES)]


def _worker(rank, port, out, use_global):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from oracle.windows import device_table, device_victims, device_windows
    from paper_2605_08581_b200.wave import WaveEngine

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cache, sched = _configs()
    eng = WaveEngine(cache, sched, S.C4.nseg, S.C4.sys_len, S.C4.chunk, device=0)

    def reduce(G):
        h = G.cpu()
        dist.all_reduce(h)
        G.copy_(h.to(dev))

    d = device_windows(eng, _windows(rank), dev, reduce_demand=reduce if use_global else None)
    out[rank] = {k: (np.asarray(v).tolist() if not isinstance(v, dict) else v) for k, v in d.items()
                 if k != "stats"}
    eng.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("use_global", [True, False])
def test_two_replicas_global_demand(use_global):
    from oracle.oracle import build
    from oracle.windows import OracleReplica, oracle_windows, oracle_windows_global

    build()
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(port, out, use_global), nprocs=WORLD, join=True)
        res = dict(out)
    cache, sched = _configs()
    wins = [_windows(r) for r in range(WORLD)]
    for r in range(WORLD):
        if use_global:
            reps = [OracleReplica(cache, sched, S.C4.nseg, S.C4.sys_len, S.C4.chunk) for _ in range(WORLD)]
            o = oracle_windows_global(reps, wins, record_rank=r)
        else:
            o = oracle_windows(OracleReplica(cache, sched, S.C4.nseg, S.C4.sys_len, S.C4.chunk), wins[r])
        d = res[r]
        for j in range(WAVES):
            assert d[f"m{j}"] == o[f"m{j}"].tolist(), (r, j, "dispatch")
            assert d[f"h{j}"] == o[f"h{j}"].tolist(), (r, j, "hits")
            assert d[f"l{j}"] == o[f"l{j}"].tolist(), (r, j, "leaves")
        assert d["vfirst"] == 0 and d["victims"] == o["victims"].tolist(), r
        assert len(d["victims"]) > 1000  # eviction stress: the budget turns over every window
        assert d["table"] == o["table"].tolist(), r
