#!/usr/bin/env python
"""bench.py -- PRISM scheduling-memory hot path (QAS + DART) on B200.

Metric (BASELINE.json): prefix-match+admit+evict decisions/sec at a ~1M-node
DART tree.  One *decision* = one admitted request: its exact-prefix match and
its insert including _reserve/evict, with the wave's QAS round and
protection pass amortised.

Workloads (traces/synth.py); ``--workload``:
  c3   (default) the agent / tool-output trace: 40 segments of 32 tokens after
       a 1024-token system prompt plus a 128-token private suffix (2432-token
       paths), Zipf(1.1)-skewed 24-level segment chains, reorderable=false;
       capacity sized so the steady-state tree holds ~1M nodes.
  mu1m the 1M-node micro-benchmark (8 x 16-token segments, uniform).
  c4   the RAG generator's shape at 100K segments (the sharded 10M trace).
A *step* is one serving-loop wave (engine.py:189-213) per replica: device QAS
round -> protection hand-off -> serialization -> ordered match+insert+evict
-> release of the previous wave's pins.  Synthetic data, deterministic seeds.

Multi-GPU: one replica tree per GPU; requests of ONE global stream are routed
to replicas by splitmix64(skeleton[0]) mod N; each replica's
wave takes the next M requests of its shard (weak scaling); one NCCL
all-reduce of the per-window demand counters per step.  ``--gpus N`` without
torchrun re-launches itself under torch.distributed.run.

Parity (``cpu_baseline`` leg, N=1, rank 0): the CPU oracle (oracle/, the
reference algorithm restated in C and pinned to the reference's own outputs)
runs the same warm start and ``--parity-waves`` evicting windows as a fresh
device replica, in a background process started before CUDA is touched; the
line reports whether dispatch order, hits, leaf ids, every victim and the whole
final tree are identical, and times the oracle on those windows.

    python bench.py [--gpus N --steps K --warmup W --workload c3|mu1m|c4]
    python bench.py --impl reference ...     # the reference algorithm on host cores

Prints exactly one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from traces import synth as S  # noqa: E402

METRIC = "prefix-match+admit+evict decisions/sec @1M-node DART; hit-rate parity; HBM GB/s"
UNIT = "decisions/s"

# per-workload defaults: requests in the warm start, capacity (tokens), wave size
DEFAULTS = {
    "c2": {"warm": 0, "capacity": 5760, "wave": 8},  # serve mode only (--mode serve): the QPS sweep
    "c3": {"warm": 8 * 4096, "capacity": 36_000_000, "wave": 4096},
    "mu1m": {"warm": 125_000, "capacity": 16_000_000, "wave": 4096},
    "c4": {"warm": 16 * 1024, "capacity": 4_000_000, "wave": 1024},
    # C5: the C4 shape at a KV budget of 10% of the 12.8M-token segment catalog
    # per replica, the replicas' per-window demand all-reduced into P-hat
    "c5": {"warm": 4 * 1024, "capacity": 1_280_000, "wave": 1024},
}
DESCR = {
    "c3": "C3 agent trace: 2432-token paths (sys 1024 + 40 x 32-token segments + 128-token suffix), Zipf(1.1) "
          "24-level segment chains over a 2^20 catalog, reorderable=false; DART tree warm-started to capacity "
          "(~1M nodes), every wave evicts",
    "mu1m": "mu1M: 172-token paths (sys 28 + 8 x 16 + 16), slot 0 uniform over 50, others over 2M; DART tree "
            "warm-started with 125K paths (~1M nodes, ~16M tokens), every admission evicts",
    "c4": "C4 RAG shape: 768-token paths (sys 28 + 5 x 128 + 100), 100K-segment catalog, Zipf(1.1) over 1000 hot, "
          "r_hot 0.7",
    "c5": "C5 eviction stress: the C4 shape at a per-replica KV budget of 1.28M tokens (10% of the 12.8M-token "
          "segment catalog), every wave turns most of the tree over; per window the replicas' pending demand is "
          "all-reduced and feeds P-hat (global-demand knob)",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(DEFAULTS))
    ap.add_argument("--wave", type=int, default=0)
    ap.add_argument("--warm", type=int, default=-1, help="warm-start requests per replica")
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--protect", type=int, default=20)
    ap.add_argument("--cold-quota", type=int, default=64)
    ap.add_argument("--parity-waves", type=int, default=-1,
                    help="evicting windows checked against the CPU oracle (default 2 at N=1, 0 at N>1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=-1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--same-device", action="store_true", help="all ranks on cuda:0 (tests on one GPU)")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no baseline/e2e/parity)")
    ap.add_argument("--profile-steps", type=int, default=3,
                    help="extra waves AFTER the timed region with the per-phase device profile on (roofline)")
    ap.add_argument("--ref-seconds", type=float, default=0.5, help="reference arm: seconds per step per worker")
    ap.add_argument("--kv-bytes", type=int, default=0,
                    help="wave mode: attach a paged KV payload of this many bytes per token (copy-in of the new "
                         "tokens, copy-out of the victims, req_to_token tables inside every timed step)")
    ap.add_argument("--mode", default="wave", choices=["wave", "serve"],
                    help="wave: timed fused waves on a warm tree; serve: the whole serving loop over a trace")
    ap.add_argument("--requests", type=int, default=10_000_000, help="serve mode: requests in the global trace")
    ap.add_argument("--qps", type=float, default=20000.0, help="serve mode: global arrival rate")
    ap.add_argument("--total-capacity", type=int, default=16_000_000,
                    help="serve mode: KV capacity (tokens) of the whole job, split evenly over the replicas")
    ap.add_argument("--parity-requests", type=int, default=60000, help="serve mode: per-shard parity prefix")
    a = ap.parse_args()
    d = DEFAULTS[a.workload]
    a.wave = a.wave or d["wave"]
    a.capacity = a.capacity or d["capacity"]
    a.warm = d["warm"] if a.warm < 0 else a.warm
    return a


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _configs(args):
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig

    return (CacheConfig(capacity_tokens=args.capacity, policy=CachePolicy.DART, protect_budget=args.protect),
            SchedulerConfig(dispatch_budget=args.wave, cold_quota=args.cold_quota))


# ---------------------------------------------------------------- clocks


class Clocks:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        if os.environ.get("PRISM_BENCH_NO_CLOCKS"):  # (diagnostics only: the bench line then has no clocks)
            self.proc = None
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- oracle legs (checker / CPU baseline)


def parity_windows(args, world: int, rank: int):
    """The windows both sides of the parity check run: the warm start (to
    capacity) then ``--parity-waves`` evicting windows, from a dedicated
    stream of this replica's shard."""
    st = S.ShardStream(args.workload, args.seed + 7_777, world, rank)
    warm = [st.take(min(args.wave, args.warm - i)) for i in range(0, args.warm, args.wave)]
    check = [st.take(args.wave) for _ in range(args.parity_waves)]
    return warm, check


def oracle_parity_job(args, world: int, rank: int, out_path: str) -> None:
    """Background process: the oracle replica through the parity windows."""
    from oracle.oracle import build
    from oracle.windows import OracleReplica, oracle_windows

    build()
    cache, sched = _configs(args)
    spec = S.SPECS[args.workload]
    rep = OracleReplica(cache, sched, spec.nseg, spec.sys_len, spec.chunk)
    warm, check = parity_windows(args, world, rank)
    t0 = time.perf_counter()
    if args.workload == "c5":  # every replica in lockstep, P-hat from the summed demand
        from oracle.windows import oracle_windows_global

        reps = [rep if r == rank else OracleReplica(cache, sched, spec.nseg, spec.sys_len, spec.chunk)
                for r in range(world)]
        wins = [(lambda w, c: w + c)(*parity_windows(args, world, r)) for r in range(world)]
        res = oracle_windows_global(reps, wins, rank, record_from=len(warm))
    else:
        res = oracle_windows(rep, warm + check, record_from=len(warm))
    res["timing"] = np.append(res["timing"], time.perf_counter() - t0)
    np.savez(out_path, **res)


def _kv_line(acc: dict, args, peak: float) -> dict:
    """The paged KV payload's share of the timed steps: copy-in of the new tokens' KV,
    copy-out of the victims' KV (each read once + written once), req_to_token tables."""
    w = max(acc["waves"], 1)
    moved = 2 * (acc["new"] + acc["freed"]) * args.kv_bytes + acc["table_bytes"]
    gbs = moved / max(acc["ms"], 1e-9) / 1e6
    return {"bytes_per_token": args.kv_bytes, "ms_per_wave": acc["ms"] / w, "new_tokens_per_wave": acc["new"] / w,
            "freed_tokens_per_wave": acc["freed"] / w, "bytes_per_wave": moved / w, "achieved_gbs": gbs,
            "peak_gbs": peak, "frac": gbs / peak,
            "note": "prism_kv_sync (row alloc + copy-in of the new tokens' KV, victim copy-out + free-stack "
                    "push; device-driven, no host wait) + req_to_token gather; bytes = each copied row read once "
                    "and written once + the tables"}


def _demand_reducer(args, world: int, dev):
    """In-place sum of a demand vector over the replicas (NCCL over NVLink; gloo via the host)."""
    import torch.distributed as dist

    def reduce(G):
        if world == 1:
            return
        if args.backend == "nccl":
            dist.all_reduce(G)
        else:
            h = G.cpu()
            dist.all_reduce(h)
            G.copy_(h.to(dev))

    return reduce


def kv_leg(args, engine_kw, world: int, rank: int, dev, peak: float, bpt: int = 256, waves: int = 6) -> dict:
    """The paged KV payload measured beside the headline (north_star item 4):
    a fresh replica with a pool row of ``bpt`` bytes per resident token, warm-
    started to capacity, then ``waves`` waves each followed by the device-
    driven payload sync (copy-in of the new tokens' KV, copy-out of the
    victims' KV, free stack) and the req_to_token tables; the payload's own
    CUDA events on the pool's stream give its HBM throughput."""
    import torch

    from paper_2605_08581_b200.kv import KvPool
    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    spec = S.SPECS[args.workload]
    B = args.wave
    eng = WaveEngine(**engine_kw)
    max_new = B * spec.path_len
    kv = KvPool(eng.t, args.capacity + 2 * max_new, bpt)
    src = torch.randint(0, 255, (max_new, bpt), dtype=torch.uint8, device=dev)
    dst = torch.empty((args.capacity, bpt), dtype=torch.uint8, device=dev)
    st = S.ShardStream(args.workload, args.seed + 99, world, rank)
    tst = torch.cuda.ExternalStream(eng.L.prism_tree_stream(eng.t), device=dev)
    prev, evs, tb, k0s = 0, [], 0, None
    nwarm = (args.warm + B - 1) // B
    for w in range(nwarm + 2 + waves):
        p = st.take(B)
        _, prev = eng.step(DevicePending.from_host(p["ids"], p["arrival"], p["sk_off"], p["sk"], p["reorderable"],
                                                   p["suffix"], dev), release_n=prev)
        timed = w >= nwarm + 2
        if timed and k0s is None:
            torch.cuda.synchronize()
            k0s = kv.stats()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(tst)
        kv.sync(src, dst, counts=False)
        kv.gather(eng.leaf_slots, prev, spec.path_len, wait=False)
        b.record(tst)
        eng.stream.wait_event(b)
        if timed:
            evs.append((a, b))
            tb += prev * spec.path_len * 4
    torch.cuda.synchronize()
    k1 = kv.stats()
    eng.close()
    acc = {"ms": sum(a.elapsed_time(b) for a, b in evs), "new": k1["allocated"] - k0s["allocated"],
           "freed": k1["freed"] - k0s["freed"], "table_bytes": tb, "waves": waves}
    ns = argparse.Namespace(kv_bytes=bpt)
    out = _kv_line(acc, ns, peak)
    out["note"] = (f"measured beside the headline on a fresh replica ({waves} evicting waves after the warm start): "
                   + out["note"])
    return out


def device_parity(args, engine_kw, world: int, rank: int, dev) -> dict:
    """A fresh device replica through the same windows."""
    from oracle.windows import device_windows
    from paper_2605_08581_b200.wave import WaveEngine

    eng = WaveEngine(**engine_kw)
    warm, check = parity_windows(args, world, rank)
    out = device_windows(eng, warm + check, dev, record_from=len(warm),
                         reduce_demand=_demand_reducer(args, world, dev) if args.workload == "c5" else None)
    eng.close()
    return out


# ---------------------------------------------------------------- reference arm


def _ref_worker(job):
    args, world, rank, seconds = job
    from oracle.windows import OracleReplica, concat_pools, drop_members

    cache, sched = _configs(args)
    spec = S.SPECS[args.workload]
    rep = OracleReplica(cache, sched, spec.nseg, spec.sys_len, spec.chunk)
    st = S.ShardStream(args.workload, args.seed + 31 * rank + 1, world, rank)
    pend = None
    for i in range(0, args.warm, args.wave):  # warm start (untimed)
        pend = concat_pools(pend, st.take(min(args.wave, args.warm - i)))
        r = rep.step(pend)
        pend = drop_members(pend, r["members"][: r["n_admitted"]])
    rep.decisions, rep.decision_seconds = 0, 0.0
    deadline = time.perf_counter() + seconds
    while time.perf_counter() < deadline:
        pend = concat_pools(pend, st.take(args.wave))
        r = rep.step(pend, deadline=deadline)
        pend = drop_members(pend, r["members"][: r["n_admitted"]])
    return {"decisions": rep.decisions, "seconds": rep.decision_seconds}


def run_reference(args) -> None:
    if int(os.environ.get("RANK", "0")) != 0:
        return  # rank 0 alone runs and prints the host-core baseline
    import multiprocessing as mp

    from oracle import oracle as O

    O.build()
    cores = max(1, min(len(os.sched_getaffinity(0)), 32))
    seconds = max(args.steps, 1) * args.ref_seconds
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_ref_worker, [(args, cores, w, seconds) for w in range(cores)])
    value = sum(r["decisions"] / max(r["seconds"], 1e-9) for r in res)
    decisions = sum(r["decisions"] for r in res)
    secs = max(r["seconds"] for r in res)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": DESCR[args.workload], "wave": args.wave, "capacity_tokens": args.capacity,
                   "warm_requests": args.warm, "policy": "DART"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{decisions} decisions: {cores} replica processes (one per host core, each a "
                                   f"segment-hash shard of one global stream), each warm-started to capacity and "
                                   f"then timed for {seconds:.1f}s of evicting windows (oracle/: C restatement of "
                                   f"kvcache.py/scheduler.py, full scan + heap per evict, pinned to the "
                                   f"reference's outputs; the Python reference itself is ~100x slower)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm


def run_ours(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec = S.SPECS[args.workload]
    if args.parity_waves < 0:  # C5's parity (the summed demand) is checked at every N; the others at N=1
        args.parity_waves = 2 if (world == 1 or args.workload == "c5") else 0
    if args.profile_only:
        args.parity_waves = 0
    # the oracle parity replica starts BEFORE CUDA is initialised (fork-safe)
    par_proc = par_path = None
    if args.parity_waves > 0 and not args.no_cpu_baseline:
        import multiprocessing as mp

        fd, par_path = tempfile.mkstemp(suffix=".npz")
        os.close(fd)
        par_proc = mp.get_context("fork").Process(target=oracle_parity_job, args=(args, world, rank, par_path))
        par_proc.start()

    import torch
    import torch.distributed as dist

    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    if world > 1:
        dist.init_process_group(args.backend)
    gpu = 0 if args.same_device else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    B = args.wave
    cache, sched = _configs(args)
    engine_kw = dict(cache=cache, sched=sched, nseg=spec.nseg, sys_len=spec.sys_len, chunk=spec.chunk, device=gpu,
                     initial_slots=1 << 21, initial_arena_tokens=max(1 << 26, 32 * args.capacity))
    engine = WaveEngine(**engine_kw)
    stream = engine.stream
    stream_in = S.ShardStream(args.workload, args.seed, world, rank)
    demand = torch.zeros(spec.nseg, dtype=torch.int32, device=dev) if world > 1 else None

    kv = None
    if args.kv_bytes > 0:  # the paged KV payload (kv.cuh): a pool row per resident token
        from paper_2605_08581_b200.kv import KvPool

        max_new = B * spec.path_len
        kv = KvPool(engine.t, args.capacity + 2 * max_new, args.kv_bytes)
        kv_src = torch.randint(0, 255, (max_new, args.kv_bytes), dtype=torch.uint8, device=dev)  # the prefill's KV
        kv_dst = torch.empty((args.capacity, args.kv_bytes), dtype=torch.uint8, device=dev)  # the offload tier
        kv_acc = {"ms": 0.0, "new": 0, "freed": 0, "table_bytes": 0, "waves": 0, "events": []}

    def kv_step(na, timed):
        if kv is None:
            return
        tst = torch.cuda.ExternalStream(engine.L.prism_tree_stream(engine.t), device=dev)  # (the pool's stream)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(tst)
        kv.sync(kv_src, kv_dst, counts=False)  # device-driven: no host wait
        kv.gather(engine.leaf_slots, na, spec.path_len, wait=False)
        k1.record(tst)
        stream.wait_event(k1)  # the next wave follows the payload work
        if timed:
            kv_acc["events"].append((k0, k1))
            kv_acc["table_bytes"] += na * spec.path_len * 4
            kv_acc["waves"] += 1

    glob = args.workload == "c5"
    if glob:  # the global-demand knob: P-hat from the replicas' summed per-window demand
        demand = torch.zeros(spec.nseg, dtype=torch.int32, device=dev)
        engine.set_global_demand(demand)
    reduce_demand = _demand_reducer(args, world, dev)

    def pre_step(pend):
        if glob:  # this window's demand, summed over the replicas before the wave's hand-off
            with torch.cuda.stream(stream):
                engine.demand(pend, demand)
                reduce_demand(demand)

    def allreduce_demand():
        if demand is None or glob:
            return
        with torch.cuda.stream(stream):  # per-window demand counters across replicas (NVLink)
            engine.demand_counters(demand)
            if args.backend == "nccl":
                dist.all_reduce(demand)
            else:
                h = demand.cpu()
                dist.all_reduce(h)
                demand.copy_(h)

    def to_dev(pool):
        return DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"],
                                       pool["reorderable"], pool["suffix"], dev)

    # warm start (untimed): the tree through the same fused path, to capacity
    prev = 0
    t_ws = time.perf_counter()
    for i in range(0, args.warm, B):
        engine.release(engine.leaf_slots, prev)
        wp = to_dev(stream_in.take(min(B, args.warm - i)))
        pre_step(wp)
        _, prev = engine.step(wp)
        kv_step(prev, False)
    torch.cuda.synchronize()
    warm_s = time.perf_counter() - t_ws

    nsteps = args.warmup + args.steps
    nprof = max(args.profile_steps, 1)
    dpools = [to_dev(stream_in.take(B)) for _ in range(nsteps + nprof)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    hitsum = torch.zeros(1, dtype=torch.int64, device=dev)

    timed_now = [False]

    def one_step(pend):
        nonlocal prev
        pre_step(pend)
        nm, na = engine.step(pend, release_n=prev)  # the previous wave's pins drop inside the wave
        kv_step(na, timed_now[0])
        allreduce_demand()
        prev = na
        return nm, na

    for s in range(args.warmup):
        one_step(dpools[s])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof0 = engine.profile_read()
    st1 = engine.stats()
    cmp0 = engine.compactions()
    clocks = Clocks(gpu)
    clocks.start()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" scopes profiles here
    evs = []
    admitted = members = 0
    timed_now[0] = True
    kv0 = kv.stats() if kv is not None else None
    trace_take(engine)  # (diagnostics builds only: the ring starts empty at the timed region)
    for s in range(args.warmup, nsteps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nm, na = one_step(dpools[s])
        e1.record(stream)
        evs.append((e0, e1))
        with torch.cuda.stream(stream):  # outside the events: the hit-rate numerator
            hitsum.add_(engine.hits[:na].sum())
        admitted += na
        members += nm
    torch.cuda.synchronize()
    timed_now[0] = False
    if os.environ.get("PRISM_TRACE_OUT"):
        with open(os.environ["PRISM_TRACE_OUT"], "w") as f:
            json.dump(trace_take(engine), f)
    if kv is not None:  # the payload's share of the timed steps (its own events, on the pool's stream)
        kv1 = kv.stats()
        kv_acc["ms"] = sum(a.elapsed_time(b) for a, b in kv_acc["events"])
        kv_acc["new"] = kv1["allocated"] - kv0["allocated"]
        kv_acc["freed"] = kv1["freed"] - kv0["freed"]
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    prof1 = engine.profile_read()
    st2 = engine.stats()
    cmp1 = engine.compactions()
    per_step = [a.elapsed_time(b) for a, b in evs]
    ms = sum(per_step)
    hit_tokens = int(hitsum.item())
    hit_rate = hit_tokens / max(admitted * spec.path_len, 1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([admitted], dtype=torch.int64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(c)
        admitted_all = int(c.item())
    else:
        admitted_all = admitted
    value = admitted_all / (ms / 1000.0)

    # ---- e2e: host pinned inputs, H2D + step + D2H of results inside the timed region
    e2e_steps = args.steps if args.e2e_steps < 0 else args.e2e_steps
    e2e = None
    if e2e_steps > 0 and not args.profile_only:
        ew = max(args.warmup, 3)  # untimed: the first waves of the host-buffer shape capture its graph
        hpools = [stream_in.take(B) for _ in range(e2e_steps + ew)]
        pinned = [{k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in p.items()} for p in hpools]
        out_mem = np.empty(B, dtype=np.int64)
        out_hits = np.empty(B, dtype=np.int64)
        h2d = sum(v.numel() * v.element_size() for v in pinned[0].values())
        for s in range(ew):
            pre_step(pinned[e2e_steps + s])
            _, prev = engine.step_host(pinned[e2e_steps + s], out_mem, out_hits, release_n=prev)
            kv_step(prev, False)
            allreduce_demand()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        adm2 = d2h = 0
        wall = []
        for s in range(e2e_steps):
            tw = time.perf_counter()
            pre_step(pinned[s])
            nm, na = engine.step_host(pinned[s], out_mem, out_hits, release_n=prev)
            kv_step(na, False)
            wall.append((time.perf_counter() - tw) * 1e3)
            prev = na
            allreduce_demand()
            d2h += 8 * (na + nm)
            adm2 += na
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms2], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2 = float(t.item())
            c = torch.tensor([adm2], dtype=torch.int64, device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(c)
            adm2 = int(c.item())
        e2e = {"value": adm2 / (ms2 / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h // e2e_steps, "api": "prism_wave_step_host via WaveEngine.step_host "
               "(pinned host pending arrays read in place by the wave's staging kernel; admission order + hits "
               "copied to host inside the wave; the previous wave's pins released by the same call)",
               "host_ms_per_call": {"median": round(statistics.median(wall), 4), "max": round(max(wall), 4)}}

    # ---- roofline of the dominant phase: a few more waves AFTER the timed
    # region with the live per-phase profile on (its per-phase event syncs
    # would otherwise sit inside the timed region)
    gpu_launches = int(sum(prof1[p]["launches"] - prof0[p]["launches"]
                           for p in ("commit", "build", "protect", "prematch", "release", "qas")))
    torch.cuda.synchronize()
    engine.profile(True)
    prof2 = engine.profile_read()
    st3 = engine.stats()
    for s in range(nsteps, nsteps + nprof):
        one_step(dpools[s])
    torch.cuda.synchronize()
    prof3 = engine.profile_read()
    st4 = engine.stats()
    engine.profile(False)
    phases = ("commit", "build", "protect", "prematch", "release", "qas")
    d = {p: {k: prof3[p][k] - prof2[p][k] for k in ("ms", "calls", "launches")} for p in phases}
    victims = st4["victims"] - st3["victims"]
    created = st4["next_id"] - st3["next_id"]
    chain = prof3["chain_nodes"] - prof2["chain_nodes"]
    toks = prof3["inserted_tokens"] - prof2["inserted_tokens"]
    live = st4["live_nodes"]
    anchors = engine.reusable_anchors()
    members_prof = nprof * B
    algo = {  # SURVEY.md 8(d) algorithmic bytes over the profiled waves: per request 8l + 32(d + c + v)
        "prematch": 4 * toks + 32 * chain,              # read the query + the matched resident chain
        "commit": 4 * toks + 32 * (created + victims),  # write the new tokens + created / victim records
        "build": 16 * live * min(d["build"]["calls"], nprof),       # eviction-key scan, <= once per wave
        "protect": 16 * anchors * min(d["protect"]["calls"], nprof),  # protection scan over A anchors
        "qas": members_prof * (4 * spec.k + 16),
        "release": 0,
    }
    dom = max(("commit", "build", "protect", "prematch", "qas"), key=lambda p: d[p]["ms"])
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    peak = float(peaks.get("hbm_gbs", 7672.0))
    peak_src = ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks
                else "B200_PROFILING.md fallback")
    per_wave_bytes = algo[dom] / nprof
    per_wave_s = d[dom]["ms"] / 1000.0 / nprof
    achieved = per_wave_bytes / per_wave_s / 1e9 if per_wave_s > 0 else 0.0
    traffic = None
    summ = os.path.join(ROOT, "profiles", f"ncu_summary_{args.workload}.json")
    if os.path.exists(summ):
        try:
            traffic = json.load(open(summ)).get("phases", {}).get(dom, {}).get("dram_bytes_per_wave")
        except Exception:
            traffic = None
    wave_bytes = sum(algo.values()) / nprof
    step_ms = ms / max(args.steps, 1)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom,
                "launch": f"one wave's {dom} phase (its kernels back to back)", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": per_wave_bytes, "launch_ms": per_wave_s * 1000.0,
                "phase_ms_per_wave": {p: round(d[p]["ms"] / nprof, 4) for p in d}, "profiled_waves": nprof,
                "algorithmic_bytes_per_wave": {p: round(algo[p] / nprof) for p in algo},
                "wave": {"algorithmic_bytes": wave_bytes, "ms": step_ms,
                         "achieved_gbs": wave_bytes / (step_ms / 1000.0) / 1e9,
                         "frac": wave_bytes / (step_ms / 1000.0) / 1e9 / peak}}

    # ---- the paged KV payload beside the headline (its own replica; skipped when --kv-bytes ran it inline)
    kv_side = None
    if kv is None and not args.profile_only and args.workload in ("c3", "mu1m", "c5"):
        kv_side = kv_leg(args, engine_kw, world, rank, dev, peak)

    # ---- parity + CPU baseline (the oracle replica started at the top)
    cpu = parity = None
    if par_proc is not None:
        dres = device_parity(args, engine_kw, world, rank, dev)
        par_proc.join()
        if par_proc.exitcode == 0:
            o = np.load(par_path)
            from oracle.windows import compare_windows

            parity = compare_windows(dres, o, args.parity_waves, spec.path_len)
            ndec, secs, total_s = o["timing"].tolist()
            if rank == 0 and world == 1:
                cpu = {"value": ndec / max(secs, 1e-9), "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": f"{int(ndec)} decisions in {secs:.1f}s: the {args.parity_waves} evicting "
                                 f"{B}-request parity windows after a {args.warm}-request warm start to capacity "
                                 f"(oracle/: C restatement of kvcache.py/scheduler.py, full scan + heap per evict, "
                                 f"one thread; {total_s:.0f}s including the warm start)"}
        else:
            parity = {"waves_checked": 0, "identical": False, "differences": ["oracle process failed"]}
        os.unlink(par_path)
    if world > 1 and parity is not None:
        flag = torch.tensor([1 if parity["identical"] else 0], dtype=torch.int64,
                            device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        parity["identical_all_shards"] = bool(flag.item())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": DESCR[args.workload], "name": spec.name, "wave": B, "path_tokens": spec.path_len,
                "warm_requests": args.warm, "capacity_tokens": args.capacity, "policy": "DART",
                "protect_budget": args.protect, "cold_quota": args.cold_quota,
                "parallelism": f"replicas x{world} (splitmix64(skeleton[0]) mod {world} shards of one stream)",
                "l2": "flushed between timed steps (256 MiB write)",
                "tree_nodes": st2["live_nodes"], "resident_tokens": st2["resident"],
                "warm_start_s": round(warm_s, 2), "admitted_per_rank": admitted,
                "members_per_rank": members, "victims": st2["victims"] - st1["victims"],
                "fast_path_members": st2["fast_members"] - st1["fast_members"],
                "slow_path_members": st2["slow_members"] - st1["slow_members"],
                "profile": "per-phase device profile taken on extra waves after the timed region",
                "commit": engine.wave_stats(),
                "step_ms": {"min": round(min(per_step), 4), "median": round(statistics.median(per_step), 4),
                            "max": round(max(per_step), 4)},
                "arena_compactions_timed": cmp1 - cmp0,
                "arena_tokens": engine_kw["initial_arena_tokens"],
                "cuda_graph": engine.graph_stats(),
            },
            "hit_rate": hit_rate,
            "parity": parity,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "kv_payload": kv_side if kv is None else _kv_line(kv_acc, args, peak),
            "gpu_launches": gpu_launches,
            "lib_calls": prof1["lib_calls"] - prof0["lib_calls"],
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    engine.close()
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- serve mode (C4)


def _serve_config(args, world: int):
    """SimConfig (engine.py:35-48) of one replica: per-shard capacity = total / world,
    prefill rate sized so the shard keeps up (R_pf ~ 1.25 qps_shard L (1 - h))."""
    from types import SimpleNamespace

    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig

    spec = S.SPECS[args.workload]
    rate = 1.25 * (args.qps / world) * spec.path_len * 0.7
    return SimpleNamespace(prefill_rate=rate, decode_rate=1e6, output_tokens=32, decode_attenuation_enabled=False,
                           cache=CacheConfig(capacity_tokens=args.total_capacity // world, policy=CachePolicy.DART,
                                             protect_budget=args.protect),
                           scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=args.wave,
                                                     cold_quota=args.cold_quota))


def serve_oracle_job(args, world: int, rank: int, out_path: str) -> None:
    """Background process: the oracle serving loop on this shard's parity prefix."""
    from oracle.oracle import build
    from oracle.serve_loop import oracle_serve

    build()
    tr = S.prefix_trace(S.shard_trace(S.serve_trace(args.workload, args.requests, args.qps, args.seed), world, rank),
                        args.parity_requests)
    t0 = time.perf_counter()
    o = oracle_serve(tr, _serve_config(args, world))
    o["timing"] = np.array([o["decisions"], o["seconds"], time.perf_counter() - t0, tr.n])
    np.savez(out_path, **{k: v for k, v in o.items() if isinstance(v, np.ndarray)})


def run_serve(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    par_proc = par_path = None
    if args.parity_requests > 0 and not args.no_cpu_baseline:
        import multiprocessing as mp

        fd, par_path = tempfile.mkstemp(suffix=".npz")
        os.close(fd)
        par_proc = mp.get_context("fork").Process(target=serve_oracle_job, args=(args, world, rank, par_path))
        par_proc.start()
    import torch
    import torch.distributed as dist

    from paper_2605_08581_b200.serve import DeviceServingLoop

    if world > 1:
        dist.init_process_group(args.backend)
    gpu = 0 if args.same_device else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    t_gen = time.perf_counter()
    trace = S.serve_trace(args.workload, args.requests, args.qps, args.seed)  # every rank: the same global trace
    mine = S.shard_trace(trace, world, rank)
    gen_s = time.perf_counter() - t_gen
    cfg = _serve_config(args, world)
    kw = dict(device=gpu, initial_slots=1 << 20, initial_arena_tokens=max(1 << 24, 32 * cfg.cache.capacity_tokens))
    t0 = time.perf_counter()
    loop = DeviceServingLoop(cfg, mine, **kw)  # the trace's H2D copy (end-to-end)
    stream = torch.cuda.ExternalStream(loop.L.prism_qas_stream(loop.q), device=dev)
    loop.run(max_waves=args.warmup)  # untimed: the first waves (allocations, first captures)
    c0 = loop.counts()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(gpu)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw = time.perf_counter()
    e0.record(stream)
    loop.run()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - tw
    clk = clocks.stop()
    res = loop.result()  # the metrics' D2H copy (end-to-end)
    e2e_s = time.perf_counter() - t0
    c1 = loop.counts()
    ms = e0.elapsed_time(e1)
    admitted = c1["admitted"] - c0["admitted"]
    waves = c1["waves"] - c0["waves"]
    summ = res.summary()
    if world > 1:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = (float(x) for x in t.tolist())
        cnt = torch.tensor([admitted, mine.n], dtype=torch.int64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(cnt)
        admitted_all, n_all = (int(x) for x in cnt.tolist())
    else:
        admitted_all, n_all = admitted, mine.n
    loop.close()
    parity = cpu = None
    if par_proc is not None:
        from paper_2605_08581_b200.serve import DeviceServingLoop as DSL

        sub = S.prefix_trace(mine, args.parity_requests)
        pl = DSL(cfg, sub, **kw)
        pl.run()
        d = pl.result()
        dv = pl.cache_view().victim_log()
        pl.close()
        par_proc.join()
        if par_proc.exitcode == 0:
            o = np.load(par_path)
            diffs = []
            for name, a, b in (("hits", d.hit_tokens, o["hit"]), ("first_token", d.first_token, o["first_token"]),
                               ("completion", d.completion, o["completion"]), ("admit", d.admit, o["admit"]),
                               ("admission order", d.wave_members, o["wave_members"]),
                               ("wave durations", d.wave_duration, o["wave_duration"])):
                if not np.array_equal(np.asarray(a), np.asarray(b)):
                    diffs.append(name)
            if dv != o["victims"].tolist():
                diffs.append("victims")
            ndec, secs, tot, nreq = o["timing"].tolist()
            parity = {"requests_checked": int(nreq), "waves_checked": int(len(o["wave_launch"])),
                      "victims_checked": int(len(o["victims"])), "identical": not diffs, "differences": diffs,
                      "scope": "this shard's first requests through the whole serving loop (admission, hits, "
                               "TTFT / completion times, every victim)"}
            if rank == 0:
                cpu = {"value": ndec / max(secs, 1e-9), "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": f"{int(ndec)} decisions in {secs:.1f}s inside the waves of the oracle serving loop "
                                 f"over shard {rank}'s first {int(nreq)} requests ({tot:.0f}s in total)"}
        else:
            parity = {"identical": False, "differences": ["oracle process failed"]}
        os.unlink(par_path)
        if world > 1:
            flag = torch.tensor([1 if parity["identical"] else 0], dtype=torch.int64,
                                device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            parity["identical_all_shards"] = bool(flag.item())
    if rank == 0:
        spec = S.SPECS[args.workload]
        line = {
            "metric": METRIC, "value": admitted_all / (ms / 1000.0), "unit": UNIT, "n_gpus": world,
            "steps": waves, "warmup": args.warmup, "ms_per_step": ms / max(waves, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{spec.name} serving loop: {args.requests} requests "
                                   f"({DESCR.get(args.workload, '')}), Poisson arrivals at {args.qps:g} QPS, "
                                   f"routed by splitmix64(skeleton[0]) mod {world}; each replica replays its shard "
                                   f"through the device-resident run_simulation (windows of 50 ms, budget "
                                   f"{args.wave}, per-shard capacity {cfg.cache.capacity_tokens} tokens)",
                       "mode": "serve", "requests": args.requests, "requests_rank0": mine.n,
                       "requests_all": n_all, "qps": args.qps, "prefill_rate": cfg.prefill_rate,
                       "capacity_per_shard": cfg.cache.capacity_tokens, "wave_budget": args.wave,
                       "parallelism": f"replicas x{world}", "trace_gen_s": round(gen_s, 2),
                       "steps_are": "waves of the serving loop after the untimed warm-up waves, to the trace's end",
                       "windows": c1["windows"], "host_wall_s": round(wall, 3)},
            "hit_rate": summ["hit_rate"], "ttft_p50": summ["p50"], "ttft_p99": summ["p99"],
            "parity": parity, "roofline": None, "cpu_baseline": cpu,
            "e2e": {"value": admitted_all / e2e_s, "unit": UNIT, "h2d_bytes_per_step": mine.n * 41 // max(waves, 1),
                    "d2h_bytes_per_step": mine.n * 48 // max(waves, 1),
                    "api": "DeviceServingLoop (prism_serve_create / run / requests): the shard's trace copied in, "
                           "the per-request metrics copied out"},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_serve_c2(args) -> None:
    """C2: the reference's default RAG trace (WorkloadSpec:
    981 segments, chunk 128, 20 hot, k 5, r_hot 0.7, Zipf 1.2, 2048 requests,
    seed 1) at the 13B-model KV budget of 5760 tokens, QPS swept over
    {10, 15, 20, 25, 30}; the whole serving loop on the device per point, each
    point checked against the oracle serving loop (every request's hit / TTFT,
    the admission order, every victim)."""
    from types import SimpleNamespace

    import torch

    from oracle.oracle import build
    from oracle.serve_loop import oracle_serve
    from paper_2605_08581_b200.serve import DeviceServingLoop, TraceCSR
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig, SegmentCatalog
    from traces.refgen import WorkloadConfig, generate_trace

    build()
    torch.cuda.set_device(0)
    cat = SegmentCatalog(num_segments=981, chunk_tokens=128, hot_set=tuple(range(20)), sys_prefix_tokens=28)
    cfg = SimpleNamespace(prefill_rate=1e4, decode_rate=4e4, output_tokens=32, decode_attenuation_enabled=False,
                          cache=CacheConfig(capacity_tokens=5760, policy=CachePolicy.DART, protect_budget=20),
                          scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=8, cold_quota=2))
    points, adm_all, ms_all, ok_all, cpu_dec, cpu_s = [], 0, 0.0, True, 0, 0.0
    clocks = Clocks(0)
    clocks.start()
    for qps in (10.0, 15.0, 20.0, 25.0, 30.0):
        tr = TraceCSR.from_trace(generate_trace(WorkloadConfig(qps=qps, num_requests=2048, k=5, r_hot=0.7,
                                                               zipf_alpha=1.2, suffix_tokens=100, seed=1), cat))
        loop = DeviceServingLoop(cfg, tr)
        stream = torch.cuda.ExternalStream(loop.L.prism_qas_stream(loop.q), device=torch.device("cuda", 0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        loop.run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res = loop.result()
        victims = loop.cache_view().victim_log()
        loop.close()
        o = oracle_serve(tr, cfg)
        same = (np.array_equal(res.hit_tokens, o["hit"]) and np.array_equal(res.first_token, o["first_token"])
                and np.array_equal(res.wave_members, o["wave_members"]) and victims == o["victims"].tolist())
        ok_all &= same
        cpu_dec += o["decisions"]
        cpu_s += o["seconds"]
        sm = res.summary()
        points.append({"qps": qps, "decisions_per_s": tr.n / (ms / 1000.0), "ms": round(ms, 3),
                       "waves": int(len(res.wave_launch)), "hit_rate": sm["hit_rate"], "ttft_p50": sm["p50"],
                       "ttft_p99": sm["p99"], "victims": len(victims), "identical_to_oracle": bool(same)})
        adm_all += tr.n
        ms_all += ms
    clk = clocks.stop()
    line = {
        "metric": METRIC, "value": adm_all / (ms_all / 1000.0), "unit": UNIT, "n_gpus": 1,
        "steps": sum(p["waves"] for p in points), "warmup": 0, "ms_per_step": ms_all / max(sum(p["waves"] for p in points), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "C2: the reference default RAG trace (981 segments, chunk 128, 20 hot, k 5, r_hot 0.7, "
                               "Zipf 1.2, 2048 requests, seed 1) at the 13B-model KV budget (5760 tokens), QPS sweep "
                               "10..30, whole serving loop on the device (waves of <= 8)", "mode": "serve",
                   "sweep": points},
        "parity": {"identical": bool(ok_all), "scope": "every sweep point: per-request hits and TTFTs, admission "
                                                     "order, every victim vs the oracle serving loop"},
        "roofline": None,
        "cpu_baseline": {"value": cpu_dec / max(cpu_s, 1e-9), "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{cpu_dec} decisions in {cpu_s:.2f}s inside the oracle serving loop's waves, "
                                   f"all five sweep points"},
        "e2e": None, "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def trace_take(engine):
    """Kernel start stamps of a -DPRISM_TRACE diagnostics build (pdl.cuh), both
    units merged in time order; [] for the product build."""
    import ctypes as C

    out = []
    for unit in ("dart", "qas"):
        fn = getattr(getattr(engine, "L", None), f"prism_trace_dump_{unit}", None)
        if fn is None:
            return []
        cap = 8192
        t = (C.c_ulonglong * cap)()
        names = C.create_string_buffer(24 * cap)
        n = fn(t, names, cap)
        out += [(int(t[i]), names.raw[24 * i:24 * i + 24].split(b"\0")[0].decode()) for i in range(n)]
    return sorted(out)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "serve" and args.workload == "c2":
        run_serve_c2(args)
    elif args.mode == "serve" and not (args.gpus > 1 and "WORLD_SIZE" not in os.environ):
        run_serve(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
