#!/usr/bin/env python
"""bench.py -- PRISM scheduling-memory hot path (QAS + DART) on B200.

Metric (BASELINE.json): prefix-match+admit+evict decisions/sec at a ~1M-node
DART tree.  One *decision* = one admitted request: its exact-prefix match and
its insert including _reserve/evict, with the wave's QAS round and
protection pass amortised.

Workload ("mu1M"): a DART tree warm-started with 125,000
paths (system prefix 28 tokens + 8 segments x 16 tokens + 16-token private
suffix; segment 0 uniform over 50, the others uniform over 2M) -- about
1.0M nodes / 16M tokens at capacity_tokens = 16,000,000, so every admission
evicts.  A *step* is one serving-loop wave (engine.py:189-213) of 4096 new
requests: device QAS round -> protection hand-off -> serialization -> ordered
match+insert+evict -> release of the previous wave's pins.  Synthetic data,
deterministic seeds; one independent replica tree per GPU (weak scaling) with
one NCCL all-reduce of the per-window demand counters per step when N > 1.

    python bench.py [--gpus N --steps K --warmup W]       # our B200 path
    python bench.py --impl reference ...                   # reference algorithm on host cores

Prints exactly one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefix-match+admit+evict decisions/sec @1M-node DART; hit-rate parity; HBM GB/s"
UNIT = "decisions/s"
SYS_LEN, K_SEG, CHUNK, SUFFIX = 28, 8, 16, 16
SLOT0, OTHERS = 50, 2_000_000
NSEG = SLOT0 + OTHERS


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--wave", type=int, default=4096)
    ap.add_argument("--paths", type=int, default=125_000)
    ap.add_argument("--capacity", type=int, default=16_000_000)
    ap.add_argument("--protect", type=int, default=20)
    ap.add_argument("--cold-quota", type=int, default=64)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=-1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no baseline/e2e)")
    ap.add_argument("--profile-steps", type=int, default=3,
                    help="extra waves AFTER the timed region with the per-phase device profile on (roofline)")
    return ap.parse_args()


# ---------------------------------------------------------------- workload


def make_pool(first_id: int, n: int, rng: np.random.Generator) -> dict:
    """n synthetic requests (ids first_id..): mu1M skeletons, dense segment ids."""
    sk = np.empty((n, K_SEG), dtype=np.int32)
    sk[:, 0] = rng.integers(0, SLOT0, size=n)
    sk[:, 1:] = SLOT0 + rng.integers(0, OTHERS, size=(n, K_SEG - 1))
    ids = np.arange(first_id, first_id + n, dtype=np.int64)
    return {
        "ids": ids,
        "arrival": ids.astype(np.float64) * 1e-3,
        "sk_off": np.arange(n + 1, dtype=np.int64) * K_SEG,
        "sk": sk.reshape(-1),
        "reorderable": np.ones(n, dtype=np.uint8),
        "suffix": np.full(n, SUFFIX, dtype=np.int32),
    }


def pool_bytes(pool: dict) -> int:
    return int(sum(v.nbytes for v in pool.values()))


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


# ---------------------------------------------------------------- CPU oracle sample


def oracle_sample(seconds: float, paths: int, capacity: int, protect: int, wave: int, seed: int) -> dict:
    """The reference algorithm (oracle/ C restatement, full scan + heap per
    evict) on the same workload: warm start, then one wave timed for a bounded
    number of decisions.  TEST/BASELINE INFRASTRUCTURE ONLY."""
    from oracle.oracle import OracleRadixCache, _ptr, lib as olib, oracle_round_arrays
    from paper_2605_08581_b200.qas_host import MarshaledRound
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig

    rng = np.random.default_rng(seed)
    cache = OracleRadixCache(CacheConfig(capacity_tokens=capacity, policy=CachePolicy.DART, protect_budget=protect))
    L = olib()
    plen = SYS_LEN + K_SEG * CHUNK + SUFFIX
    a_off = np.array([SYS_LEN] + [SYS_LEN + CHUNK * (j + 1) for j in range(K_SEG)] + [plen], dtype=np.int64)
    a_kind = np.array([0] + [1] * K_SEG + [2], dtype=np.int8)
    seg_none = -(2**63)
    leaf = np.zeros(1, np.int64)
    nv = np.zeros(1, np.int64)

    def path_of(rid: int, segs: np.ndarray) -> np.ndarray:
        p = np.empty(plen, dtype=np.uint32)
        p[:SYS_LEN] = np.arange(SYS_LEN)
        p[SYS_LEN:SYS_LEN + K_SEG * CHUNK] = (1_000_000 + segs[:, None].astype(np.int64) * CHUNK
                                              + np.arange(CHUNK)).reshape(-1)
        p[SYS_LEN + K_SEG * CHUNK:] = 2_000_000_000 + rid * SUFFIX + np.arange(SUFFIX)
        return p

    def insert(rid, segs, snaps):
        p = path_of(rid, segs)
        a_seg = np.concatenate([[seg_none], segs.astype(np.int64), [seg_none]])
        L.ot_match(cache._h, _ptr(p), plen, None, _ptr(nv))
        return L.ot_insert(cache._h, _ptr(p), plen, len(a_off), _ptr(a_off), _ptr(a_kind), _ptr(a_seg),
                           _ptr(snaps), _ptr(leaf))

    zero_snap = np.zeros(3 * len(a_off), np.int64)
    pool = make_pool(0, paths, rng)
    sk = pool["sk"].reshape(paths, K_SEG)
    for i in range(paths):  # warm start (untimed)
        insert(i, sk[i], zero_snap)
        L.ot_release(cache._h, int(leaf[0]))
    # one timed wave: QAS round + protection + ordered admissions until the budget
    pend = make_pool(paths, wave, rng)
    sched = SchedulerConfig(dispatch_budget=wave, cold_quota=64)
    t0 = time.perf_counter()
    m = MarshaledRound(list(range(wave)), np.arange(NSEG, dtype=np.int64), pend["ids"], pend["arrival"],
                       pend["sk_off"], pend["sk"], pend["reorderable"], np.zeros(1, np.int64),
                       np.zeros(0, np.int32))
    out = oracle_round_arrays(m, sched)
    dom = np.flatnonzero(out.dom)
    cache.set_protection(dict(zip(dom.tolist(), out.prio[dom].tolist())))
    members = np.concatenate([out.hot, out.cold])
    done = 0
    for i in members:
        al = out.aligned[i * K_SEG:(i + 1) * K_SEG]
        snaps = np.zeros(3 * len(a_off), np.int64)
        snaps[3:3 + 3 * K_SEG] = np.stack([out.g[al], out.a[al], out.nd[al]], axis=1).reshape(-1)
        rc = insert(int(pend["ids"][i]), al, snaps)
        if rc != 0:
            break
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    el = time.perf_counter() - t0
    return {"decisions": done, "seconds": el, "value": done / el}


def _ref_worker(args):
    seconds, paths, capacity, protect, wave, seed = args
    return oracle_sample(seconds, paths, capacity, protect, wave, seed)


# ---------------------------------------------------------------- reference arm


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs and prints the host-core baseline
    import multiprocessing as mp

    from oracle import oracle as O

    O.build()
    cores = max(1, min(len(os.sched_getaffinity(0)), 8))
    per_step = 0.5  # seconds of decisions per step per worker (bounded sample)
    total = max(args.steps, 1) * per_step
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_ref_worker, [(total, args.paths, args.capacity, args.protect, args.wave,
                                      args.seed + 17 * w) for w in range(cores)])
    value = sum(r["value"] for r in res)
    decisions = sum(r["decisions"] for r in res)
    secs = max(r["seconds"] for r in res)
    ms_per_step = 1000.0 * secs / max(args.steps, 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "mu1M DART tree (125K warm paths, ~1M nodes, cap 16M tokens), waves of 4096",
                   "wave": args.wave, "policy": "DART"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{decisions} decisions over {cores} replica processes x {total:.1f}s after "
                                   f"a {args.paths}-path warm start (oracle/ C restatement of kvcache.py/"
                                   f"scheduler.py: full scan + heap per evict)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig
    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B = args.wave
    engine = WaveEngine(
        CacheConfig(capacity_tokens=args.capacity, policy=CachePolicy.DART, protect_budget=args.protect),
        SchedulerConfig(dispatch_budget=B, cold_quota=args.cold_quota),
        NSEG, SYS_LEN, CHUNK, device=local, initial_slots=1 << 21, initial_arena_tokens=1 << 28,
    )
    rng = np.random.default_rng(args.seed + 1000 * rank)  # shard = independent sub-trace
    stream = engine.stream
    demand = torch.zeros(NSEG, dtype=torch.int32, device=dev) if world > 1 else None

    def to_dev(pool):
        return DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"],
                                       pool["reorderable"], pool["suffix"], dev)

    # warm start (untimed): the mu1M tree through the same fused path
    next_id, prev = 0, 0
    t_ws = time.perf_counter()
    while next_id < args.paths:
        n = min(B, args.paths - next_id)
        engine.release(engine.leaf_slots, prev)
        _, prev = engine.step(to_dev(make_pool(next_id, n, rng)))
        next_id += n
    engine.release(engine.leaf_slots, prev)
    prev = 0
    torch.cuda.synchronize()
    warm_s = time.perf_counter() - t_ws
    st0 = engine.stats()

    nsteps = args.warmup + args.steps
    nprof = max(args.profile_steps, 1)
    pools = [make_pool(next_id + s * B, B, rng) for s in range(nsteps + nprof)]
    next_id += (nsteps + nprof) * B
    dpools = [to_dev(p) for p in pools]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def one_step(pend):
        nonlocal prev
        engine.release(engine.leaf_slots, prev)
        nm, na = engine.step(pend)
        if demand is not None:  # per-window demand counters across replicas (NVLink)
            with torch.cuda.stream(stream):
                engine.demand_counters(demand)
                dist.all_reduce(demand)
        prev = na
        return nm, na

    for s in range(args.warmup):
        one_step(dpools[s])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof0 = engine.profile_read()  # (launch counters; the profile itself stays off while timing)
    st1 = engine.stats()
    clocks = Clocks(local)
    clocks.start()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" scopes profiles here
    evs = []
    admitted = members = 0
    for s in range(args.warmup, nsteps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nm, na = one_step(dpools[s])
        e1.record(stream)
        evs.append((e0, e1))
        admitted += na
        members += nm
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    prof1 = engine.profile_read()
    st2 = engine.stats()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([admitted], dtype=torch.int64, device=dev)
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
        hpools = [make_pool(next_id + s * B, B, rng) for s in range(e2e_steps + ew)]
        next_id += (e2e_steps + ew) * B
        pinned = [{k: torch.from_numpy(v).pin_memory() for k, v in p.items()} for p in hpools]
        out_mem = np.empty(B, dtype=np.int64)
        out_hits = np.empty(B, dtype=np.int64)
        h2d = sum(v.numel() * v.element_size() for v in pinned[0].values())
        for s in range(ew):
            _, prev = engine.step_host(pinned[e2e_steps + s], out_mem, out_hits, release_n=prev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        adm2 = 0
        d2h = 0
        wall = []
        for s in range(e2e_steps):
            # host pinned inputs read in place by the wave, results back in host arrays,
            # the previous wave's pins released by the same call
            tw = time.perf_counter()
            nm, na = engine.step_host(pinned[s], out_mem, out_hits, release_n=prev)
            wall.append((time.perf_counter() - tw) * 1e3)
            prev = na
            if demand is not None:
                with torch.cuda.stream(stream):
                    engine.demand_counters(demand)
                    dist.all_reduce(demand)
            d2h += 8 * (na + nm)
            adm2 += na
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms2], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2 = float(t.item())
            c = torch.tensor([adm2], dtype=torch.int64, device=dev)
            dist.all_reduce(c)
            adm2 = int(c.item())
        e2e = {"value": adm2 / (ms2 / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h // e2e_steps, "api": "prism_wave_step_host via WaveEngine.step_host "
               "(pinned host pending arrays read in place by the wave's staging kernel; admission order + hits "
               "copied to host inside the wave; the previous wave's pins released by the same call)",
               "host_ms_per_call": {"median": round(statistics.median(wall), 4), "max": round(max(wall), 4)}}

    # ---- roofline of the dominant kernel: a few more waves of the same workload
    # AFTER the timed region with the live per-phase profile on (its per-phase
    # event syncs would otherwise sit inside the timed region)
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
    d = {p: {k: prof3[p][k] - prof2[p][k] for k in ("ms", "calls", "launches")}
         for p in ("commit", "build", "protect", "prematch", "release", "qas")}
    victims = st4["victims"] - st3["victims"]
    created = st4["next_id"] - st3["next_id"]
    chain = prof3["chain_nodes"] - prof2["chain_nodes"]
    toks = prof3["inserted_tokens"] - prof2["inserted_tokens"]
    live = st4["live_nodes"]
    members_prof = nprof * B
    algo = {  # SURVEY.md 8(d) algorithmic bytes, per phase over the timed region
        "commit": 8 * toks + 32 * (chain + created + victims),
        "build": 16 * live * d["build"]["calls"],
        "protect": 16 * live * d["protect"]["calls"],
        "prematch": 4 * toks + 32 * chain,
        "qas": members_prof * (4 * K_SEG + 16),
        "release": 0,
    }
    # dominant phase by device time; "one launch" = one wave's worth of that
    # phase (its kernels back to back, SURVEY.md 8(d) bytes per wave)
    dom = max(("commit", "build", "protect", "prematch", "qas"), key=lambda p: d[p]["ms"])
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    per_wave_bytes = algo[dom] / nprof
    per_wave_s = d[dom]["ms"] / 1000.0 / nprof
    achieved = per_wave_bytes / per_wave_s / 1e9 if per_wave_s > 0 else 0.0
    traffic = None
    summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(summ):
        try:
            traffic = json.load(open(summ)).get("phases", {}).get(dom, {}).get("dram_bytes_per_wave")
        except Exception:
            traffic = None
    wave_bytes = sum(algo.values()) / nprof
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom,
                "launch": f"one wave's {dom} phase (its kernels back to back)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                "algorithmic_bytes_per_launch": per_wave_bytes, "launch_ms": per_wave_s * 1000.0,
                "phase_ms_per_wave": {p: round(d[p]["ms"] / nprof, 4) for p in d}, "profiled_waves": nprof,
                "wave": {"algorithmic_bytes": wave_bytes, "ms": ms / max(args.steps, 1),
                         "achieved_gbs": wave_bytes / (ms / max(args.steps, 1) / 1000.0) / 1e9}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        r = oracle_sample(args.cpu_seconds, args.paths, args.capacity, args.protect, B, args.seed + 99)
        cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{r['decisions']} decisions in {r['seconds']:.1f}s: one QAS round + set_protection + "
                         f"ordered match/insert(+evict) on a {args.paths}-path (~1M-node) oracle tree "
                         f"(oracle/ C restatement, single thread)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": "mu1M: DART tree warm-started with 125K paths (~1M nodes, ~16M tokens, "
                            "capacity 16M tokens so every admission evicts); step = one 4096-request wave "
                            "(device QAS round + protection + serialization + ordered match/insert/evict + "
                            "release)",
                "wave": B, "paths": args.paths, "capacity_tokens": args.capacity, "policy": "DART",
                "protect_budget": args.protect, "cold_quota": args.cold_quota,
                "parallelism": f"replicas x{world} (segment-hash shards)",
                "l2": "flushed between timed steps (256 MiB write)",
                "tree_nodes": st2["live_nodes"], "resident_tokens": st2["resident"],
                "warm_start_s": round(warm_s, 2), "admitted_per_rank": admitted,
                "members_per_rank": members, "victims": st2["victims"] - st1["victims"],
                "fast_path_members": st2["fast_members"] - st1["fast_members"],
                "slow_path_members": st2["slow_members"] - st1["slow_members"],
                "profile": "per-phase device profile taken on extra waves after the timed region",
                "commit": engine.wave_stats(),
                "cuda_graph": engine.graph_stats(),
                "last_list_build": engine.build_timeline(),
            },
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "lib_calls": prof1["lib_calls"] - prof0["lib_calls"],
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
