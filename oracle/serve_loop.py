"""CPU oracle of the serving loop (engine.py:141-266) over a trace CSR.

TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's baseline legs): the
checker for the device serving loop (paper_2605_08581_b200/serve.py) at sizes
the per-request Python restatement in tests/sim_harness.py cannot reach.  Every
decision is the C oracle (oracle/*.c, pinned to the reference's recorded
outputs); this module only restates the loop's bookkeeping, window by window:

  t = k * window_s                                             (engine.py:167)
  completions with completion <= t + 1e-12 release their leaf  (171-175)
  arrivals with arrival_time <= t + 1e-12 join pending         (176-178)
  idle (t + 1e-12 >= busy_until) and pending: one wave         (180-213)
  cost model: duration = uncached / rate, first token, completion, busy_until (215-232)
"""

from __future__ import annotations

import heapq
import time

import numpy as np

from oracle.windows import OracleReplica

MAX_WINDOWS = 50_000_000  # engine.py:137


def _sub(tr, idx: np.ndarray) -> dict:
    """Pending / in-flight CSR of the trace rows ``idx`` (in that order)."""
    lens = np.diff(tr.sk_off)[idx]
    off = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    rows = [tr.sk[tr.sk_off[i]:tr.sk_off[i + 1]] for i in idx.tolist()]
    sk = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    return {"ids": tr.ids[idx], "arrival": tr.arrival[idx], "sk_off": off, "sk": sk,
            "reorderable": tr.reorderable[idx], "suffix": tr.suffix[idx]}


def oracle_serve(tr, config, max_requests: int | None = None) -> dict:
    """Replay ``tr`` (a TraceCSR in (arrival, id) order) on the oracle.  Returns
    per-request arrays in trace order (admit, first_token, completion, hit),
    the waves (launch, duration, members as trace indices), the victim log and
    the decision timing (admitted requests, seconds inside the waves)."""
    n = tr.n if max_requests is None else min(tr.n, max_requests)
    cache, sched = config.cache, config.scheduler
    rep = OracleReplica(cache, sched, tr.num_segments, tr.sys_prefix_tokens, tr.chunk_tokens)
    h = rep.cache._h
    plen = tr.path_len()
    window = sched.window_s
    for i in range(n):
        if plen[i] > cache.capacity_tokens:
            raise RuntimeError(f"request {tr.ids[i]} path ({plen[i]} tokens) exceeds cache capacity "
                               f"({cache.capacity_tokens})")
    admit, first, comp = (np.zeros(n) for _ in range(3))
    hit = np.zeros(n, np.int64)
    waves_t, waves_d, waves_m = [], [], []
    pending: list[int] = []
    inflight: list = []  # (completion, trace index, leaf id)
    active: set[int] = set()
    nxt = completed = k = 0
    busy = 0.0
    while completed < n:
        k += 1
        if k > MAX_WINDOWS:
            raise RuntimeError("simulation failed to make progress")
        t = k * window
        while inflight and inflight[0][0] <= t + 1e-12:
            _, ti, leaf = heapq.heappop(inflight)
            rep.L.ot_release(h, leaf)
            active.discard(ti)
            completed += 1
        while nxt < n and tr.arrival[nxt] <= t + 1e-12:
            pending.append(nxt)
            nxt += 1
        if not pending or t + 1e-12 < busy:
            continue
        pidx = np.array(pending, np.int64)
        act = _sub(tr, np.array(sorted(active), np.int64))
        r = rep.step(_sub(tr, pidx), active=(act["sk_off"], act["sk"]), release_prev=False)
        na = r["n_admitted"]
        if na == 0:
            continue
        taken = pidx[r["members"][:na]]
        hits = r["hits"]
        uncached = int((plen[taken] - hits).sum())
        te = completed / t if t > 0 else 0.0
        rate = config.prefill_rate
        if config.decode_attenuation_enabled:
            alpha = min(max(te * config.output_tokens / config.decode_rate, 0.0), 0.95)
            rate = config.prefill_rate * (1.0 - alpha)
        duration = uncached / rate
        pe = t + duration
        ft = pe + na / config.decode_rate
        cp = ft + (config.output_tokens - 1) * na / config.decode_rate
        busy = pe
        waves_t.append(t)
        waves_d.append(duration)
        waves_m.append(taken)
        admit[taken], first[taken], comp[taken], hit[taken] = t, ft, cp, hits
        for ti, leaf in zip(taken.tolist(), r["leaf_ids"].tolist()):
            active.add(ti)
            heapq.heappush(inflight, (cp, ti, leaf))
        done = set(taken.tolist())
        pending = [i for i in pending if i not in done]
    return {"admit": admit, "first_token": first, "completion": comp, "hit": hit,
            "wave_launch": np.array(waves_t), "wave_duration": np.array(waves_d),
            "wave_members": np.concatenate(waves_m) if waves_m else np.zeros(0, np.int64),
            "wave_sizes": np.array([len(m) for m in waves_m], np.int64),
            "victims": rep.victims(), "decisions": rep.decisions, "seconds": rep.decision_seconds}


def serve_timing(tr, config, seconds: float, max_requests: int | None = None) -> dict:
    """The oracle serving loop on a prefix of ``tr`` sized to ~``seconds`` of
    CPU work (the bounded CPU baseline sample): decisions / s inside the waves."""
    t0 = time.perf_counter()
    n = min(tr.n, max_requests or tr.n)
    lo, res = 256, None
    while True:
        res = oracle_serve(tr, config, max_requests=min(lo, n))
        if time.perf_counter() - t0 > seconds / 3 or lo >= n:
            break
        lo *= 4
    return {"requests": min(lo, n), "decisions": res["decisions"], "seconds": res["seconds"]}
