"""Crossover of the one-CTA QAS round (qas_small.cuh) vs the multi-kernel
round: wall time per round through DeviceScheduler.round_arrays (same host
marshalling and copies on both sides) for a range of pending-set sizes.

    python tools/qas_crossover.py  ->  one JSON line per P
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_08581_b200.qas import DeviceScheduler  # noqa: E402
from paper_2605_08581_b200.qas_host import marshal_round  # noqa: E402
from paper_2605_08581_b200.types import Request, SchedulerConfig  # noqa: E402


def round_inputs(P, nseg, rng):
    pend = []
    for i in range(P):
        k = int(rng.integers(3, 8))
        sk = [int(min(rng.zipf(1.3), nseg) - 1)] + [int(x) for x in rng.integers(0, nseg, size=k - 1)]
        pend.append(Request(i, float(rng.random()), sk, bool(rng.random() < 0.9), [], 28, 128 * k, 100))
    act = [Request(10**7 + j, 0.0, [int(x) for x in rng.integers(0, nseg, size=5)], True, [], 28, 640, 100)
           for j in range(256)]
    return pend, act


def main():
    rng = np.random.default_rng(0)
    ds = DeviceScheduler()
    def timed(m, cfg, n=40):
        for _ in range(5):
            ds.round_arrays(m, cfg)
        t0 = time.perf_counter()
        for _ in range(n):
            ds.round_arrays(m, cfg)
        return round((time.perf_counter() - t0) / n * 1e6, 1)

    for P in (64, 256, 512, 1024, 2048, 3072, 4096):
        pend, act = round_inputs(P, 981, rng)
        cfg = SchedulerConfig(dispatch_budget=min(P, 4096), cold_quota=min(P, 64))
        m = marshal_round(pend, act)
        out = {"P": P}
        ds.set_small(0)
        out["multi_us"] = timed(m, cfg)
        ds.set_small(4096)
        for G in (1, 8, 32, 74, 148, 0):
            ds.tune(grid=G)
            out[f"grid{G or 'auto'}_us"] = timed(m, cfg)
        ds.tune(grid=0)
        ds.profile(True)
        ds.round_arrays(m, cfg)
        ts = ds.small_timeline()
        ds.profile(False)
        out["auto_grid"] = ds.last_grid()
        out["auto_phases_us"] = [round((b - a) / 1e3, 1) for a, b in zip(ts, ts[1:])]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
