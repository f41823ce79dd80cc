"""Per-phase diagnostics of the bench wave (run on a GPU box).

    python tools/diag_wave.py [--steps 5]

Prints, per timed wave: the wave's CUDA-event time, host wall time, the
live per-phase device profile, the one-launch QAS round timeline and the
cooperative eviction-list build timeline.  Diagnostics only (not a bench).
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(bench.DEFAULTS))
    args = ap.parse_args()
    import torch

    from traces import synth as S
    from paper_2605_08581_b200.wave import DevicePending, WaveEngine

    d = bench.DEFAULTS[args.workload]
    spec = S.SPECS[args.workload]
    B = d["wave"]
    ns = argparse.Namespace(capacity=d["capacity"], protect=20, wave=B, cold_quota=64)
    cache, sched = bench._configs(ns)
    eng = WaveEngine(cache, sched, spec.nseg, spec.sys_len, spec.chunk, device=0, initial_slots=1 << 21,
                     initial_arena_tokens=max(1 << 26, 4 * d["capacity"]))
    L = eng.L
    L.prism_qas_small_timeline.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    st = S.ShardStream(args.workload, 0, 1, 0)

    def dev(pool):
        return DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"],
                                       pool["reorderable"], pool["suffix"], torch.device("cuda", 0))

    prev = 0
    for i in range(0, d["warm"], B):
        eng.release(eng.leaf_slots, prev)
        _, prev = eng.step(dev(st.take(min(B, d["warm"] - i))))
    pools = [dev(st.take(B)) for s in range(args.steps + 2)]
    for s in range(2):
        eng.release(eng.leaf_slots, prev)
        _, prev = eng.step(pools[s])
    torch.cuda.synchronize()
    eng.profile(True)
    for s in range(2, args.steps + 2):
        p0 = eng.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(eng.stream)
        eng.release(eng.leaf_slots, prev)
        nm, prev = eng.step(pools[s])
        e1.record(eng.stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e6
        p1 = eng.profile_read()
        ph = {k: round((p1[k]["ms"] - p0[k]["ms"]) * 1000, 1) for k in ("qas", "protect", "build", "commit",
                                                                         "prematch", "release")}
        ts = np.zeros(11, dtype=np.int64)
        L.prism_qas_small_timeline(eng.q, ts.ctypes.data, 11)
        print(f"wave {s}: event {e0.elapsed_time(e1) * 1000:.1f} us, wall {wall:.1f} us, phases(us) {ph}")
        print("  qas one-launch phases (us):", (np.diff(ts) / 1e3).round(1).tolist())
        print("  build:", eng.build_timeline())
        cnt = np.zeros(4, dtype=np.int64)
        L.prism_coop_counts.argtypes = [C.c_void_p, C.c_void_p]
        L.prism_coop_counts(eng.t, cnt.ctypes.data)
        print(f"  coop counts (tf_n, prot_n, order candidates, selected): {cnt.tolist()}")
        off = np.zeros(4097, dtype=np.uint32)
        nb = np.zeros(1, dtype=np.int32)
        L.prism_coop_buckets.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        L.prism_coop_buckets(eng.t, off.ctypes.data, 4096, nb.ctypes.data)
        sz = np.diff(off[: min(int(nb[0]), 4096) + 1].astype(np.int64))
        if sz.size:
            print(f"  buckets: {sz.size}, sum {sz.sum()}, max {sz.max()}, >384: {(sz > 384).sum()}, "
                  f">1024: {(sz > 1024).sum()}, top: {sorted(sz.tolist())[-8:]}, first/last: {sz[:3].tolist()} {sz[-3:].tolist()}")
    eng.close()


if __name__ == "__main__":
    main()
