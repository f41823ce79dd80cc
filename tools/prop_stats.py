"""Shape of the subtree-maximum propagation on the bench tree (run on a GPU box).

    python tools/prop_stats.py

Warms the C3 bench tree, snapshots it and reports, on the CPU: depth
distribution, how many nodes beat their parent's own key, and the minimal
walk of every node (the ancestors whose subtree maximum it is) -- what
bounds k_propagate's critical path.  Keys approximated as (class, last, id)
(P-hat and protection ignored).  Diagnostics only.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
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
    st = S.ShardStream(args.workload, 0, 1, 0)

    def dev(pool):
        return DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"],
                                       pool["reorderable"], pool["suffix"], torch.device("cuda", 0))

    prev = 0
    for i in range(0, d["warm"] + 4 * B, B):
        eng.release(eng.leaf_slots, prev)
        _, prev = eng.step(dev(st.take(B)))
    torch.cuda.synchronize()
    s = eng.cache_view()._snapshot()
    par, nid, last, kind, ref = s["par"], s["nid"], s["last"], s["kind"], s["ref"]
    n = len(par)
    live = (nid >= 0) & (par >= 0)
    live[0] = False
    idx = np.nonzero(live)[0]
    # depth by pointer doubling
    depth = np.zeros(n, np.int32)
    anc = par.copy()
    anc[~live] = 0
    anc[0] = 0
    cur = anc.copy()
    depth[live] = 1
    for _ in range(64):
        step = live & (cur > 0)
        if not step.any():
            break
        depth[step] += 1
        cur = np.where(step, anc[cur], cur)
    print("live nodes", idx.size, "max depth", depth.max(), "depth pct (50/90/99/max):",
          np.percentile(depth[idx], [50, 90, 99, 100]).tolist())
    blocked = live & ((ref > 0) | (kind == 2))
    cls = np.where(kind == 0, 0, 1).astype(np.int64)  # (0 private per the key's class 0; approximate)
    key = (cls << 100) if False else None
    # lexicographic (cls, last, nid) as a sortable rank
    order = np.lexsort((nid, last, cls))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    rank[~live] = -1
    p = par[idx]
    pl = p > 0
    beats = (rank[idx][pl] > rank[p[pl]]) & ~blocked[idx][pl] & ~blocked[p[pl]]
    print("blocked", int(blocked.sum()), "nodes beating their parent's own key", int(beats.sum()))
    # subtree argmax (blocked -> +inf) bottom-up by depth
    val = np.where(blocked, n + 1, rank).astype(np.int64)
    arg = np.arange(n, dtype=np.int64)
    best = val.copy()
    for dd in range(depth.max(), 1, -1):
        c = np.nonzero(live & (depth == dd))[0]
        pc = par[c]
        # max into parents (np.maximum.at over the values, then fix argmax)
        np.maximum.at(best, pc, best[c])
    # minimal walk: ancestors whose subtree max equals the node's own value
    own = val.copy()
    walk = np.zeros(n, np.int32)
    cur = np.where(live, par, 0)
    alive = live & ~blocked
    for _ in range(int(depth.max()) + 1):
        m = alive & (cur > 0)
        m &= best[np.maximum(cur, 0)] == own
        if not m.any():
            break
        walk[m] += 1
        alive = m
        cur = np.where(m, par[np.maximum(cur, 0)], 0)
    w = walk[live & ~blocked]
    print("minimal walk hops pct (50/90/99/99.9/max):", np.percentile(w, [50, 90, 99, 99.9, 100]).tolist(),
          "nodes walking >= 10 hops:", int((w >= 10).sum()), ">= 20:", int((w >= 20).sum()))
    eng.close()


if __name__ == "__main__":
    main()
