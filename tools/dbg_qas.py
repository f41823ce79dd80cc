import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import golden_util as G
from oracle.oracle import oracle_schedule_round, OracleRadixCache
from paper_2605_08581_b200.qas import DeviceScheduler
from sim_harness import run_simulation
run, trace, cfg = G.engine_case(0)
ds = DeviceScheduler()
n = [0]
def sched(p, a, c, t):
    a = list(a)
    bd = ds.schedule_round(p, a, c, t)
    bo = oracle_schedule_round(p, a, c, t)
    n[0] += 1
    fields = []
    if [r.id for r in bd.hot] != [r.id for r in bo.hot]: fields.append("hot")
    if [r.id for r in bd.cold] != [r.id for r in bo.cold]: fields.append("cold")
    if bd.priorities != bo.priorities: fields.append("prio")
    if bd.bucket_scores != bo.bucket_scores: fields.append("scores")
    for rid in bo.hints:
        h, d = bo.hints[rid], bd.hints.get(rid)
        if d is None or (d.aligned_skeleton, d.counter_snapshot, d.rank, d.signature) != (h.aligned_skeleton, h.counter_snapshot, h.rank, h.signature):
            fields.append(f"hint{rid}"); break
    if fields:
        print("round", n[0], "P", len(p), "A", len(a), fields)
        if "prio" in fields:
            diff = {k: (bd.priorities.get(k), bo.priorities.get(k)) for k in set(bd.priorities) | set(bo.priorities) if bd.priorities.get(k) != bo.priorities.get(k)}
            print(" prio diff", list(diff.items())[:5])
        if "hot" in fields: print(" hot", [r.id for r in bd.hot], [r.id for r in bo.hot])
        raise SystemExit(1)
    return bo
run_simulation(trace, cfg, cache_factory=OracleRadixCache, schedule_fn=sched)
print("all", n[0], "rounds equal")
