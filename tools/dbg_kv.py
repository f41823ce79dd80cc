import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from traces import synth as S
import bench
from paper_2605_08581_b200.wave import WaveEngine, DevicePending
from paper_2605_08581_b200.kv import KvPool
w = sys.argv[1] if len(sys.argv) > 1 else "c5"
d = bench.DEFAULTS[w]; spec = S.SPECS[w]; B = d["wave"]
import argparse
cache, sched = bench._configs(argparse.Namespace(capacity=d["capacity"], protect=20, wave=B, cold_quota=64))
eng = WaveEngine(cache, sched, spec.nseg, spec.sys_len, spec.chunk, device=0, initial_slots=1 << 21, initial_arena_tokens=max(1 << 26, 4 * d["capacity"]))
kv = KvPool(eng.t, d["capacity"] + 2 * B * spec.path_len, 64)
st = S.ShardStream(w, 0, 1, 0); dev = torch.device("cuda", 0); prev = 0
for i in range(30):
    eng.release(eng.leaf_slots, prev)
    p = st.take(B)
    nm, prev = eng.step(DevicePending.from_host(p["ids"], p["arrival"], p["sk_off"], p["sk"], p["reorderable"], p["suffix"], dev))
    s0 = eng.stats()
    new, freed = kv.sync(None, None)
    k = kv.stats()
    print(i, "adm", prev, "new", new, "freed", freed, "inuse", k["rows"] - k["free"], "resident", s0["resident"], "arena", s0["arena_used"], "victims", s0["victims"], eng.wave_stats(), flush=True)
