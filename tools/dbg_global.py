"""Debug: two replicas with the global-demand knob in ONE process (no collective)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from traces import synth as S
from oracle.oracle import build
from oracle.windows import OracleReplica, concat_pools, drop_members, pool_demand, device_victims
from paper_2605_08581_b200.wave import WaveEngine, DevicePending
import test_global_demand as T

build()
use_global = len(sys.argv) < 2 or sys.argv[1] == "1"
cache, sched = T._configs()
dev = torch.device("cuda", 0)
W = T.WORLD
wins = [T._windows(r) for r in range(W)]
engs = [WaveEngine(cache, sched, S.C4.nseg, S.C4.sys_len, S.C4.chunk, device=0) for _ in range(W)]
G = torch.zeros(S.C4.nseg, dtype=torch.int32, device=dev)
Gs = [torch.zeros(S.C4.nseg, dtype=torch.int32, device=dev) for _ in range(W)]
if use_global:
    for e in engs: e.set_global_demand(G)
reps = [OracleReplica(cache, sched, S.C4.nseg, S.C4.sys_len, S.C4.chunk) for _ in range(W)]
pd, po, prev = [None]*W, [None]*W, [0]*W
for i in range(T.WAVES):
    dps = []
    for r in range(W):
        pd[r] = concat_pools(pd[r], wins[r][i]); po[r] = concat_pools(po[r], wins[r][i])
        engs[r].release(engs[r].leaf_slots, prev[r])
        dp = DevicePending.from_host(pd[r]["ids"], pd[r]["arrival"], pd[r]["sk_off"], pd[r]["sk"], pd[r]["reorderable"], pd[r]["suffix"], dev)
        dps.append(dp)
        engs[r].demand(dp, Gs[r])
    torch.cuda.synchronize()
    G.copy_(sum(Gs))
    torch.cuda.synchronize()
    Go = sum(pool_demand(po[r], S.C4.nseg) for r in range(W))
    assert np.array_equal(G.cpu().numpy(), Go), "G differs"
    for r in range(W):
        nm, na = engs[r].step(dps[r])
        out = reps[r].step(po[r], global_g=Go if use_global else None)
        m = engs[r].members[:nm].cpu().numpy()
        ok = np.array_equal(m, out["members"]) and np.array_equal(engs[r].hits[:na].cpu().numpy(), out["hits"])
        dv, f = device_victims(engs[r].cache_view())
        ov = reps[r].victims()
        vok = np.array_equal(dv, ov[f:])
        print(f"window {i} rank {r}: dispatch/hits {ok} victims {vok} ({len(ov)}) na {na} stats {engs[r].wave_stats()}")
        if not vok and i == 0:
            from oracle.windows import device_table
            dt, ot = device_table(engs[r].cache_view()), reps[r].table()
            print("  tables equal:", dt.shape == ot.shape and np.array_equal(dt, ot), dt.shape, ot.shape)
            if dt.shape == ot.shape:
                bad = np.flatnonzero((dt != ot).any(axis=1))
                print("  differing rows (id parent elen kind seg ref last hits prot hasanc ftok):")
                for b in bad[:8]: print("   dev", dt[b].tolist(), "\n   ora", ot[b].tolist())
            print("  dev protected", sorted(dt[dt[:, 8] == 1, 0].tolist())[:30])
            print("  ora protected", sorted(ot[ot[:, 8] == 1, 0].tolist())[:30])
        if not vok:
            k = int(np.argmax(dv != ov[f:len(dv)+f])) if len(dv) == len(ov) - f else -1
            print("  first diff at", k, dv[max(k-3,0):k+5], ov[f+max(k-3,0):f+k+5], len(dv), len(ov))
        prev[r] = na
        pd[r] = drop_members(pd[r], m[:na]); po[r] = drop_members(po[r], out["members"][:out["n_admitted"]])
