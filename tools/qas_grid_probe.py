"""Time the one-launch QAS round of C3-shaped pending sets at several grid sizes (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from traces import synth as S
from paper_2605_08581_b200.qas import DeviceScheduler
from paper_2605_08581_b200.types import SchedulerConfig
import ctypes as C

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec = S.SPECS[w]
st = S.ShardStream(w, 0, 1, 0)
pool = st.take(4096)
ds = DeviceScheduler()
ds.set_small(4096)
L = ds._L
L.prism_qas_round_device.argtypes = None
cfg = SchedulerConfig(dispatch_budget=4096, cold_quota=64)
dev = torch.device("cuda", 0)
from paper_2605_08581_b200.wave import DevicePending, WaveEngine
from paper_2605_08581_b200.types import CacheConfig
eng = WaveEngine(CacheConfig(capacity_tokens=10**9), cfg, spec.nseg, spec.sys_len, spec.chunk, device=0)
pend = DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"], pool["reorderable"], pool["suffix"], dev)
L2 = eng.L
L2.prism_qas_tune.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]
for grid in (64, 96, 128, 148):
    L2.prism_qas_tune(eng.q, 1, grid, None)
    eng.profile(True)
    ts = []
    for r in range(6):
        p0 = eng.profile_read()
        eng.step(pend, release_n=0)
        eng.release(eng.leaf_slots, 4096)
        torch.cuda.synchronize()
        ts.append((eng.profile_read()["qas"]["ms"] - p0["qas"]["ms"]) * 1000)
    eng.profile(False)
    print("grid", grid, "qas us", [round(x, 1) for x in ts[2:]])
