"""Per-phase device profile of the serving loop on the C2 sweep point (diagnostic)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from types import SimpleNamespace
from paper_2605_08581_b200.serve import DeviceServingLoop, TraceCSR
from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig, SegmentCatalog
from paper_2605_08581_b200.wave import _bind
from traces.refgen import WorkloadConfig, generate_trace

qps = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
cat = SegmentCatalog(num_segments=981, chunk_tokens=128, hot_set=tuple(range(20)), sys_prefix_tokens=28)
cfg = SimpleNamespace(prefill_rate=1e4, decode_rate=4e4, output_tokens=32, decode_attenuation_enabled=False,
                      cache=CacheConfig(capacity_tokens=5760, policy=CachePolicy.DART, protect_budget=20),
                      scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=8, cold_quota=2))
tr = TraceCSR.from_trace(generate_trace(WorkloadConfig(qps=qps, num_requests=2048, k=5, r_hot=0.7, zipf_alpha=1.2,
                                                       suffix_tokens=100, seed=1), cat))
loop = DeviceServingLoop(cfg, tr)
L = _bind(loop.L)
PROF = len(sys.argv) < 3
if PROF:
    L.prism_profile(loop.t, 1); L.prism_qas_profile(loop.q, 1)
t0 = time.perf_counter(); loop.run(); wall = time.perf_counter() - t0
out = np.zeros(27); L.prism_profile_read(loop.t, out.ctypes.data)
qc = np.zeros(4, np.int64); L.prism_qas_counts(loop.q, qc.ctypes.data)
ph = ("commit", "build", "protect", "prematch", "release", "note", "maint")
c = loop.counts()
print("qps", qps, "waves", c["waves"], "wall ms", round(wall * 1e3, 1), "per wave us", round(wall * 1e6 / c["waves"], 1))
for i, p in enumerate(ph):
    print(f"  {p}: {out[i]:.1f} ms, calls {int(out[8+i])}, launches {int(out[16+i])}")
print("  qas: ms", qc[3] / 1000.0, "rounds", qc[2], "launches", qc[0])
ws = np.zeros(4, np.int64); L.prism_wave_stats(loop.t, ws.ctypes.data); print("  wave stats", ws)

L.prism_serve_wave_times.argtypes = [C.c_void_p, C.c_void_p]
wt = np.zeros(c["waves"], np.float32)
L.prism_serve_wave_times(loop.s, wt.ctypes.data)
print("  wave host us: median", float(np.median(wt)), "p99", float(np.percentile(wt, 99)), "max", float(wt.max()),
      "sum ms", float(wt.sum() / 1e3))
print("  slowest waves:", [(int(i), round(float(wt[i]))) for i in np.argsort(wt)[-8:]])
