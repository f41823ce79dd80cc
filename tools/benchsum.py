"""One-screen summary of bench JSON lines: python tools/benchsum.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    c = d.get("config", {})
    print(f"== {f}: {d['value']:.0f} {d['unit']}  {d['ms_per_step']:.3f} ms/step  n_gpus {d['n_gpus']}")
    if "hit_rate" in d:
        print(f"  hit {d['hit_rate']:.4f} nodes {c.get('tree_nodes')} res {c.get('resident_tokens')} "
              f"adm {c.get('admitted_per_rank')}/{c.get('members_per_rank')} victims {c.get('victims')} "
              f"commit {c.get('commit')} graph {c.get('cuda_graph')}")
    print("  parity", d.get("parity"))
    print("  cpu", d.get("cpu_baseline"))
    r = d.get("roofline")
    if r:
        print(f"  roof {r['kernel']} frac {r['frac']:.4f} phases {r['phase_ms_per_wave']}")
        print(f"  bytes {r.get('algorithmic_bytes_per_wave')} wave {r['wave']}")
    e = d.get("e2e") or {}
    print(f"  e2e {e.get('value')} {e.get('host_ms_per_call')} launches {d.get('gpu_launches')} clocks {d.get('clocks')}")
