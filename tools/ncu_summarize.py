"""Summarise an ncu launch list (tools/ncu_capture.sh) per kernel and per phase.

    python tools/ncu_summarize.py gpurun_out/launches.csv profiles/r01_ncu_launches.md \
        [profiles/ncu_summary.json] [steps]

Shares are computed over the kernels of the NVTX "timed" range (cold-cache,
serialised by ncu: compare SHARES, not absolute times).  The JSON carries the
per-launch DRAM bytes that bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import sys

PHASE = [  # (phase, kernel-name substrings); first match wins
    ("protect", ("k_prot_", "k_protect_coop", "<prism::ProtCand>", "k_tf_")),
    ("build", ("k_build_keys", "k_propagate", "k_gather", "k_list_ready", "k_build_coop", "<prism::EvictCand>")),
    ("select", ("k_ss_",)),  # shared sample-select kernels (build and protection)
    ("commit", ("k_wp_", "k_wc_", "k_dscan_", "k_vscan_", "k_commit")),
    ("prematch", ("k_prematch",)),
    ("release", ("k_release",)),
    ("qas", ("k_qas_small", "q_")),
]


def phase_of(name: str) -> str:
    for ph, keys in PHASE:
        if any(k in name for k in keys):
            return ph
    if "cub::" in name or "DeviceRadixSort" in name or "DeviceScan" in name or "Onesweep" in name:
        return "cub"
    if "at::" in name:
        return "torch (L2 flush / copies, outside the timed events)"
    return "other"


def main():
    src, dst = sys.argv[1], sys.argv[2]
    jdst = sys.argv[3] if len(sys.argv) > 3 else None
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    per = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0, "hit": []})
    for r in rows:
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        if "<" in name.split("(")[0]:  # keep template arguments (ProtCand / EvictCand instances)
            short = name.split("(")[0].replace("void ", "")[:120]
        m, v = r["Metric Name"], r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        a = per[short]
        if m == "gpu__time_duration.sum":
            a["n"] += 1
            a["ns"] += v
        elif m == "dram__bytes_read.sum":
            a["rd"] += v
        elif m == "dram__bytes_write.sum":
            a["wr"] += v
        elif m == "lts__t_sector_hit_rate.pct":
            a["hit"].append(v)
    ours = {k: a for k, a in per.items() if not phase_of(k).startswith("torch")}
    tot = sum(a["ns"] for a in ours.values())
    phases = collections.defaultdict(lambda: {"ns": 0.0, "n": 0, "dram": 0.0})
    for k, a in ours.items():
        p = phases[phase_of(k)]
        p["ns"] += a["ns"]
        p["n"] += a["n"]
        p["dram"] += a["rd"] + a["wr"]
    out = io.StringIO()
    out.write(f"# ncu launch list -- {src}\n\n")
    out.write(f"{steps} timed wave(s); {sum(a['n'] for a in ours.values())} launches of the library "
              f"(hand-written + CUB); total serialised device time {tot / 1e3:.1f} us.\n\n")
    out.write("## per phase\n\n| phase | share | us/wave | launches/wave | DRAM MB/wave |\n|---|---|---|---|---|\n")
    for ph, p in sorted(phases.items(), key=lambda x: -x[1]["ns"]):
        out.write(f"| {ph} | {100 * p['ns'] / tot:.1f}% | {p['ns'] / 1e3 / steps:.1f} | {p['n'] / steps:.1f} | "
                  f"{p['dram'] / 1e6 / steps:.2f} |\n")
    out.write("\n## per kernel\n\n| kernel | phase | share | launches | us/launch | DRAM MB/launch | L2 hit % |\n"
              "|---|---|---|---|---|---|---|\n")
    for k, a in sorted(ours.items(), key=lambda x: -x[1]["ns"]):
        hit = sum(a["hit"]) / len(a["hit"]) if a["hit"] else float("nan")
        out.write(f"| `{k}` | {phase_of(k)} | {100 * a['ns'] / tot:.1f}% | {a['n']} | {a['ns'] / 1e3 / a['n']:.2f} | "
                  f"{(a['rd'] + a['wr']) / 1e6 / a['n']:.3f} | {hit:.1f} |\n")
    open(dst, "w").write(out.getvalue())
    if jdst:
        js = {"source": src, "steps": steps, "kernels": {}, "phases": {}}
        for ph, p in phases.items():
            js["phases"][ph] = {"us_per_wave": p["ns"] / 1e3 / steps, "share": p["ns"] / tot,
                                "dram_bytes_per_wave": p["dram"] / steps,
                                "dram_bytes_per_launch": p["dram"] / max(p["n"], 1)}
        for k, a in ours.items():
            js["kernels"][k] = {"launches": a["n"], "us_per_launch": a["ns"] / 1e3 / a["n"],
                                "dram_bytes_per_launch": (a["rd"] + a["wr"]) / a["n"]}
        # phase-level traffic under the names bench.py uses for roofline.kernel
        for ph in ("build", "commit", "protect", "prematch", "qas"):
            if ph in phases:
                js["kernels"].setdefault(ph, {})["dram_bytes_per_launch"] = phases[ph]["dram"] / steps
        json.dump(js, open(jdst, "w"), indent=1)
    print(out.getvalue()[:3000])


if __name__ == "__main__":
    main()
