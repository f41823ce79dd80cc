"""Summarise an `ncu --set full` capture (raw page CSV) as a markdown table.

    ncu -i prof_full.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_full_md.py raw.csv out.md "title"
"""

import csv
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else "ncu --set full"
    rows = list(csv.reader(open(src)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]

    def f(r, k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")

    out = [f"# {title}", "",
           "Cold-cache, serialised replay (ncu): compare shares and DRAM traffic, not absolute wave times.", "",
           "| kernel | grid x block | us | DRAM rd MB | DRAM wr MB | DRAM TB/s | L2 hit % | warps active % | regs | top stalls (per issue) |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        name = r[ix["Kernel Name"]].split("(")[0]
        us = f(r, "gpu__time_duration.sum")
        unit = rows[1][ix["gpu__time_duration.sum"]]
        if unit == "nsecond":
            us /= 1000.0
        elif unit == "msecond":
            us *= 1000.0
        rd = f(r, "dram__bytes_read.sum")
        wr = f(r, "dram__bytes_write.sum")
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = rows[1][ix[k]]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            if k.endswith("read.sum"):
                rd *= scale
            else:
                wr *= scale
        tbs = (rd + wr) / (us * 1e-6) / 1e12 if us > 0 else 0.0
        st = sorted(((f(r, h), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for h in stall),
                    reverse=True)[:2]
        out.append(f"| `{name}` | {r[ix['launch__grid_size']]} x {r[ix['launch__block_size']]} | {us:.1f} | "
                   f"{rd / 1e6:.2f} | {wr / 1e6:.2f} | {tbs:.2f} | {f(r, 'lts__t_sector_hit_rate.pct'):.1f} | "
                   f"{f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                   f"{r[ix['launch__registers_per_thread']]} | "
                   + ", ".join(f"{n} {v:.1f}" for v, n in st) + " |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
