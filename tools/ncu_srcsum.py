"""Per-CUDA-line warp-stall samples of one kernel from an ncu --set full report.

    python tools/ncu_srcsum.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, fname, cur = {}, None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 6 or r[0] == "Line No" or r[0] == "":
            continue
        try:
            agg[(fname, int(r[0]), r[1].strip()[:100])] = agg.get((fname, int(r[0]), r[1].strip()[:100]), 0) + int(r[4])
        except ValueError:
            pass
    tot = sum(agg.values()) or 1
    print(f"{kre}: {tot} stall samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:7d} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
