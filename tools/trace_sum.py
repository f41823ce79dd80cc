"""Per-wave kernel start timeline from a -DPRISM_TRACE bench run (PRISM_TRACE_OUT).

    python tools/trace_sum.py trace.json [first_kernel]

Waves are split at each start of `first_kernel` (default q_stage); prints the
median wave's kernels in start order: offset from the wave start and the gap
to the next start (on either stream), plus per-kernel median gaps over waves.
"""
import collections
import json
import statistics
import sys


def main():
    recs = json.load(open(sys.argv[1]))
    first = sys.argv[2] if len(sys.argv) > 2 else "q_stage"
    waves, cur = [], None
    ends = collections.defaultdict(list)
    for t, n in recs:
        if n.endswith("$"):  # per-CTA end stamps: the wave's last one per kernel
            if cur is not None:
                ends[(len(waves), n)].append(t - cur[0][0])
            continue
        if n == first:
            cur = []
            waves.append(cur)
        if cur is not None:
            cur.append((t, n))
    waves = [w for w in waves if len(w) > 5]
    spans = [w[-1][0] - w[0][0] for w in waves]
    print(f"{len(waves)} waves; first->last kernel start span median {statistics.median(spans) / 1e3:.1f} us")
    gaps = collections.defaultdict(list)
    for w in waves:
        for i, (t, n) in enumerate(w):
            nxt = w[i + 1][0] if i + 1 < len(w) else t
            gaps[(i, n)].append((t - w[0][0], nxt - t))
    last = collections.defaultdict(list)
    for (w, n), v in ends.items():
        last[n].append(max(v))
    for n, v in sorted(last.items()):
        print(f"end of {n[:-1]}: median {statistics.median(v) / 1e3:.1f} us after the wave start")
    for (i, n), v in sorted(gaps.items()):
        off = statistics.median(x for x, _ in v) / 1e3
        g = statistics.median(y for _, y in v) / 1e3
        print(f"{i:3d} {off:8.1f} us  +{g:6.1f}  {n}")


if __name__ == "__main__":
    main()
