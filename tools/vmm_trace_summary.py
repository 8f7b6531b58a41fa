"""Summarise a PRISM_VMM_TRACE file against bench.py's timed-region marker:
per 10 ms bucket of the timed region, the worker's driver calls (count,
pages, mean us per page by kind) and the caller's waits."""
import collections
import re
import sys


def main(trace_path, err_path, region="timed-region"):
    lo = hi = None
    for ln in open(err_path):
        m = re.match(region + r" (\d+) (\d+)", ln)
        if m:
            lo, hi = int(m.group(1)), int(m.group(2))
    recs = []
    for ln in open(trace_path):
        t, k, p, us = ln.split()
        recs.append((int(t), k, int(p), float(us)))
    recs.sort()
    print(f"timed region {(hi - lo) / 1e6:.1f} ms; {len(recs)} trace records total")
    b = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0, 0.0]))
    for t, k, p, us in recs:
        if lo - 50_000_000 <= t <= hi:
            key = (t - lo) // 10_000_000
            e = b[key][k]
            e[0] += 1
            e[1] += p
            e[2] += us
    for key in sorted(b):
        parts = []
        for k, (n, p, us) in sorted(b[key].items()):
            parts.append(f"{k}: n={n} pages={p} us/page={us / max(p, 1):.0f}" if k != "W" else f"W: n={n} ms={us / 1e3:.2f}")
        print(f"{key * 10:+5d} ms  " + "; ".join(parts))


if __name__ == "__main__":
    main(*sys.argv[1:4])
