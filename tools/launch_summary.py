#!/usr/bin/env python
"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys


def main(path, skip_frac=0.0):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            v = float(r[idx["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("eig::<unnamed>::", "")
        recs.append((short, v))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in recs:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':55s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:55]:55s} {v[0]:8d} {v[1] / 1e6:10.2f} {v[1] / tot * 100:6.1f}% {v[1] / v[0] / 1e3:9.1f}")
    print(f"{'TOTAL':55s} {len(recs):8d} {tot / 1e6:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
