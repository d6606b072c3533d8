#!/usr/bin/env python3
"""Per-kernel mean duration from an ncu --csv launch list (gpu__time_duration)."""
import collections
import csv
import sys


def summary(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[i + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            if r[mi] == "gpu__time_duration.sum":
                v *= {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1)
            d[r[ki].split("(")[0].split("<")[0].replace("void ", "")][r[mi]].append(v)
    return d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        d = summary(p)
        tot = 0
        for k, m in sorted(d.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
            t = m["gpu__time_duration.sum"]
            extra = " ".join(f"{mn.split('__')[1][:18]}={sum(v) / len(v):.0f}" for mn, v in m.items() if mn != "gpu__time_duration.sum")
            print(f"  {k[:44]:44s} n={len(t):4d} mean={sum(t) / len(t):8.1f}us  {extra}")
