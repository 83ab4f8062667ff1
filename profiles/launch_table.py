#!/usr/bin/env python3
"""ncu launch-list CSV (gpu__time_duration.sum) -> markdown table of per-kernel time and share.

    python profiles/launch_table.py profiles/r1_launches.csv > profiles/r1_launches.md
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "").replace("unnamed>::", "")
    return name


def main(path):
    lines = open(path).read().splitlines()
    head = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))  # skip program / ncu chatter
    rows = [r for r in csv.DictReader(lines[head:]) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = OrderedDict()
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if r["Metric Unit"] == "ns" else v  # -> us
        k = short(r["Kernel Name"])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + v)
    tot = sum(t for _, t in agg.values())
    print("# ncu launch list, one config-1 training view\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv "
          "python profiles/capture_step.py`; per-launch times are cold-cache and serialised: compare shares, "
          "not absolutes.\n")
    print("| kernel | launches | us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {t / tot:.1%} |")
    print(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:.1f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
