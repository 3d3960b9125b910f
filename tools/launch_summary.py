"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file ...).

python tools/launch_summary.py launches.csv [--timed N]   # N = launches of the timed region (last N)
Prints per-kernel launch count, total / average ns and share of the device time.
"""
import argparse
import csv
import io
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--timed", type=int, default=0)
    a = ap.parse_args()
    lines = open(a.csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:])))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    if a.timed:
        rows = rows[-a.timed:]
    t, n = defaultdict(float), defaultdict(int)
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1.0)
        t[k] += float(r["Metric Value"]) * scale
        n[k] += 1
    tot = sum(t.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'avg_ms':>9s} {'share':>6s}")
    for k in sorted(t, key=t.get, reverse=True):
        print(f"{k[:70]:70s} {n[k]:8d} {t[k] / 1e6:10.3f} {t[k] / n[k] / 1e6:9.4f} {t[k] / tot:6.3f}")


if __name__ == "__main__":
    main()
