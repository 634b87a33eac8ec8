"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/launch_summary.py gpurun_out/launches.csv [steps] > profiles/x_launches.txt
Times are ncu's serialised, cold-cache per-launch durations: compare SHARES, not absolutes.
"""
import collections
import csv
import io
import sys


def main(path, steps=1):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        tot[k] += v / 1e3 if r["Metric Unit"] == "ns" else v
        cnt[k] += 1
    s = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {s / 1e3:.3f} ms summed (ncu, serialised)")
    print(f"{'kernel':58s} {'launches':>8s} {'us':>11s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:58s} {cnt[k]:8d} {v:11.1f} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
