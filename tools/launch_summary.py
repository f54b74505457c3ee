"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name the launch count, total and mean duration and the share of
all kernel time (cold-cache, serialised per-launch times: the SHARE is what
compares with the live bench, not the absolute)."""
import collections
import csv
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.DictReader(lines)
    for d in r:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        rows.append((name, v * scale))
    tot = sum(t for _, t in rows)
    agg = collections.OrderedDict()
    for n, t in rows:
        c, s = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, s + t)
    print(f"{len(rows)} launches, {tot / 1e3:.1f} ms total kernel time")
    print(f"{'kernel':40s} {'launches':>9s} {'total ms':>10s} {'mean us':>9s} {'share':>7s}")
    for n, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:40s} {c:9d} {s / 1e3:10.2f} {s / c:9.2f} {s / tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
