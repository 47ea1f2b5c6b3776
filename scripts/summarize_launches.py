"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, total/mean device time and share of the total.

    python scripts/summarize_launches.py gpurun_out/launches.csv > profiles/rNN_launches.md
"""
import collections
import csv
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        rows.append((name, r["Grid Size"], r["Block Size"], ns))
    agg = collections.OrderedDict()
    for name, grid, block, ns in rows:
        a = agg.setdefault(name, {"n": 0, "ns": 0.0, "grid": set(), "block": block})
        a["n"] += 1
        a["ns"] += ns
        a["grid"].add(grid)
    total = sum(a["ns"] for a in agg.values())
    print(f"source: {path} ({len(rows)} launches, {total / 1e6:.3f} ms device time, "
          "cold-cache + serialised under ncu: compare shares, not absolutes)\n")
    print("| kernel | launches | total ms | mean us | share | grid | block |")
    print("|---|---:|---:|---:|---:|---|---|")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        print(f"| `{name}` | {a['n']} | {a['ns'] / 1e6:.3f} | {a['ns'] / a['n'] / 1e3:.1f} | "
              f"{100 * a['ns'] / total:.1f}% | {' '.join(sorted(a['grid']))[:40]} | {a['block']} |")


if __name__ == "__main__":
    main(sys.argv[1])
