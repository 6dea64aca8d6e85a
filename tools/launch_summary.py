"""ncu --metrics gpu__time_duration.sum --csv launch list -> markdown share table.

usage: python tools/launch_summary.py LAUNCHES.csv "COMMAND" > SUMMARY.md
"""
import collections
import csv
import sys


def main():
    path, cmd = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        k = r[iN].split("(")[0].replace("rrgpu::", "").replace("(anonymous namespace)::", "")
        k = k.replace("<unnamed>::", "").replace("void ", "")
        agg[k] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
        cnt[k] += 1
    tot = sum(agg.values())
    print(f"# Launch list of `{cmd}` (ncu gpu__time_duration.sum, --clock-control none)\n")
    print("Cold-cache, serialised per-launch times; use the shares, not the absolute ms.\n")
    print("| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / tot:.1f}% |")
    print(f"| total | {sum(cnt.values())} | {tot:.3f} | 100% |")


if __name__ == "__main__":
    main()
