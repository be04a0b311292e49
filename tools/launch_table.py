"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum CSV launch list
(python tools/launch_table.py LAUNCHES.csv [steps]): launches per step, mean us, share."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    order = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"][:60]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        if k not in tot:
            order.append(k)
        tot[k] += us
        cnt[k] += 1
    allt = sum(tot.values())
    for k in order:
        print(f"{k:60s} {cnt[k] / steps:5.1f}/step {tot[k] / cnt[k]:8.2f} us  {100 * tot[k] / allt:5.1f}%")
    print(f"total per step {allt / steps:.1f} us")


if __name__ == "__main__":
    main()
