"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of tools/profile_step.py:
per kernel, launches and the share of the summed kernel time (setup kernels -- the map upload and
torch fills -- excluded).  python tools/launch_summary.py launches.csv [more.csv ...]"""
import csv
import re
import sys
from collections import defaultdict

SETUP = ("pack_map", "vectorized_elementwise", "gather_features", "ffma_peak")


def summary(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    name_i, val_i, unit_i = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[i + 1:]:
        name = re.sub(r"\(.*", "", r[name_i]).replace("void ", "").replace("lgs::", "")
        name = re.sub(r"<.*", "", name)
        if any(s in name for s in SETUP):
            continue
        v = float(r[val_i].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[unit_i]]
        tot[name] += v * scale
        cnt[name] += 1
    all_us = sum(tot.values())
    out = [f"| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / all_us:.1f} % |")
    out.append(f"| **all** | {sum(cnt.values())} | {all_us:.1f} | 100 % |")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"\n### {p}\n")
        print(summary(p))
