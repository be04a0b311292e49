"""Stall samples per straight-line SASS segment of one kernel in an ncu report (with --import-source):
python tools/stall_segments.py REPORT KERNEL_REGEX [top]."""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[1]
    rows = []
    for x in r[2:]:
        if x and x[0] == "Kernel Name":
            break
        if len(x) == len(h):
            rows.append(x)
    iE, iS, iN = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
    segs, cur = [], None
    for n, x in enumerate(rows):
        e = int(x[iE] or 0)
        if cur is None or e != cur["e"]:
            cur = {"a": n, "b": n, "e": e, "samples": 0, "st": {}}
            segs.append(cur)
        cur["b"] = n
        cur["samples"] += int(x[iN] or 0)
        for i in stall_cols:
            v = int(x[i] or 0)
            if v:
                cur["st"][h[i]] = cur["st"].get(h[i], 0) + v
    tot = sum(sg["samples"] for sg in segs)
    for sg in sorted(segs, key=lambda s: -s["samples"])[:top]:
        st = sorted(sg["st"].items(), key=lambda kv: -kv[1])[:4]
        print(f"[{sg['a']:5d}-{sg['b']:5d}] x{sg['e']:8d} len {sg['b'] - sg['a'] + 1:4d} samples {sg['samples']:6d} "
              f"({100 * sg['samples'] / max(tot, 1):4.1f}%) " + " ".join(f"{k[6:]}={v}" for k, v in st) +
              f"  | {rows[sg['a']][iS][:50]}")


if __name__ == "__main__":
    main()
