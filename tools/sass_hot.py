"""Hot SASS segments of one kernel in an ncu report (python tools/sass_hot.py REPORT KERNEL_REGEX [min_M]).

Prints the instruction mix and the straight-line segments (runs of instructions with the same
execution count) that together make up the kernel's executed warp instructions."""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[1]
    rows = []
    for x in r[2:]:  # first kernel section only (several launches may match)
        if x and x[0] == "Kernel Name":
            break
        if len(x) == len(h):
            rows.append(x)
    iE, iS = h.index("Instructions Executed"), h.index("Source")
    tot = sum(int(x[iE]) for x in rows)
    print(r[0][1][:100], f"total {tot / 1e6:.2f}M warp instructions")
    ops = collections.Counter()
    for x in rows:
        t = x[iS].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[op.split(".")[0]] += int(x[iE])
    print("  ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(16)))
    segs, prev, start = [], None, 0
    for i, x in enumerate(rows):
        c = int(x[iE])
        if c != prev:
            if prev is not None:
                segs.append((start, i - 1, prev))
            prev, start = c, i
    segs.append((start, len(rows) - 1, prev))
    for a, b, c in segs:
        n = b - a + 1
        if c * n >= thr * 1e6:
            print(f"  [{a:5d}-{b:5d}] {c:9d} x {n:4d} = {c * n / 1e6:7.2f}M  {rows[a][iS].strip()[:60]}")


if __name__ == "__main__":
    main()
