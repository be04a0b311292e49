"""Markdown table of the last timed plan replay in an ncu launch list (bench.py --steps 3 under
`ncu --metrics gpu__time_duration.sum --csv`): the kernels from the preprocess_kernel
launch before the last fused blend up to the next preprocess_kernel,
each with grid, duration and share.  python tools/last_replay.py CONFIG LAUNCHES.csv"""
import csv
import sys


def main():
    name, path = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i], rows[i + 1:]
    col = {h: j for j, h in enumerate(hdr)}
    kern = [(r[col["Kernel Name"]], r[col["Grid Size"]], float(r[col["Metric Value"]]) / 1e3) for r in data
            if r[col["Metric Name"]] == "gpu__time_duration.sum"]
    short = [x[0].split("(")[0].split("<")[0].split("::")[-1] for x in kern]
    kern = [(n, g, t) for n, (_, g, t) in zip(short, kern)]
    last = max(k for k, x in enumerate(kern) if x[0].startswith("blend_fused"))
    start = max(k for k, x in enumerate(kern[:last]) if x[0] == "preprocess_kernel")
    end = next((k for k in range(last, len(kern)) if kern[k][0] == "preprocess_kernel"), len(kern))
    rep = [x for x in kern[start:end] if x[0] not in ("ffma_peak_kernel", "l2_flush_kernel", "vectorized_elementwise_kernel", "fill_kernel")]
    tot = sum(x[2] for x in rep)
    print(f"## {name}: {len(rep)} kernels, {tot:.1f} µs serialised\n")
    print("| kernel | grid | µs | share |\n|---|---|---|---|")
    for k, g, t in rep:
        print(f"| {k.split('(')[0][:48]} | {g} | {t:.1f} | {100 * t / tot:.1f} % |")
    print()


if __name__ == "__main__":
    main()
