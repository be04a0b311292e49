"""Summarise ncu output into profiles/ (python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.md).

REPORT is one `ncu --set full --clock-control none --import-source on` capture of
tools/profile_step.py (one headline step); LAUNCHES is the `--metrics gpu__time_duration.sum`
launch list of `bench.py --steps 2 --warmup 3`.  Writes a markdown table per kernel: duration,
DRAM bytes, issue activity, occupancy and the top stall reasons, plus the per-step share of each
kernel in the launch list."""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "not_selected", "selected", "math_pipe_throttle",
          "branch_resolving", "barrier", "dispatch_stall", "mio_throttle", "lg_throttle", "no_instructions"]


BYTES_TO_MB = {"byte": 1e-6, "B": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}
TIME_TO_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
# launched by bench.py around the step, not part of it: the L2 flush and the FP32 peak measurement
NOT_STEP = ("FillFunctor", "ffma_peak_kernel", "mma_selftest")


def ncu_raw(rep):
    cols = METRICS + [f"smsp__pcsamp_warps_issue_stalled_{s}" for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(cols)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def short(name):
    name = name.split("(")[0]
    for p in ("void ", "lgs::", "cub::", "at::native::"):
        name = name.replace(p, "")
    return name[:48]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        if any(x in d["Kernel Name"] for x in NOT_STEP):
            continue
        us = float(d["Metric Value"].replace(",", "")) * TIME_TO_US[d.get("Metric Unit", "ns")]
        k = short(d["Kernel Name"])
        per.setdefault(k, []).append(us)
    return per


def main():
    rep, lcsv, out = sys.argv[1:4]
    hdr, units, data = ncu_raw(rep)
    ix = {n: i for i, n in enumerate(hdr)}
    lines = [f"# ncu summary: `{rep.split('/')[-1]}`", "",
             "One headline step (tools/profile_step.py c1_500k 1: 640x480, 500k Gaussians, SH3, 16-D "
             "features, fused L1, pose gradient), `ncu --set full --clock-control none --import-source on`. "
             "Per-launch times are cold-cache and serialised (replay); shares, not absolutes, carry over "
             "to bench.py.", "",
             "| kernel | us | DRAM MB (r+w) | issue % elapsed | issue % active | warps % | regs | grid x block | "
             "warp inst (M) | top stalls (pc samples) |", "|---|---|---|---|---|---|---|---|---|---|"]
    for r in data:
        def g(n, f=float):
            try:
                return f(r[ix[n]].replace(",", ""))
            except (KeyError, ValueError):
                return float("nan")
        st = sorted(((g(f"smsp__pcsamp_warps_issue_stalled_{s}"), s) for s in STALLS), reverse=True)[:3]
        tot = sum(g(f"smsp__pcsamp_warps_issue_stalled_{s}") for s in STALLS) or 1.0
        mb = (g("dram__bytes_read.sum") * BYTES_TO_MB[units[ix["dram__bytes_read.sum"]]]
              + g("dram__bytes_write.sum") * BYTES_TO_MB[units[ix["dram__bytes_write.sum"]]])
        t = g("gpu__time_duration.sum") * TIME_TO_US[units[ix["gpu__time_duration.sum"]]]
        lines.append(
            f"| {short(r[ix['Kernel Name']])} | {t:.1f} | {mb:.1f} | {g('sm__issue_active.avg.pct_of_peak_sustained_elapsed'):.0f} | "
            f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
            f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | {g('launch__registers_per_thread'):.0f} | "
            f"{g('launch__grid_size'):.0f} x {g('launch__block_size'):.0f} | {g('smsp__inst_executed.sum') / 1e6:.1f} | "
            + ", ".join(f"{s} {100 * v / tot:.0f}%" for v, s in st) + " |")
    per = launches(lcsv)
    total = sum(sum(v) for v in per.values())
    lines += ["", f"## Launch list `{lcsv.split('/')[-1]}` (bench.py --steps 2 --warmup 3: warm-up, timed and "
              "phase-profile steps; the L2-flush fills and the FP32-peak microbenchmark excluded)", "", "| kernel | launches | mean us | share of GPU time |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
