#!/usr/bin/env python
"""Benchmark: fwd+bwd render iterations/s, 640x480 RGB + depth + 16-D feature, 500k Gaussians.

BASELINE.json metric, configs[1] distributions at the metric's 500k Gaussians (SH degree 3,
16-D normalized features, identity pose), seeded synthetic inputs (no dataset ships with the
reference).  One step = one view: preprocess -> binning -> blend forward with the
fused L1 loss -> blend backward -> preprocess backward (all map gradients + the 6-DoF pose
gradient, read back to the host).  With N > 1 (torchrun) every rank renders its own view of the
replicated map and the flat fp32 gradient (500k x 75 floats) is all-reduced over NCCL (weak
scaling: one view per GPU per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W >= 3 untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
library's stream, with a 512 MiB L2 flush (not timed) before every step; barrier + synchronize
on both sides; max over ranks.  SM clocks and throttle reasons are sampled through NVML between
the timed steps (outside each step's event bracket).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd render iters/s, 640x480 RGB+depth+16-D feat, 500k Gaussians"
UNIT = "it/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c1_500k",
                   help="c0 | c1 | c1_500k (headline) | c2 | c4 (one view of the 16-view arc) | c3")
    p.add_argument("--view", type=int, default=None, help="camera of the config (default 0; c4: 8, mid-arc)")
    p.add_argument("--multiview", choices=["auto", "none", "c3", "c4"], default="auto",
                   help="also time a multi-view mapping batch (BASELINE configs 3/4); auto: c3 with c1_500k")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-mapping", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-pruning", action="store_true")
    p.add_argument("--no-speculative-plans", action="store_true",
                   help="always capture the layered binning's second pass (LGS_OPT_SPECULATIVE_PLANS = 0)")
    p.add_argument("--rng", choices=["pcg64", "reference"], default="pcg64",
                   help="scene generator: numpy PCG64, or the reference's lego::Rng stream (scenes.RefRng)")
    p.add_argument("--e2e-steps", type=int, default=30)
    p.add_argument("--e2e-threads", type=int, default=0,
                   help="host threads of the e2e leg (0: 6 up to 1M Gaussians, else 3)")
    p.add_argument("--sampler", choices=["nvml", "smi", "none"], default="nvml", help=argparse.SUPPRESS)
    return p.parse_args()


class NvmlClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML during the timed region.

    Samples are taken by the benchmark thread BETWEEN steps (after a step's end event, before the
    next step's L2 flush), never concurrently with a step: an NVML query takes a driver lock, and a
    sampling thread (or an nvidia-smi process) polling during a step stalled single steps by up to
    37 ms on the box."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.smax = [], set(), None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # first queries are slow (driver state setup): take them before the timed region starts
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.ok = True
        except Exception:  # NVML unavailable: fall back to nvidia-smi after the region
            self.ok = False
        return self

    def sample(self):
        """One sample; call between steps while the GPU is still busy with the previous one."""
        if not self.ok:
            return
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def __exit__(self, *a):
        pass

    def summary(self):
        if not self.ok or not self.samples:
            return ClockSampler.snapshot(self.index)
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "nvml, sampled between timed steps"}


class NullSampler:
    def __init__(self, index):
        self.index = index

    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def sample(self):
        pass

    def summary(self):
        return ClockSampler.snapshot(self.index)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    @staticmethod
    def snapshot(index):
        s = ClockSampler(index)
        s.__enter__()
        time.sleep(0.3)
        s.__exit__()
        out = s.summary()
        out["source"] = "nvidia-smi (after the timed region)"
        return out

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def sample(self):
        pass

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload_metric(cam, n, d):
    """BASELINE metric string for a workload (the headline's is METRIC)."""
    ng = f"{n // 1000}k" if n < 1_000_000 else f"{n / 1e6:g}M"
    return f"fwd+bwd render iters/s, {cam['width']}x{cam['height']} RGB+depth+{d}-D feat, {ng} Gaussians"


def default_view(config):
    return 8 if config == "c4" else 0


def rank_camera(base_cam, rank, world):
    """Rank r renders the headline view translated by 2 cm per rank (same work, distinct views)."""
    import numpy as np
    cam = dict(base_cam)
    if world > 1:
        cam["t"] = np.array([0.02 * rank, 0.0, 0.0])
    return cam


def traffic_for(phase):
    """DRAM bytes per launch of the phase's kernel from one `ncu --set full` capture, committed in
    profiles/traffic.json (bench.py cannot run ncu itself); None when not recorded."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    ent = rec.get(phase)
    return int(ent["dram_bytes_per_launch"]) if ent else None


def measure_fp32_peak(device):
    """FFMA throughput of this device (TFLOP/s) from the bench-only microbenchmark library
    (paper_2511_16144_b200/bench_csrc, built by build.py; not part of liblgs.so)."""
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "paper_2511_16144_b200", "libbench_peak.so"))
    lib.bench_measure_fp32_peak.restype = C.c_int
    lib.bench_measure_fp32_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    v = C.c_double()
    if lib.bench_measure_fp32_peak(device, C.byref(v)) != 0:
        raise RuntimeError("FP32 peak microbenchmark failed")
    return v.value


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_16144_b200 import _lib
    from paper_2511_16144_b200 import renderer as R
    from paper_2511_16144_b200 import scenes

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    _lib.load()  # fails loudly without the CUDA library: there is no fallback

    scene, cams, info = scenes.make_config(args.config, rng=args.rng)
    view = default_view(args.config) if args.view is None else args.view
    cam = rank_camera(cams[view], rank, world)
    d = scene["feat"].shape[0]
    K = scene["sh"].shape[1]
    n = scene["pos"].shape[0]
    tg = scenes.make_targets(cam, d, info["depth_range"], 7 + rank)

    stream = torch.cuda.Stream(device=local)
    ctx = R.Context(local, stream=stream.cuda_stream, speculative_plans=not args.no_speculative_plans)
    with torch.cuda.stream(stream):
        dscene = {k: torch.from_numpy(v).cuda(local) for k, v in scene.items()}
        dtg = {k: torch.from_numpy(v).cuda(local) for k, v in tg.items()}
        dmap = R.DeviceMap(dscene, ctx)
        grads = R.alloc_grads(n, d, K, device=local)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    del dscene
    comm = None
    if world > 1:
        from paper_2511_16144_b200.multiview import NativeComm
        comm = NativeComm(ctx)  # liblgs.so's own NCCL communicator (torch.distributed only bootstraps it)

    pose_host = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    H, W = cam["height"], cam["width"]
    with torch.cuda.stream(stream):
        imgs = {"rgb": torch.empty(H, W, 3, device=f"cuda:{local}"), "depth": torch.empty(H, W, device=f"cuda:{local}"),
                "feat": torch.empty(H, W, d, device=f"cuda:{local}"), "acc": torch.empty(H, W, device=f"cuda:{local}")}
        # the step as ONE CUDA graph: render (fused L1, images written) -> backward (all map grads,
        # pose grad copied to pinned host memory in stream order); lgs_plan, include/lgs.h
        plan = R.Plan(dmap, cam, dtg, grads, images=imgs, pose_out=pose_host)

    def enqueue():
        plan.run()
        if comm is not None:
            # the view's step must be final before the exchange (a re-run after a tile-list overflow
            # would otherwise leave this rank's sum stale on every rank): wait, then enqueue the sum
            # over ranks of the 500k x 75 fp32 gradient exchanging only the rows some view reached
            # (lgs_allreduce_grads_sparse_async: capacity-sized row blocks, no host wait inside;
            # dense NCCL all-reduce when the rows are not sparse)
            plan.sync()
            comm.all_reduce_grads_sparse_async(dmap, grads)
        return None

    def finish():
        plan.sync()  # the step's pose gradient has reached the host (re-captures on overflow)
        if comm is not None:
            comm.wait_grads_sparse(dmap, grads)  # exact re-run if a rank outgrew the capacity

    def step():
        """Eager (uncaptured) step through the same API: used for the per-phase profile."""
        out = R.render(dmap, cam, targets=dtg, ctx=ctx)
        R.render_backward_loss_async(out, into=grads, pose_out=pose_host)
        if comm is not None:
            comm.all_reduce_grads_sparse(dmap, grads)
        torch.cuda.current_stream().synchronize()
        return out, grads

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            enqueue()
            finish()
    torch.cuda.synchronize()

    # ---- timed region --------------------------------------------------------------------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    sampler = {"nvml": NvmlClockSampler, "smi": ClockSampler, "none": NullSampler}[args.sampler]
    every = max(1, args.steps // 40)  # ~40 clock samples over the timed region
    gc.collect()
    gc.disable()  # a collection inside a step stalls the host-driven pipeline
    with sampler(local) as clk, torch.cuda.stream(stream):
        host_ms = []
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            h0 = time.perf_counter()
            out = enqueue()
            evs[k][1].record(stream)  # on the stream before the host waits: host wake-up is outside
            host_ms.append(1e3 * (time.perf_counter() - h0))
            finish()
            if k % every == every - 1:
                clk.sample()
        torch.cuda.synchronize()
    gc.enable()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    per_step = [a.elapsed_time(b) for a, b in evs]
    ms = sum(per_step) / len(per_step)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * 1000.0 / ms_max

    # ---- phase profile (separate, untimed passes) -----------------------------------------------
    # per-phase device times of the captured step itself: events recorded inside the graph, over
    # n_prof replays with the same L2 flush; the work counters come from one eager profiled render
    n_prof = 5
    acc_ph = {}
    plan.set_profiling(True)
    with torch.cuda.stream(stream):
        for k in range(n_prof):
            flush.fill_(float(k))
            enqueue()
            finish()
            for name, v in plan.phase_times().items():
                acc_ph[name] = acc_ph.get(name, 0.0) + v
    phases = {k: (v / n_prof, 1) for k, v in acc_ph.items()}
    plan.set_profiling(False)
    ctx.profile(True)
    with torch.cuda.stream(stream):
        out, g = step()
    torch.cuda.synchronize()
    ctx.profile(False)
    ctx.phase_times()  # discard the eager marks
    st = out.stats()
    evaluated, contributed = out.work()
    peak = {}
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = float(peak.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peak else "B200_PROFILING.md fallback"
    fp32 = measure_fp32_peak(local)

    # algorithmic work per launch
    npix = cam["width"] * cam["height"]
    V, P, LST, A = st["visible"], st["pairs"], st["listed"], st["active"]
    ntiles = ((cam["width"] + 15) // 16) * ((cam["height"] + 15) // 16)
    F_EVAL, F_FWD, F_BWD = 13.0, 45.0, 100.0
    # algorithmic bytes: preprocess = parameters read + records written (+ the
    # 8 B depth-bucket slot / atomic); depth order = the 2^18-bucket u64 scan, key read and
    # (key, index) scatter of the visible Gaussians, + the listed Gaussians' SH rows and colours; binning (depth-layered) = the listed pairs
    # written and ranges, each tile reading the layer-A candidate rects is not counted
    work = {
        # (layered: K1 reads no SH and writes no colour; the colours of the A active Gaussians are
        # evaluated where the depth order first lists them)
        "preprocess": ("hbm", n * 16 * 3 + n * (16 * 2 + 8 + 12) + V * 8),
        "depth_sort_scan": ("hbm", 2 * 8 * (1 << 18) + n * 4 + V * 8 + A * (12 * K + 16)),
        "duplicate_keys": ("hbm", V * 16 + P * 6),
        "tile_sort_ranges": ("hbm", LST * 4 + ntiles * 8),
        "blend_fwd": ("fp32", F_EVAL * evaluated + F_FWD * contributed),
        "blend_bwd": ("fp32", F_EVAL * evaluated + F_BWD * contributed),
        # the chain over the A active rows (flags scanned, accumulator + map rows read, rows written);
        # the zero rows of every other Gaussian stream out in grad_zero (a side branch in the plan)
        "preprocess_bwd": ("hbm", n + A * (16 * 3 + 12 * K + 16 + 128) + A * 4 * (11 + 3 * K + d)),
        "grad_zero": ("hbm", n * 4 * (11 + 3 * K + d)),
    }
    if "blend_bwd" not in phases and "blend_fwd" in phases:  # captured fused-L1 step: one kernel
        phases["blend_fused"] = phases.pop("blend_fwd")
        work["blend_fused"] = ("fp32", 2 * F_EVAL * evaluated + (F_FWD + F_BWD) * contributed)
    phase_rows = {}
    for name, (pms, cnt) in phases.items():
        if name not in work:
            continue
        bound, amount = work[name]
        if bound == "hbm":
            ach = amount / (pms * 1e-3) / 1e9
            frac = ach / hbm_peak
            phase_rows[name] = {"ms": round(pms, 4), "bound": "hbm", "achieved": round(ach, 1), "unit": "GB/s",
                                "frac": round(frac, 4), "algorithmic_bytes": int(amount)}
        else:
            ach = amount / (pms * 1e-3) / 1e12
            phase_rows[name] = {"ms": round(pms, 4), "bound": "fp32", "achieved": round(ach, 3), "unit": "TFLOP/s",
                                "frac": round(ach / fp32, 4), "algorithmic_flops": int(amount)}
    dom = max(phase_rows, key=lambda k: phase_rows[k]["ms"])
    dr = phase_rows[dom]
    t_roof = 0.0
    for name, row in phase_rows.items():
        if row["bound"] == "hbm":
            t_roof += row["algorithmic_bytes"] / (hbm_peak * 1e9)
        else:
            t_roof += row["algorithmic_flops"] / (fp32 * 1e12)
    roofline = {
        "kernel": dom,
        "bound": dr["bound"],
        "achieved": dr["achieved"],
        "peak": round(hbm_peak if dr["bound"] == "hbm" else fp32, 2),
        "peak_source": hbm_src if dr["bound"] == "hbm" else "bench_measure_fp32_peak (FFMA microbenchmark, this box; libbench_peak.so)",
        "unit": dr["unit"],
        "frac": dr["frac"],
        "traffic": traffic_for(dom),
        "step_t_roof_ms": round(t_roof * 1e3, 4),
        "step_frac": round(t_roof * 1e3 / ms_max, 4),
        "phases": phase_rows,
    }

    data = {"c0": "configs[0]", "c1": "configs[1]", "c1_500k": "configs[1] distributions at 500k",
            "c2": "configs[2] (200 blobs, Replica-shaped)", "c3": "configs[3] map",
            "c4": f"configs[4] (70% in a 0.5 m ball), view {view} of the 16-view arc"}[args.config]
    result = {
        "metric": METRIC if args.config == "c1_500k" else workload_metric(cam, n, d), "value": round(value, 3),
        "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_max, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded, {args.rng} generator; BASELINE {data}; no dataset ships with the reference)",
        "config": {"workload": args.config, "view": view, "image": f"{cam['width']}x{cam['height']}", "gaussians": n,
                   "sh_degree": int(math.isqrt(K) - 1), "feature_dim": d, "views_per_gpu_per_step": 1,
                   "loss": "L1 rgb+depth+feat (fused)", "pose_grad": True,
                   "parallelism": (f"views over {world} GPU(s), fp32 row-sparse grad all-reduce by liblgs.so (NCCL)"
                                   if world > 1
                                   else "1 GPU"),
                   "l2": "512 MiB L2 flush before every timed step"},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        # speculative: the plan was captured without the layered binning's second pass (every tile
        # saturated on its first-pass list at warm-up); recaptures: steps sync() re-ran
        "plan": {"speculative": plan.speculative, "recaptures": plan.recaptures},
        "roofline": roofline,
        "work": {"visible": V, "pairs": P, "listed": LST, "active": A, "evaluated": evaluated, "contributed": contributed,
                 "max_tile_list": st["max_tile_list"]},
        "per_step_ms": [round(x, 4) for x in per_step],
        "host_enqueue_ms": [round(x, 3) for x in host_ms],
    }

    if not args.no_mapping:
        result["mapping_step"] = run_mapping_step(args, dmap, cam, ctx, stream, flush, info, hbm_peak, fp32, local)

    # ---- end to end through the public API with host buffers -----------------------------------
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, scene, cam, tg, R, local)
        # the same with the whole map copied every step (LGS_MEM_HOST): 150 MB more H2D per step
        full = run_e2e(args, scene, cam, tg, R, local, mapped=False)
        result["e2e"]["whole_map_copied"] = {k: full[k] for k in ("value", "ms_per_step", "h2d_bytes_per_step")}
        # and with every gradient row downloaded every step (no delta rows): 150 MB D2H per step
        dense = run_e2e(args, scene, cam, tg, R, local, delta=False)
        result["e2e"]["dense_grad_download"] = {k: dense[k] for k in ("value", "ms_per_step", "d2h_bytes_per_step")}
        result["e2e"]["dense_grad_download"]["single_thread"] = dense["single_thread"]

    mv = args.multiview if args.multiview != "auto" else ("c3" if args.config == "c1_500k" else "none")
    if mv != "none":
        result["multiview_batch"] = run_multiview(args, mv, local, world, rank, flush)

    if rank == 0 and world == 1 and not args.no_pruning:
        result["pruning"] = run_pruning(local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(scene, cam, tg, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def run_mapping_step(args, dmap, cam, ctx, stream, flush, info, hbm_peak, fp32, device):
    """Secondary line: one full mapping iteration on the same map and view:
    render -> lgs_mapping_loss (0.8 L1 + 0.2 D-SSIM, masked depth L1, 16->64->32 decoder chain)
    -> backward -> per-attribute Adam step, all on the device, timed like the headline step."""
    import numpy as np
    import torch

    from paper_2511_16144_b200 import renderer as R
    from paper_2511_16144_b200 import scenes

    H, W = cam["height"], cam["width"]
    D = 32
    r = np.random.default_rng(11)
    lo, hi = info["depth_range"]
    kd = r.uniform(lo, hi, (H, W)).astype(np.float32)
    kd[r.uniform(size=(H, W)) < 0.1] = 0.0
    with torch.cuda.stream(stream):
        kf = {"rgb": torch.from_numpy(r.uniform(0, 1, (H, W, 3)).astype(np.float32)).cuda(device),
              "depth": torch.from_numpy(kd).cuda(device),
              "feat_gt": torch.from_numpy(r.normal(0, 0.5, (H, W, D)).astype(np.float32)).cuda(device)}
        dec = tuple(torch.from_numpy(x).cuda(device) for x in scenes.make_decoder(D, 64, dmap.d, 1))
        grads = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=device)
        opt = R.Adam(dmap)

    def step():
        out = R.render(dmap, cam, ctx=ctx)
        R.mapping_loss(out, kf, dec, readback=False)
        R.render_backward_loss(out, into=grads)
        opt.step(grads)
        return out

    steps = max(10, min(args.steps, 50))
    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        ctx.profile(True)
        n_prof = 5
        for k in range(n_prof):
            flush.fill_(float(k))
            step()
        torch.cuda.synchronize()
        ph = {k: v[0] / n_prof for k, v in ctx.phase_times().items() if v[1]}
        ctx.profile(False)
    npix = H * W
    q = 11 + 3 * dmap.K + dmap.d
    loss_bytes = npix * 416  # stencils 2 x (rgb, gt, depth, acc, kf depth, A/B/C) + decoder feat, F_gt, cotangents
    dec_flops = 2.0 * npix * 2 * 64 * (dmap.d + D)
    adam_bytes = dmap.n * 4 * q * 7  # params + 2 moments read and written, gradients read
    rows = {}
    if "mapping_loss" in ph:
        t = ph["mapping_loss"] * 1e-3
        rows["mapping_loss"] = {"ms": round(ph["mapping_loss"], 4), "algorithmic_bytes": loss_bytes,
                                "algorithmic_flops": int(dec_flops),
                                "t_roof_ms": round(1e3 * (loss_bytes / (hbm_peak * 1e9) + dec_flops / (fp32 * 1e12)), 4),
                                "frac": round((loss_bytes / (hbm_peak * 1e9) + dec_flops / (fp32 * 1e12)) / t, 4)}
    if "adam" in ph:
        t = ph["adam"] * 1e-3
        rows["adam"] = {"ms": round(ph["adam"], 4), "bound": "hbm", "algorithmic_bytes": adam_bytes,
                        "achieved_gbs": round(adam_bytes / t / 1e9, 1), "frac": round(adam_bytes / t / 1e9 / hbm_peak, 4)}
    for k in ("preprocess", "depth_sort_scan", "tile_sort_ranges", "blend_fwd", "blend_bwd", "grad_zero", "preprocess_bwd"):
        if k in ph:
            rows[k] = {"ms": round(ph[k], 4)}
    return {"metric": "mapping iterations/s (render + loss + backward + Adam), same map and view", "value":
            round(1000.0 / ms, 3), "unit": "it/s", "ms_per_step": round(ms, 4), "steps": steps, "teacher_dim": D,
            "decoder": f"{dmap.d}->64->{D}", "phases": rows}


def run_multiview(args, name, local, world, rank, flush):
    """BASELINE configs[3] (c3: 500k Gaussians, 8 views on a 1 m circle) or configs[4] (c4: 3M, 16 views
    on a 2 m arc) as one data-parallel mapping batch: the views are split over the ranks (longest
    processing time first on their pair counts -- deterministic, so every rank derives the same
    split), each rank runs its views as captured steps accumulating into one gradient buffer
    (lgs_plan, accumulate), and the batch gradient is summed over ranks by the row-sparse exchange
    (lgs_allreduce_grads_sparse_async).  T(N) = max over ranks of the batch step (device events);
    value = views per second of the whole batch.  The view total is fixed (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_16144_b200 import multiview
    from paper_2511_16144_b200 import renderer as R
    from paper_2511_16144_b200 import scenes

    scene, cams, info = scenes.make_config(name, rng=args.rng)
    n, d, K = scene["pos"].shape[0], scene["feat"].shape[0], scene["sh"].shape[1]
    stream = torch.cuda.Stream(device=local)
    ctx = R.Context(local, stream=stream.cuda_stream)
    with torch.cuda.stream(stream):
        dmap = R.DeviceMap({k: torch.from_numpy(v).cuda(local) for k, v in scene.items()}, ctx)
        tgs = [{k: torch.from_numpy(v).cuda(local) for k, v in
                scenes.make_targets(c, d, info["depth_range"], 50 + v).items()} for v, c in enumerate(cams)]
        grads = R.alloc_grads(n, d, K, device=local)
        costs = [R.render(dmap, c, targets=tgs[v], ctx=ctx).stats()["pairs"] for v, c in enumerate(cams)]
    del scene
    mine = multiview.assign_views(len(cams), world, rank, costs)
    comm = multiview.NativeComm(ctx) if world > 1 else None
    poses = [torch.zeros(6, dtype=torch.float32, pin_memory=True) for _ in mine]
    with torch.cuda.stream(stream):
        plans = [R.Plan(dmap, cams[v], tgs[v], grads, pose_out=poses[i], accumulate=i > 0) for i, v in enumerate(mine)]

    def step():
        for p in plans:
            p.run()
        if comm is not None:
            # every view final before the exchange (a view that outgrew its lists or missed its
            # speculation re-runs here; renderer.sync_plans)
            R.sync_plans(plans)
            comm.all_reduce_grads_sparse_async(dmap, grads)

    def finish():
        R.sync_plans(plans)
        return comm.wait_grads_sparse(dmap, grads) if comm is not None else 0

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
            finish()
    torch.cuda.synchronize()
    steps = max(5, min(args.steps, 20))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    rows = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for k in range(steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
            rows.append(finish())
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in evs]
    ms = sum(per) / len(per)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        comm.close()
    ms_max = float(t.item())
    recaptures = sum(p.recaptures for p in plans)
    del plans
    return {"metric": f"views/s of the {len(cams)}-view mapping batch (fwd+bwd per view + gradient sum over ranks)",
            "value": round(len(cams) * 1000.0 / ms_max, 3), "unit": "views/s", "n_gpus": world,
            "ms_per_step": round(ms_max, 4), "steps": steps, "scaling": "strong",
            "config": {"workload": name, "views": len(cams), "gaussians": n, "image": f"{cams[0]['width']}x"
                       f"{cams[0]['height']}", "views_this_rank": mine, "pairs_per_view": [int(c) for c in costs],
                       "exchange": "row-sparse all-gather (lgs_allreduce_grads_sparse_async)" if world > 1 else
                       "none (1 GPU: the views accumulate into one buffer)",
                       "l2": "512 MiB L2 flush before every timed step"},
            "rows_max": int(max(rows)) if rows else 0, "plan_recaptures": int(recaptures),
            "per_step_ms": [round(x, 4) for x in per]}


def pinned_like(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def run_e2e(args, scene, cam, tg, R, device, mapped=True, delta=True):
    """Same step through the reference-facing API with HOST buffers: every step uploads the map
    and targets (H2D), renders, reads back the images, the gradients, the pose gradient and the
    loss (D2H).  PCIe, not the GPU, bounds this path (~350 MB moved per step), so the headline
    number runs ``--e2e-threads`` host threads, each with its own context / stream and its own
    output buffers, rendering concurrently as the reference API allows (renders are pure with
    respect to the map): one thread's gradient download overlaps the next
    thread's map upload on the full-duplex link.  The single-thread number is reported beside it.

    ``mapped`` (the headline): the host map is page-locked and passed as LGS_MEM_HOST_MAPPED, so
    positions / rotations / scales / opacities are copied (22 MB) while the SH rows and features of
    just the listed Gaussians are read in place over PCIe; otherwise the whole map is copied.
    ``delta`` (the headline): each worker passes the same host gradient buffers to every backward
    and its context runs LGS_OPT_HOST_GRAD_DELTA -- the buffers hold the dense MapGradients after
    every call, but only the rows nonzero now cross the link (the rows nonzero in the previous call
    are zeroed on the host); otherwise all 150 MB come back every step.  Bytes per step are the
    library's own copy counters (lgs_ctx_transfer_bytes) plus the mapped-memory reads."""
    import numpy as np
    import torch

    hscene = {k: pinned_like(v) for k, v in scene.items()}
    htg = {k: pinned_like(v) for k, v in tg.items()}
    H, W = cam["height"], cam["width"]
    d = scene["feat"].shape[0]
    n = scene["pos"].shape[0]
    K = scene["sh"].shape[1]
    total = n * (11 + 3 * K + d)

    class Worker:
        def __init__(self):
            self.img = {"rgb": pinned_like(np.zeros((H, W, 3), np.float32)),
                        "depth": pinned_like(np.zeros((H, W), np.float32)),
                        "feat": pinned_like(np.zeros((H, W, d), np.float32)),
                        "acc": pinned_like(np.zeros((H, W), np.float32))}
            self.flat = pinned_like(np.zeros(total, np.float32))
            self.grads = R.alloc_grads(n, d, K, flat=self.flat)
            self.ctx = R.Context(device, stream="own", host_grad_delta=delta)
            self.loss = None

        def step(self):
            out = R.render(hscene, cam, targets=htg, ctx=self.ctx, out=self.img, host_mapped=mapped)
            R.render_backward_l1(out, pose=True, into=self.grads)
            self.loss = out.l1_loss()

    def timed(workers, steps):
        for w in workers:  # warm-up (allocator pools, pinned staging)
            w.step()
            w.step()
        torch.cuda.synchronize()
        errs = []
        b0 = [w.ctx.transfer_bytes() for w in workers]

        def loop(w):
            try:
                for _ in range(steps):
                    w.step()
            except Exception as e:  # surfaced below
                errs.append(e)

        ths = [threading.Thread(target=loop, args=(w,)) for w in workers]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if errs:
            raise errs[0]
        b1 = [w.ctx.transfer_bytes() for w in workers]
        per = steps * len(workers)  # bytes the library copied per timed step (its own counters)
        moved = (sum(b[0] - a[0] for a, b in zip(b0, b1)) / per, sum(b[1] - a[1] for a, b in zip(b0, b1)) / per)
        return 1e3 * dt / per, moved

    # host threads, each with its own context: PCIe transfers of one overlap the others' compute;
    # 6 measured +10% over 3 at the headline (profiles/r2_e2e_threads.log), big maps keep 3
    # (each context holds its own tile-list blocks: 2 x 8.8 GB at configs[4])
    nthreads = args.e2e_threads if args.e2e_threads > 0 else (6 if n <= 1_000_000 else 3)
    workers = [Worker() for _ in range(nthreads)]
    # three measurement windows, the median reported: concurrent host-mapped contexts occasionally
    # stall for hundreds of ms together (PCIe zero-copy reads beside other contexts' DMA), which
    # one window of 30 steps cannot average out; every window is in the JSON
    windows = [timed(workers, args.e2e_steps) for _ in range(3)]
    wms = sorted(w[0] for w in windows)
    ms = wms[1]
    h2d, d2h = windows[0][1]
    # single-threaded: the same three-window median (a window with one of the rare host stalls
    # would otherwise stand for the whole figure); all windows listed
    w1 = sorted(timed(workers[:1], args.e2e_steps)[0] for _ in range(3)) if nthreads > 1 else wms
    ms1 = w1[1]
    d2h += 6 * 4 + 8  # + the pose gradient and the loss
    if mapped:  # + the listed Gaussians' SH rows and features read in place over PCIe (zero-copy mode)
        rows = R.render(hscene, cam, ctx=workers[0].ctx, host_mapped=True).stats()["host_rows"]
        h2d += rows * 4 * (3 * K + d)
    return {"value": round(1000.0 / ms, 3), "unit": UNIT, "ms_per_step": round(ms, 3), "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "host_threads": nthreads,
            "windows_it_s": [round(1000.0 / w[0], 1) for w in windows], "aggregate": "median of 3 windows",
            "single_thread": {"value": round(1000.0 / ms1, 3), "ms_per_step": round(ms1, 3),
                              "windows_it_s": [round(1000.0 / w, 1) for w in w1], "aggregate": "median of 3 windows"},
            "api": f"renderer.render(host numpy map{', host_mapped' if mapped else ''}, host targets) + "
                   f"render_backward_l1(host grads{', delta rows' if delta else ''}) + l1_loss(); "
                   f"{nthreads} host threads x own lgs_ctx/stream, wall clock over all steps"}


def run_pruning(device, n=500_000, reps=5):
    """the language-pruning sweep (SPEC.md Eq. 4) + geometric rule on a 500k
    cluttered map (scenes.make_prune_scene: 600 objects in a 6 m box, half the Gaussians inserted
    twice 4 mm apart), through the public API (host flags out), against the CPU: oracle/prune_oracle.c
    (the SPEC sweep, 1 thread) and the same sweep on the reference's own KdTree3 (oracle/_ref)."""
    import numpy as np
    import torch
    from paper_2511_16144_b200 import pruning as P
    from paper_2511_16144_b200 import renderer as R
    from paper_2511_16144_b200 import scenes
    s = scenes.make_prune_scene(n, seed=9, objects=600, extent=6.0)
    dm = R.DeviceMap(s, R.Context(device))
    cfg = P.PruneConfig()
    P.find_language_redundant(dm, cfg)  # warm-up (allocator, module load)
    torch.cuda.synchronize(device)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        idx = P.find_language_redundant(dm, cfg)
        t.append(time.perf_counter() - t0)
    st = P.prune_stats(dm)
    tg = []
    for _ in range(reps):
        t0 = time.perf_counter()
        gidx = P.find_geometric(dm, cfg)
        tg.append(time.perf_counter() - t0)
    out = {"workload": f"make_prune_scene({n}, objects=600, extent=6 m, 50% duplicated at 4 mm), K 8, tau 0.02 m, "
                       "tau_sim 0.9; wall time of the API call (host flags out, includes the host round checks)",
           "gpu_language_ms": round(1e3 * min(t), 3), "gpu_geometric_ms": round(1e3 * min(tg), 3),
           "removed_language": int(idx.size), "removed_geometric": int(gidx.size), **st}
    from oracle import oracle as orc
    t0 = time.perf_counter()
    want = orc.find_language_redundant(s)
    out["cpu_port_ms"] = round(1e3 * (time.perf_counter() - t0), 1)
    flags = np.zeros(n, np.uint8)
    flags[idx] = 1
    out["matches_oracle"] = bool(np.array_equal(flags, want))
    ref = _ref_build()
    if ref is not None:
        t0 = time.perf_counter()
        ref.find_language_redundant(s)
        out["cpu_ref_kdtree_ms"] = round(1e3 * (time.perf_counter() - t0), 1)
    out["cpu_cores"] = 1
    return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _ref_build():
    """oracle/_ref/liblgs_ref.so: the reference's own renderer.cpp / geometry.cpp, unmodified, compiled by
    oracle/Makefile (None where it was not built: then the oracle A port stands in)."""
    try:
        from oracle import ref
        return ref if ref.available() else None
    except Exception:  # noqa: BLE001 -- any load failure means "not available"
        return None


def _sh0(scene):
    """The reference renders colours (SH degree 0): higher bands are dropped for its arm -- the
    per-pixel work (the blend and its reverse pass) is the same, the colour is a per-Gaussian constant."""
    import numpy as np
    return dict(scene, sh=np.ascontiguousarray(scene["sh"][:, :1, :]))


def reference_step(scene, cam, tg, threads):
    """Seconds of one full fwd+bwd of the headline image on `threads` host threads (row bands) with
    the L1 cotangents: the reference itself (lego::render + lego::render_backward per band,
    ref_bridge.cpp ref_bench_bands) when oracle/_ref is built, else oracle A (the fp64 port of
    renderer.cpp:94-356).  Returns (seconds, kind)."""
    ref = _ref_build()
    if ref is not None:
        secs, _ = ref.bench_bands(_sh0(scene), cam, tg, threads, 1)
        return secs, "reference"
    from oracle import oracle as orc
    t0 = time.perf_counter()
    orc.fwd_bwd_bands(scene, cam, None, None, None, threads=threads, targets=tg)
    return time.perf_counter() - t0, "port"


def _sample_text(kind, threads, scene):
    what = ("the reference's own renderer.cpp (oracle/_ref, unmodified, compiled here against a "
            "self-written Eigen subset)" if kind == "reference" else "oracle A (fp64 port of renderer.cpp)")
    sh = "" if scene["sh"].shape[1] == 1 else "; the reference has colours only (SH degree 0): its arm renders the DC band"
    return f"{what}, full image fwd+bwd with L1 cotangents on {threads} row-band thread(s){sh}"


def cpu_baseline(scene, cam, tg, args):
    threads = cpu_threads()
    secs, kind = reference_step(scene, cam, tg, threads)
    res = {"value": round(1.0 / secs, 4), "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"1 step ({secs:.2f} s): " + _sample_text(kind, threads, scene)}
    if args.config == "c1_500k":  # single core, as the reference itself runs (~13 s here)
        one, _ = reference_step(scene, cam, tg, 1)
        res["single_core"] = {"value": round(1.0 / one, 4), "cores": 1, "sample": f"1 step ({one:.2f} s) on 1 thread"}
    return res


def run_reference(args):
    """--impl reference: the reference's own CPU renderer (oracle/_ref) -- else the oracle A port -- on
    all host cores (row bands), same metric / config.  Under torchrun only rank 0 runs."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2511_16144_b200 import scenes
    scene, cams, info = scenes.make_config(args.config, rng=args.rng)
    view = default_view(args.config) if args.view is None else args.view
    cam = cams[view]
    d = scene["feat"].shape[0]
    n = int(scene["pos"].shape[0])
    tg = scenes.make_targets(cam, d, info["depth_range"], 7)
    threads = cpu_threads()
    warm = 1  # one untimed step (page-in, allocator); each CPU step is seconds long
    for _ in range(warm):
        kind = reference_step(scene, cam, tg, threads)[1]
    steps = max(1, min(args.steps, 5))
    times = [reference_step(scene, cam, tg, threads)[0] for _ in range(steps)]
    ms = 1e3 * sum(times) / len(times)
    v = 1000.0 / ms
    res = {"metric": METRIC if args.config == "c1_500k" else workload_metric(cam, n, d), "value": round(v, 4),
           "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warm,
           "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (seeded, same as --impl ours)", "impl": "reference",
           "config": {"workload": args.config, "view": view, "image": f"{cam['width']}x{cam['height']}",
                      "gaussians": n},
           "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": f"{steps} steps (after {warm} warm-up), requested --steps {args.steps} capped "
                                      f"at 5 to bound CPU time: " + _sample_text(kind, threads, scene)},
           "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
