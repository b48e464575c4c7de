#!/usr/bin/env python
"""Benchmark of the hot path: Algorithm 1 reduction + skip-invalid compaction
(BASELINE.json metric: Gpoints/s reduced+compacted, % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A step = one pass of the path over one batch: K1 (chp_reduce: DL init +
Algorithm 1) then K3 (chp_compact: Lemma-1 chain + counts) over the config's
n points resident in HBM; with N > 1 ranks each rank owns n points (weak
scaling) and the partial DLs meet in one element-wise MIN all-reduce (NCCL)
before K3.  The hull (K4) is timed separately (`hull_ms`), outside `value`,
as BASELINE.json prescribes.

`e2e` is the same metric through the public C-ABI call a user makes
(chp_pipeline_host): pinned host input -> chunked H2D overlapped with K1 ->
K3 -> chain + counts back to pinned host memory, all inside the timed region.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libchpref.so: chp::reducer::reduce + build_polyline compiled
from /root/reference sources) on this host's cores over a bounded sample of
the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (n, p, seed, description)   -- BASELINE.json "configs"
    2: (100_000_000, 65536, 2, "config2: n=1e8 int32 points, x,y ~ N(p/2,(p/8)^2) rounded+clamped, p=65536"),
    3: (1_000_000_000, 16384, 3, "config3: n=1e9, uniform in the inscribed disk, p=16384"),
    4: (1_000_000_000, 1 << 20, 4, "config4: n=1e9, 64 Gaussian clusters + 1% outliers, p=2^20"),
    5: (4_000_000_000, 256, 5, "config5: n=4e9, 90% in 4 hot columns, p=256"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override points per rank (default: the config's n)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--flags", type=int, default=0, help="chp_reduce flags (variant forcing, experiments)")
    ap.add_argument("--q-unset", action="store_true",
                    help="K1 without the y bound q (the reference API's default; not the headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg_id: int, n_sample: int, p: int, seed: int, threads: int, reps: int):
    """The reference itself (oracle/_ref) on the host, or the C restatement
    when the reference library is absent.  Checker/baseline use only."""
    import numpy as np

    from paper_1505_00914_b200.device import generate_host

    xy = generate_host(cfg_id, seed, p, n_sample)
    import oracle

    if oracle.Reference.available():
        ref = oracle.Reference()
        t, s = ref.time_reduce_compact(xy, p, p, threads=threads, reps=reps)
        kind = "reference"
    else:
        orc = oracle.Oracle()
        best = 1e30
        for _ in range(reps):
            t0 = time.perf_counter()
            arr = orc.reduce(xy, p, p)
            orc.build_polyline(arr)
            best = min(best, time.perf_counter() - t0)
        t, kind, threads = best, "port", 1
    del xy
    return {"value": n_sample / t / 1e9, "unit": "Gpoints/s", "cores": threads, "kind": kind,
            "sample": f"first {n_sample:.3g} points of config {cfg_id} (same bytes as the GPU input), "
                      f"reduce+build_polyline, best of {reps}, {threads} thread(s); host {os.cpu_count()} cpus",
            "seconds": t}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    n_full, p, seed, desc = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    n_sample = min(n_full, 100_000_000)
    import numpy as np  # noqa: F401

    from paper_1505_00914_b200.device import generate_host
    import oracle

    xy = generate_host(args.config, seed, p, n_sample)
    if oracle.Reference.available():
        ref = oracle.Reference()
        kind = "reference"

        def step():
            return ref.time_reduce_compact(xy, p, p, threads=threads, reps=1)[0]
    else:
        orc = oracle.Oracle()
        kind = "port"
        threads = 1

        def step():
            t0 = time.perf_counter()
            orc.build_polyline(orc.reduce(xy, p, p))
            return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    tot = sum(times)
    value = n_sample * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": "Gpoints/s reduced+compacted", "value": value, "unit": "Gpoints/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": desc, "n_per_step": n_sample, "p": p, "seed": seed},
        "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": threads, "kind": kind,
                         "sample": f"first {n_sample:.3g} points of config {args.config} per step, "
                                   f"chp::reducer::reduce per thread chunk + merge + build_polyline"},
        "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1505_00914_b200.device import Context
    from paper_1505_00914_b200.shard import allreduce_dl

    rank, world, local = env_rank()
    # One process per GPU over NCCL.  CHP_DIST_BACKEND=gloo (with ranks
    # wrapped onto the visible devices) exists only to exercise the N > 1
    # control flow on a 1-GPU box; it is not a measurement configuration.
    backend = os.environ.get("CHP_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n_cfg, p, seed, desc = CONFIGS[args.config]
    n = args.n or n_cfg
    ctx = Context(local)
    stream = torch.cuda.Stream(dev)  # every kernel of the step and every event on one stream
    torch.cuda.set_stream(stream)

    # Workload: rank r owns points [r*n, (r+1)*n) of the config's stream.
    xy = ctx.generate(args.config, seed, p, n, offset=rank * n)
    DL = ctx.empty_dl(p)
    bufs: dict = {}
    torch.cuda.synchronize()

    k1_ev = []
    step_ev = []

    def step(mode: str = ""):
        # mode "step": an event at the step's start (per-step best/median);
        # mode "k1": events around K1 only (the roofline pass).  The headline
        # pass records nothing between K1 and K3, so K3's programmatic
        # dependent launch can overlap K1's tail as it does for a caller.
        if mode:
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
        ctx.reduce(xy, p, q=None if args.q_unset else p, out=DL, flags=args.flags)
        if mode == "k1":
            b = torch.cuda.Event(enable_timing=True)
            b.record(stream)
            k1_ev.append((a, b))
        elif mode == "step":
            step_ev.append(a)
        if world > 1:
            allreduce_dl(DL)  # the path's one exchange: element-wise MIN of the partial Ls
        return ctx.compact(DL, p, chain=True, bufs=bufs)

    for _ in range(max(args.warmup, 3)):
        comp = step()
    torch.cuda.synchronize()
    # parity guard on the benchmarked buffers (cheap, outside the timed region)
    counts = comp["counts"].cpu().tolist()
    if counts[2] != 0:
        raise SystemExit("validation error on the benchmark input")

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # The warm-up steps again, right before the timed region: the idle second
    # above lets the clocks settle low, and a first timed pass that ramps
    # them back measured ~4% slower per K1 than an identical second pass (C3).
    for _ in range(max(args.warmup, 3)):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    # Hold the stream for ~2 ms before the timed region so the host can queue
    # the steps ahead of the GPU (otherwise the first steps wait on Python's
    # launch rate, not on the device).  Outside the events.
    torch.cuda._sleep(4_000_000)
    start.record(stream)
    for _ in range(args.steps):
        comp = step("step")
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    elapsed_ms = start.elapsed_time(end)
    # Roofline pass: the same K steps again, K1 bracketed by events.
    torch.cuda._sleep(4_000_000)
    for _ in range(args.steps):
        step("k1")
    torch.cuda.synchronize()
    clk = clocks.stop()
    k1_ms = [a.elapsed_time(b) for a, b in k1_ev]
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    total_points = n * world
    value = total_points / (ms_per_step * 1e-3) / 1e9
    # Per-step times (best and median): step i runs from its K1
    # start event to the next step's (the last one to the end event).
    starts = step_ev
    step_ms = [starts[i].elapsed_time(starts[i + 1]) for i in range(len(starts) - 1)]
    step_ms.append(starts[-1].elapsed_time(end))

    # Roofline of the dominant kernel (K1 = every launch of chp_reduce).
    k1_avg = sum(k1_ms) / len(k1_ms)
    achieved = 8.0 * n / (k1_avg * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"k1_traffic_config{args.config}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # Hull (K4), outside the headline metric.
    comp_h = ctx.compact(DL, p, chain=False, lower=True, upper=True)
    ctx.hull(comp_h, p)
    torch.cuda.synchronize()
    hs = []
    for _ in range(3):
        # 10 back-to-back calls behind a short spin, so the host's launch
        # latency is queued ahead instead of timed.
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)
        a.record(stream)
        for _ in range(10):
            ctx.hull(comp_h, p)
        b.record(stream)
        torch.cuda.synchronize()
        hs.append(a.elapsed_time(b) / 10)
    hull_h = int(comp_h["_h"].item())

    # End to end through the C ABI from pinned host memory.
    e2e = None
    precondition_e2e = None
    if not args.no_e2e:
        import numpy as np

        host = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
        host.copy_(xy.cpu() if n * 8 <= 4 << 30 else xy.to("cpu"))
        chain_out = torch.empty((2 * p, 2), dtype=torch.int32, pin_memory=True)
        s_out = np.zeros(1, np.int64)
        ctx.pipeline_host_ptr(host.data_ptr(), n, p, p, chain_out.data_ptr(), s_out)  # warm-up
        ts = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.pipeline_host_ptr(host.data_ptr(), n, p, p, chain_out.data_ptr(), s_out)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        e2e_ms = statistics.median(ts)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = ctx.last_h2d_bytes
        e2e = {"value": total_points / (e2e_ms * 1e-3) / 1e9, "unit": "Gpoints/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(s_out[0]) * 8 + 64, "ms_per_step": e2e_ms,
               "path": "chp_pipeline_host (pinned int32 input; "
                       + (("8 Mi-point chunks packed to 16-bit slot|y words" if p <= 65536 else
                           "8 Mi-point chunks packed to 42-bit slot|y points, 3 per 16 bytes")
                          + " on host threads, int32 chunks DMA'd from the input's end while the host packs, "
                          if h2d < n * 8 else "16 Mi-point int32 chunks, ")
                       + "H2D overlapped with K1)"}
        # The reference's main entry, reducer::precondition (bounds unknown:
        # one pass computes them, then fold and compaction), through the same
        # pinned buffer: SURVEY 8(f) row 1, reported beside the headline.
        if world == 1:
            hn = host.numpy()
            ctx.precondition_host(hn, chain=True)  # warm-up
            pts = []
            for _ in range(args.e2e_steps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.precondition_host(hn, chain=True)
                b.record(stream)
                torch.cuda.synchronize()
                pts.append(a.elapsed_time(b))
            pre_ms = statistics.median(pts)
            precondition_e2e = {"value": n / (pre_ms * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": pre_ms,
                                "h2d_bytes_per_step": ctx.last_h2d_bytes,
                                "path": "chp_precondition_run + chp_last_outputs (pinned int32 input, bounds "
                                        "unknown: one pass, speculative 16-bit (or 42-bit) packing against a "
                                        "2^16 (2^21) window from a 64 Ki-point prefix, the bounds folded as the "
                                        "chunks land)"}
        del host

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(args.config, min(n, 100_000_000), p, seed, threads=1, reps=2)

    if rank == 0:
        line = {
            "metric": "Gpoints/s reduced+compacted", "value": value, "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "ms_per_step_best": min(step_ms), "ms_per_step_median": statistics.median(step_ms),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded counter-based generator, DESIGN.md Workloads)",
            "config": {"workload": desc, "n_per_rank": n, "p": p, "seed": seed,
                       "parallelism": f"dp{world} (point shards, MIN all-reduce of L)" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (%.1f GB > 126 MB); no flush" % (n * 8 / 1e9)
                             if n * 8 > 200e6 else "input L2-resident",
                       "k1_variant": ctx.variant, "s": int(counts[0]), "valid_slots": int(counts[1])},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": "K1 chp_reduce (all launches)", "k1_ms": k1_avg,
                         "algorithmic_bytes_per_launch": 8 * n, "peak_source": peak_src,
                         "frac_of_nominal_8TBs": achieved / 8000.0},
            "gpu_launches": launches,
            "clocks": clk,
            "hull_ms": min(hs), "hull_vertices": hull_h,
            "e2e": e2e,
            "precondition_e2e": precondition_e2e,
            "cpu_baseline": base,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
