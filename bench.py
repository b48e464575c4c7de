#!/usr/bin/env python
"""Benchmark of the hot path: Algorithm 1 reduction + skip-invalid compaction
(BASELINE.json metric: Gpoints/s reduced+compacted, % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload: BASELINE.json config 5 by default -- n = 4e9 int32 points, p = 256,
"sharded over 1/2/4/8 GPUs": the n points are split into contiguous equal
slices over the N ranks (strong scaling; rank r owns
shard_bounds(n, r, N)).  configs[1] (config 2) is where `north_star`'s
roofline target is quoted; configs 2-4 run through the same code in the same
invocation and are reported under `per_config` (same split, same timing).

A step = one pass of the path over the batch: K1 (chp_reduce: DL init +
Algorithm 1) on each rank's slice resident in HBM, then (N > 1) the path's
one exchange -- an element-wise MIN reduce of the partial device-form L onto
rank 0 over NCCL -- then K3 (chp_compact: Lemma-1 chain + counts).  `value` = n /
(max over ranks of the device-timed K steps / K).  The hull (K4) is timed
separately (`hull_ms`), outside `value`, as BASELINE.json prescribes.

`e2e` is the same metric through the public C-ABI call a user makes, from
pinned HOST memory, host<->device copies inside the timed region: at N = 1
chp_pipeline_host (chunked H2D overlapped with K1, K3, chain back); at N > 1
each rank chp_reduce_host on its slice, the NCCL MIN reduce onto rank 0, then
rank 0 chp_finish_host (K3, chain back).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libchpref.so: chp::reducer::reduce + build_polyline compiled
from the reference's sources) on this host's cores over a bounded sample of
the same workload (rank 0 only); that process loads only oracle/ libraries.
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
    5: (4_000_000_000, 256, 5, "config5: n=4e9 sharded over the GPUs, 90% in 4 hot columns, p=256"),
}
DEFAULT_CONFIG = 5
REF_SAMPLE = 100_000_000  # points per reference-arm step / cpu_baseline sample


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--total-points", type=int, default=0,
                    help="override the config's total n (tests, smoke runs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--flags", type=int, default=0, help="chp_reduce flags (variant forcing, experiments)")
    ap.add_argument("--q-unset", action="store_true",
                    help="K1 without the y bound q (the reference API's default; not the headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-config", action="store_true", help="measure only --config")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--verify", action="store_true",
                    help="rank 0 checks the final chain against the oracle (chunked, host threads; untimed)")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard_bounds(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal slices (paper_1505_00914_b200.shard.shard_bounds,
    restated so the reference arm need not import the product package)."""
    lo = n_total * rank // world
    return lo, n_total * (rank + 1) // world - lo


def config_dict(cfg: int, n_total: int, world: int) -> dict:
    """The `config` object -- identical in both arms."""
    _, p, seed, desc = CONFIGS[cfg]
    return {"workload": desc, "n_total": n_total, "p": p, "q": p, "seed": seed,
            "sharding": f"n split into {world} contiguous equal slices, one per GPU (strong scaling)",
            "l2": "inputs larger than L2 (%.1f GB > 126 MB); no flush" % (n_total * 8 / world / 1e9)
                  if n_total * 8 / world > 200e6 else "input L2-resident"}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(cfg: int):
    """DRAM bytes per K1 call from the committed ncu capture (profiles/), or
    None.  Not measured in this run (bench never runs under a profiler)."""
    prof = os.path.join(ROOT, "profiles", f"k1_traffic_config{cfg}.json")
    if not os.path.exists(prof):
        return None, None
    with open(prof) as f:
        d = json.load(f)
    return d.get("dram_bytes_per_launch"), f"profiles/k1_traffic_config{cfg}.json ({d.get('round', 'r01')}, " \
                                           f"ncu dram__bytes_read+write of one K1 call at N=1; not this run)"


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


def cpu_time_sample(cfg: int, n_sample: int, threads: int, reps: int):
    """The reference itself (oracle/_ref) on the host over the first
    n_sample points of the config, or the C restatement when the reference
    library is absent.  Baseline / checker use only; loads oracle/ libraries
    only (oracle.generate = the generator compiled for the host)."""
    import oracle

    _, p, seed, _ = CONFIGS[cfg]
    xy = oracle.generate(cfg, seed, p, n_sample)
    if oracle.Reference.available():
        ref = oracle.Reference()
        kind = "reference"

        def once():
            return ref.time_reduce_compact(xy, p, p, threads=threads, reps=1)[0]
    else:
        orc = oracle.Oracle()
        kind, threads = "port", 1

        def once():
            t0 = time.perf_counter()
            orc.build_polyline(orc.reduce(xy, p, p))
            return time.perf_counter() - t0
    return once, kind, threads


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg: int, n_sample: int, reps: int = 2):
    once, kind, threads = cpu_time_sample(cfg, n_sample, threads=1, reps=reps)
    t = min(once() for _ in range(reps))
    return {"value": n_sample / t / 1e9, "unit": "Gpoints/s", "cores": threads, "kind": kind,
            "sample": f"first {n_sample:.3g} points of config {cfg} (same bytes as the GPU input), "
                      f"chp::reducer::reduce + build_polyline, best of {reps}, {threads} thread; "
                      f"host {os.cpu_count()} cpus", "seconds": t, "host_cpu": cpu_model(), "nproc": os.cpu_count()}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    n_total = args.total_points or CONFIGS[args.config][0]
    n_sample = min(n_total, REF_SAMPLE)
    threads = os.cpu_count() or 1
    step, kind, threads = cpu_time_sample(args.config, n_sample, threads=threads, reps=1)
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    tot = sum(times)
    value = n_sample * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": "Gpoints/s reduced+compacted", "value": value, "unit": "Gpoints/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded counter-based generator, DESIGN.md Workloads)",
        "config": config_dict(args.config, n_total, world),
        "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": threads, "kind": kind,
                         "sample": f"per step the first {n_sample:.3g} of the config's {n_total:.3g} points "
                                   f"(bounded CPU sample), chp::reducer::reduce per thread chunk + element-wise "
                                   f"merge + build_polyline, {threads} host threads",
                         "host_cpu": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Arm:
    """Our arm: one rank (one GPU) of the run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.args = torch, dist, args
        self.rank, self.world, local = env_rank()
        # One process per GPU over NCCL.  CHP_DIST_BACKEND=gloo (with ranks
        # wrapped onto the visible devices) exists only to exercise the N > 1
        # control flow on a 1-GPU box; it is not a measurement configuration.
        self.backend = os.environ.get("CHP_DIST_BACKEND", "nccl")
        if self.world > 1 and "CHP_HOST_THREADS" not in os.environ:
            # the host packing pools of the ranks on this node share its cores
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", self.world))
            os.environ["CHP_HOST_THREADS"] = str(max(2, (os.cpu_count() or 2) // local_world))
        self.local = local % max(torch.cuda.device_count(), 1)
        if self.world > 1:
            torch.cuda.set_device(self.local)
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
        self.dev = torch.device("cuda", self.local)
        torch.cuda.set_device(self.dev)
        from paper_1505_00914_b200.device import Context

        self.ctx = Context(self.local)
        self.stream = torch.cuda.Stream(self.dev)  # every kernel of the step and every event on one stream
        torch.cuda.set_stream(self.stream)
        self.host = None  # pinned host buffer, sized for the largest slice (reused by every config)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def combine(self, DL):
        if self.world > 1:
            from paper_1505_00914_b200.shard import reduce_dl

            # the path's one exchange: element-wise MIN of the partial Ls onto
            # rank 0, whose K3 produces the chain (the other ranks compact
            # their partial L, which nobody reads)
            reduce_dl(DL, dst=0)

    def measure(self, cfg: int, n_total: int, e2e: bool) -> dict:
        torch, ctx, args, stream = self.torch, self.ctx, self.args, self.stream
        _, p, seed, _ = CONFIGS[cfg]
        q = None if args.q_unset else p
        start_pt, n = shard_bounds(n_total, self.rank, self.world)
        xy = ctx.generate(cfg, seed, p, n, offset=start_pt)
        DL = ctx.empty_dl(p)
        bufs: dict = {}
        torch.cuda.synchronize()
        k1_ev, step_ev = [], []

        def step(mode: str = ""):
            # mode "step": an event at the step's start (per-step best/median);
            # mode "k1": events around K1 only (the roofline pass).  The headline
            # pass records nothing between K1 and K3, so K3's programmatic
            # dependent launch can overlap K1's tail as it does for a caller.
            if mode:
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            ctx.reduce(xy, p, q=q, out=DL, flags=args.flags)
            if mode == "k1":
                b = torch.cuda.Event(enable_timing=True)
                b.record(stream)
                k1_ev.append((a, b))
            elif mode == "step":
                step_ev.append(a)
            self.combine(DL)
            return ctx.compact(DL, p, chain=True, bufs=bufs)

        warm = max(args.warmup, 3)
        for _ in range(warm):
            comp = step()
        torch.cuda.synchronize()
        counts = comp["counts"].cpu().tolist()  # guard on the benchmarked buffers, outside the timed region
        if counts[2] != 0:
            raise SystemExit("validation error on the benchmark input")
        clocks = ClockSampler(self.local)
        clocks.start()
        time.sleep(0.3)
        # The warm-up steps again, right before the timed region: the idle
        # second above lets the clocks settle low, and a first timed pass that
        # ramps them back measured ~4% slower per K1 than a second pass (C3).
        for _ in range(warm):
            step()
        self.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launches
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        # Hold the stream ~2 ms so the host queues the steps ahead of the GPU
        # (otherwise the first steps wait on Python's launch rate).  Outside
        # the events.
        torch.cuda._sleep(4_000_000)
        start.record(stream)
        for _ in range(args.steps):
            comp = step("step")
        end.record(stream)
        torch.cuda.synchronize()
        self.barrier()
        launches = ctx.launches - launches0
        elapsed_ms = self.max_over_ranks(start.elapsed_time(end))
        torch.cuda._sleep(4_000_000)  # roofline pass: the same K steps, K1 bracketed by events
        for _ in range(args.steps):
            step("k1")
        torch.cuda.synchronize()
        clk = clocks.stop()
        k1_ms = [a.elapsed_time(b) for a, b in k1_ev]
        ms_per_step = elapsed_ms / args.steps
        step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(len(step_ev) - 1)]
        step_ms.append(step_ev[-1].elapsed_time(end))
        k1_avg = sum(k1_ms) / len(k1_ms)
        achieved = 8.0 * n / (k1_avg * 1e-3) / 1e9
        peak, peak_src = measured_peak()
        traffic, traffic_src = committed_traffic(cfg) if self.world == 1 and not args.total_points else (None, None)
        out = {
            "value": n_total / (ms_per_step * 1e-3) / 1e9, "ms_per_step": ms_per_step,
            "ms_per_step_best": min(step_ms), "ms_per_step_median": statistics.median(step_ms),
            "k1_variant": ctx.variant, "s": int(counts[0]), "valid_slots": int(counts[1]),
            "n_per_rank": n, "gpu_launches": launches, "clocks": clk,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "K1 chp_reduce (all launches of one call)", "k1_ms": k1_avg,
                         "algorithmic_bytes_per_launch": 8 * n, "algorithmic_bytes_per_point": 8,
                         "peak_source": peak_src, "frac_of_nominal_8TBs": achieved / 8000.0},
        }
        # Hull (K4), outside the headline metric; on the merged L.
        comp_h = ctx.compact(DL, p, chain=False, lower=True, upper=True)
        ctx.hull(comp_h, p)
        torch.cuda.synchronize()
        hs = []
        for _ in range(3):
            # 10 back-to-back calls behind a short spin (launch latency queued, not timed)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(1_000_000)
            a.record(stream)
            for _ in range(10):
                ctx.hull(comp_h, p)
            b.record(stream)
            torch.cuda.synchronize()
            hs.append(a.elapsed_time(b) / 10)
        out["hull_ms"], out["hull_vertices"] = min(hs), int(comp_h["_h"].item())
        if args.verify:
            out["verified"] = self.verify(cfg, n_total, comp)
        if e2e:
            out["e2e"] = self.e2e(cfg, n_total, xy, p, q)
        del xy
        torch.cuda.empty_cache()
        return out

    def verify(self, cfg, n_total, comp):
        """Rank 0: the final (merged) chain against the chunked oracle over
        all n_total points (generated on the host).  Checker only."""
        ok = True
        if self.rank == 0:
            import numpy as np

            import oracle

            _, p, seed, _ = CONFIGS[cfg]
            orc = oracle.Oracle()
            acc = orc.accumulator(p, p)
            chunk = 1 << 26
            for a in range(0, n_total, chunk):
                acc.add(oracle.generate(cfg, seed, p, min(chunk, n_total - a), offset=a))
            chain = orc.build_polyline(acc.finish())
            s = int(comp["counts"][0].item())
            ok = s == len(chain) and bool(np.array_equal(comp["chain"][:s].cpu().numpy(), chain))
        self.barrier()
        return ok

    def e2e(self, cfg, n_total, xy, p, q):
        import numpy as np

        torch, ctx, stream = self.torch, self.ctx, self.stream
        n = xy.shape[0]
        if self.host is None or self.host.shape[0] < n:
            self.host = None
            self.host = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
        host = self.host[:n]
        host.copy_(xy)
        chain_out = torch.empty((2 * p, 2), dtype=torch.int32, pin_memory=True)
        s_out = np.zeros(1, np.int64)
        DL = ctx.empty_dl(p)

        def call():
            if self.world == 1:
                ctx.pipeline_host_ptr(host.data_ptr(), n, p, q, chain_out.data_ptr(), s_out)
                return ctx.last_h2d_bytes
            ctx.reduce_host_ptr(host.data_ptr(), n, p, q, DL)
            h2d = ctx.last_h2d_bytes
            self.combine(DL)
            if self.rank == 0:
                ctx.finish_host_ptr(DL, p, chain_out.data_ptr(), s_out)
            return h2d

        call()  # warm-up
        ts = []
        for _ in range(self.args.e2e_steps):
            self.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h2d = call()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        e2e_ms = self.max_over_ranks(statistics.median(ts))
        h2d = int(self.sum_over_ranks(float(h2d)))
        packed = h2d < n_total * 8
        path = ("chp_pipeline_host" if self.world == 1 else
                "per rank chp_reduce_host on its slice, NCCL MIN reduce of L onto rank 0, rank 0 chp_finish_host") + \
               " (pinned int32 input; " + \
               (("8 Mi-point chunks packed to 2-byte slot|y points (8 bits each)" if p <= 256 else
                 "8 Mi-point chunks packed to 16-bit slot|y words" if p <= 65536 else
                 "8 Mi-point chunks packed to 42-bit slot|y points, 3 per 16 bytes")
                + " on host threads, int32 chunks DMA'd from the input's end while the host packs, "
                if packed else "16 Mi-point int32 chunks, ") + "H2D overlapped with K1)"
        return {"value": n_total / (e2e_ms * 1e-3) / 1e9, "unit": "Gpoints/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": int(s_out[0]) * 8 + 64, "ms_per_step": e2e_ms, "path": path}

    def precondition_e2e(self, cfg, n_total):
        """The reference's main entry, reducer::precondition (bounds unknown:
        one pass computes them, then fold and compaction), from the same
        pinned buffer: SURVEY 8(f) row 1, reported beside the headline."""
        torch = self.torch
        hn = self.host[:n_total].numpy()
        self.ctx.precondition_host(hn, chain=True)  # warm-up
        pts = []
        for _ in range(self.args.e2e_steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            self.ctx.precondition_host(hn, chain=True)
            b.record(self.stream)
            torch.cuda.synchronize()
            pts.append(a.elapsed_time(b))
        pre_ms = statistics.median(pts)
        return {"value": n_total / (pre_ms * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": pre_ms,
                "h2d_bytes_per_step": self.ctx.last_h2d_bytes,
                "path": "chp_precondition_run + chp_last_outputs (pinned int32 input, bounds unknown: one pass, "
                        "speculative 2-byte, 4-byte or 42-bit packing against a 2^8, 2^16 or 2^21 window from a "
                        "64 Ki-point prefix, the bounds folded as the chunks land)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    arm = Arm(args)
    n_total = args.total_points or CONFIGS[args.config][0]
    head = arm.measure(args.config, n_total, e2e=not args.no_e2e)
    pre = None
    if arm.world == 1 and not args.no_e2e:
        pre = arm.precondition_e2e(args.config, n_total)
    per_config = {}
    if not args.no_per_config and args.config == DEFAULT_CONFIG and not args.total_points:
        for c in sorted(CONFIGS):
            if c == args.config:
                continue
            r = arm.measure(c, CONFIGS[c][0], e2e=not args.no_e2e)
            per_config[f"config{c}"] = {
                "workload": CONFIGS[c][3], "n_total": CONFIGS[c][0], "value": r["value"], "unit": "Gpoints/s",
                "ms_per_step": r["ms_per_step"], "k1_variant": r["k1_variant"], "s": r["s"],
                "roofline_frac": r["roofline"]["frac"], "roofline_achieved_gbs": r["roofline"]["achieved"],
                "k1_ms": r["roofline"]["k1_ms"], "traffic": r["roofline"]["traffic"],
                "e2e": r.get("e2e") and {k: r["e2e"][k] for k in ("value", "unit", "h2d_bytes_per_step",
                                                                   "d2h_bytes_per_step", "ms_per_step")},
                "hull_ms": r["hull_ms"], "hull_vertices": r["hull_vertices"], "clocks": r["clocks"]}
    base = None
    if arm.rank == 0 and arm.world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(args.config, min(n_total, REF_SAMPLE))
    if arm.rank == 0:
        line = {
            "metric": "Gpoints/s reduced+compacted", "value": head["value"], "unit": "Gpoints/s",
            "n_gpus": arm.world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": head["ms_per_step"], "ms_per_step_best": head["ms_per_step_best"],
            "ms_per_step_median": head["ms_per_step_median"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded counter-based generator, DESIGN.md Workloads)",
            "config": config_dict(args.config, n_total, arm.world),
            "k1_variant": head["k1_variant"], "result": {"s": head["s"], "valid_slots": head["valid_slots"],
                                                         "n_per_rank": head["n_per_rank"]},
            "roofline": head["roofline"], "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "hull_ms": head["hull_ms"], "hull_vertices": head["hull_vertices"],
            "e2e": head.get("e2e"), "precondition_e2e": pre, "cpu_baseline": base,
            "per_config": per_config or None,
        }
        if args.verify:
            line["verified"] = head["verified"]
        print(json.dumps(line), flush=True)
    if arm.world > 1:
        arm.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
