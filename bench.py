#!/usr/bin/env python
"""bench.py — fused Sinkhorn-UOT iterations on B200 (MAP-UOT, arxiv 2412.11079).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one fused UOT iteration (fused_iterate_parallel, reference
include/uot/fused.hpp:197-250): one sm_100a sweep over the resident matrix plus
the O(cols) finalize (for N > 1 with the per-iteration exchange of the column
sums, distributed.hpp:88-100, fused into the finalize over peer memory).

Workloads (BASELINE.json configs, gen_problem_t seed 42, reg=0.1 reg_m=1.0,
fi = 1/1.1):
  N = 1   config 3, 32768 x 32768 fp32 (the headline);
  N > 1   config 5, 131072 x 32768 fp32 row-sharded by RankPartition
          (plan.cpp:35-44) over the N GPUs — strong scaling; rank 0 also times
          the same 131072 x 32768 problem on ONE GPU first, so the line carries
          parallel_efficiency = T1 / (N * T_N) measured in the same run.
`value` counts 32768^2-equivalent iterations per second over the whole job (a
config-5 iteration is 4 of them), so value(N) / (N * value(1)) is the scaling
efficiency the driver computes.

`python bench.py --gpus N` re-launches itself under torch.distributed.run (one
process per GPU); under torchrun each rank drives its LOCAL_RANK GPU and
torch.distributed (gloo) carries only barriers, the peer-memory handles and the
max-over-ranks of the device timings.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "UOT iterations/s and HBM GB/s (% of ~8 TB/s) at 32768² fp32, 1/2/4/8 B200"
UNIT = "iterations/s (32768x32768 fp32-equivalent)"
COLS = 32768
HEADLINE_ROWS = 32768      # config 3 (N = 1)
SHARDED_ROWS = 131072      # config 5 (N > 1)
UNIT_ELEMS = 32768 * 32768
SEED = 42
ER, EP = 1.0, 0.1  # reg_m = 1.0, reg = 0.1  ->  fi = 1/1.1
KNEVER = 1e-300    # positive but unreachable: fixed-length runs (acceptance.cpp:26)


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def workload(world: int, rows_override: int = 0):
    if rows_override:  # CPU tests only: a small stand-in, never a bench value
        return rows_override, f"{rows_override}x32768 fp32 (--rows override: NOT a BASELINE config)"
    rows = HEADLINE_ROWS if world == 1 else SHARDED_ROWS
    name = ("config 3: 32768x32768 fp32" if world == 1 else
            f"config 5: 131072x32768 fp32 row-sharded over {world} GPUs (RankPartition, plan.cpp:35-44)")
    return rows, name


# --------------------------------------------------------------- plumbing --

class Group:
    """rank / world / barrier / max-reduce over the torchrun job (gloo), or a no-op."""

    def __init__(self, init: bool = True):
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        self.local_rank = env_int("LOCAL_RANK", self.rank)
        self.dist = None
        if self.world > 1 and init:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, obj):
        if not self.dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks, power and throttle reasons sampled during a timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_ms: int = 100):
        self.gpu = gpu
        self.period_ms = period_ms
        self.proc = None
        self.path = os.path.join(HERE, "gpurun_out", f".clocks_{os.getpid()}_{gpu}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (OSError, ValueError):
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    smax.append(float(p[2]))
                    power.append(float(p[3]))
                except ValueError:
                    continue
                for n, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "power_w_max": max(power) if power else None,
                "power_w_median": statistics.median(power) if power else None, "reasons": sorted(reasons)}


def peak_hbm():
    """MEASURED_PEAKS.json (driver-written) or the profiling guide's fallback."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per sweep launch from the
    committed ncu --set full capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(HERE, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except (OSError, ValueError):
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------- CPU legs --

def cpu_reference(rows: int, steps: int, warmup: int, w1_iters: int = 2):
    """The reference's fused_iterate_parallel (oracle/_ref: the unmodified
    reference compiled from its sources; else the C restatement) on the FULL
    rows x COLS workload with every host thread (W = nproc), `warmup` untimed
    then `steps` timed iterations; plus W = 1 on `w1_iters` iterations.
    Generation and init_col_sums are excluded."""
    import oracle  # test/benchmark infrastructure only: the CPU baseline leg
    threads = os.cpu_count() or 1
    o = oracle.Oracle()
    try:
        eng, kind = oracle.RefOracle(), "reference"
    except (OSError, FileNotFoundError):
        eng, kind = None, "port"
    a, rpd, cpd = o.gen_problem(SEED, rows, COLS, threads=threads)

    def timed(workers, k):
        if eng is not None:
            return list(eng.time_fused_iterate(a, rpd, cpd, ER, EP, workers, k))
        cs = o.init_col_sums(a, workers)
        fi = o.compute_fi(ER, EP)
        out = []
        for _ in range(k):
            t0 = time.perf_counter()
            o.fused_iterate(a, cs, rpd, cpd, fi, workers)
            out.append((time.perf_counter() - t0) * 1e3)
        return out

    ms = timed(threads, warmup + steps)[warmup:]
    mean_ms = sum(ms) / len(ms)
    units = rows * COLS / UNIT_ELEMS
    w1 = None
    if w1_iters > 0:
        ms1 = timed(1, w1_iters)
        m1 = sum(ms1) / len(ms1)
        w1 = {"workers": 1, "iterations": len(ms1), "ms_per_iter": m1, "value": units * 1e3 / m1,
              "model_gbs": 2 * rows * COLS * 4 / m1 / 1e6}
    return {
        "value": units * 1e3 / mean_ms, "unit": UNIT, "cores": threads, "kind": kind,
        "sample": (f"full {rows}x{COLS} gen_problem_t<float>(42) workload; fused_iterate_parallel W={threads} "
                   f"(all host threads), {len(ms)} timed iterations after {warmup} warm-up: mean {mean_ms:.1f} ms/iter, "
                   f"model {2 * rows * COLS * 4 / mean_ms / 1e6:.1f} GB/s"),
        "ms_per_iter": mean_ms, "iterations": len(ms), "warmup": warmup,
        "cpu_model": cpu_model(), "w1": w1, "same_config": True,
    }


def run_reference_arm(args, world: int):
    rows, name = workload(world, args.rows)
    cb = cpu_reference(rows, args.steps, args.warmup, w1_iters=args.cpu_w1_iters if world == 1 else 1)
    units = rows * COLS / UNIT_ELEMS
    return {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": cb["iterations"], "warmup": cb["warmup"],
        "ms_per_step": cb["ms_per_iter"] / units,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_problem_t SplitMix64 seed 42), host memory",
        "config": {"workload": f"{name}, reg=0.1 reg_m=1.0 (fi=1/1.1)", "rows": rows, "cols": COLS,
                   "parallelism": f"cpu threads (W={cb['cores']}, {cb['cpu_model']})", "same_config": True},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "w1")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------- our arm --

def single_gpu_t1(rows: int, steps: int, warmup: int, dev: int) -> float:
    """Device ms of `steps` iterations of the whole rows x COLS problem on ONE GPU
    (the T1 of the strong-scaling efficiency)."""
    from paper_2412_11079_b200 import uot
    with uot.Session(rows, COLS, dev) as s:
        s.generate_problem(SEED, ER, EP)
        s.init_col_sums()
        s.iterate(warmup, KNEVER)
        it, _, _, ms = s.iterate_timed(steps, KNEVER)
    if it != steps:
        raise RuntimeError(f"T1 run: {it} of {steps} iterations")
    return ms


def run_ours(args, grp: Group):
    from paper_2412_11079_b200 import distributed as D
    from paper_2412_11079_b200 import uot

    world, rank = grp.world, grp.rank
    rows_global, wname = workload(world, args.rows)
    units = rows_global * COLS / UNIT_ELEMS  # 32768^2-equivalents per iteration
    dev = int(os.environ.get("BENCH_DEVICE", grp.local_rank))  # BENCH_DEVICE: ranks sharing one GPU (smoke only)

    t1_ms = None
    if world > 1 and not args.no_t1:
        if rank == 0:
            t1_ms = single_gpu_t1(rows_global, args.steps, args.warmup, dev)
        grp.barrier()

    s = D.make_session(rows_global, COLS, dev, args.exchange)  # collective (peer handles / NCCL id)
    exchange = s.exchange if world > 1 else "none"
    lay = s.layout
    rows_local = s.rows

    # ---- device-resident throughput (the `value`) -------------------------
    s.generate_problem(SEED, ER, EP)  # gen_problem_t bits, generated in HBM
    s.init_col_sums()
    # The deterministic weighted schedule (uot_set_schedule): row blocks sized
    # by per-row-group weights measured once (uot_calibrate_schedule: 4
    # dynamic iterations on a scratch copy of the plan, untimed); every solve
    # with these weights is bit-reproducible. Falls back to the uniform blocks
    # where the sweep does not run one CTA on every SM.
    weights = None
    schedule = args.schedule
    if schedule == "weighted":
        if s.layout["pinned"]:
            weights = s.calibrate_schedule(4)
        else:
            schedule = "uniform"
    s.set_schedule(schedule)
    lay = s.layout
    s.iterate(args.warmup, KNEVER)
    s.set_timing(True)
    launches0 = s.kernel_launches()
    grp.barrier()
    s.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    it, err, conv, dev_ms = s.iterate_timed(args.steps, KNEVER)
    s.synchronize()
    clk = clocks.stop()
    grp.barrier()
    gpu_launches = s.kernel_launches() - launches0
    sweep_ms, fin_ms, nsweeps = s.timing()
    s.set_timing(False)
    if it != args.steps:
        raise RuntimeError(f"ran {it} of {args.steps} iterations")
    max_ms = grp.max(dev_ms)
    value = units * args.steps / (max_ms / 1e3)
    bytes_iter_local = 2.0 * rows_local * COLS * 4  # metrics.cpp:69-72 model, this GPU
    hbm_gbs = 2.0 * rows_global * COLS * 4 * args.steps / (max_ms / 1e3) / 1e9
    sweep_avg_ms = sweep_ms / max(nsweeps, 1)
    fin_avg_us = fin_ms / max(nsweeps, 1) * 1e3
    per_rank = grp.gather({"rank": rank, "rows": rows_local, "device_ms": dev_ms, "sweep_us": sweep_avg_ms * 1e3,
                           "exchange_finalize_us": fin_avg_us})

    peak, peak_src = peak_hbm()
    achieved = bytes_iter_local / (sweep_avg_ms / 1e3) / 1e9

    # ---- the other row-batch schedules, same steps (transparency) -----------
    schedules = {schedule: value}
    if not args.no_schedule_ab:
        for other in ("uniform", "weighted", "dynamic"):
            if other in schedules or (other == "weighted" and weights is None):
                continue
            s.set_schedule(other)
            s.iterate(args.warmup, KNEVER)
            grp.barrier()
            _, _, _, ms_o = s.iterate_timed(args.steps, KNEVER)
            schedules[other] = units * args.steps / (grp.max(ms_o) / 1e3)
        s.set_schedule(schedule)

    # ---- sustained: >= args.sustained_s of back-to-back iterations ---------
    sustained = None
    if args.sustained_s > 0:
        ksus = max(args.steps, int(math.ceil(args.sustained_s / (max_ms / args.steps / 1e3))))
        grp.barrier()
        s.synchronize()
        cs = ClockSampler(dev, 200)
        cs.start()
        it_s, _, _, ms_s = s.iterate_timed(ksus, KNEVER)
        s.synchronize()
        clk_s = cs.stop()
        ms_s = grp.max(ms_s)
        sustained = {"iterations": it_s, "seconds": ms_s / 1e3, "value": units * it_s / (ms_s / 1e3),
                     "hbm_gbs": 2.0 * rows_global * COLS * 4 * it_s / (ms_s / 1e3) / 1e9,
                     "frac_of_8tbs": 2.0 * rows_global * COLS * 4 * it_s / (ms_s / 1e3) / 1e9 / (8000.0 * world),
                     "clocks": clk_s}

    # ---- end to end through the public API with host buffers ---------------
    e2e = None
    if not args.no_e2e:
        pin = uot.PinnedBuffer((rows_local, COLS), np.float32)
        p = uot.gen_block(SEED, rows_global, COLS, s.row_offset, rows_local, out=pin.array)
        p.er, p.ep = ER, EP
        out = uot.PinnedBuffer((rows_local, COLS), np.float32)
        grp.barrier()
        t0 = time.perf_counter()
        phases = {}
        if world > 1:
            res = D.distributed_solve(p, KNEVER, args.steps, session=s, global_rows=rows_global)
            it2 = res.report.iterations
            out.array[...] = res.plan
        else:
            s.set_problem(p)              # H2D of A, rpd, cpd + validation (problem.hpp:64-103)
            t1 = time.perf_counter()
            s.init_col_sums()
            it2, _, _ = s.iterate(args.steps, KNEVER)
            t2 = time.perf_counter()
            s.factors()                    # D2H alpha, beta
            s.plan(out=out.array)          # D2H plan
            t3 = time.perf_counter()
            phases = {"upload_validate_ms": (t1 - t0) * 1e3, "seed_iterate_ms": (t2 - t1) * 1e3,
                      "download_ms": (t3 - t2) * 1e3,
                      "h2d_gbs": (rows_local * COLS * 4) / (t1 - t0) / 1e9,
                      "d2h_gbs": (rows_local * COLS * 4) / (t3 - t2) / 1e9}
        wall = grp.max(time.perf_counter() - t0)
        h2d = rows_local * COLS * 4 + rows_local * 8 + COLS * 8
        d2h = rows_local * COLS * 4 + rows_local * 8 + COLS * 8
        e2e = {"value": units * it2 / wall, "unit": UNIT,
               "h2d_bytes_per_step": h2d * world / args.steps, "d2h_bytes_per_step": d2h * world / args.steps,
               "wall_ms": wall * 1e3, **phases,
               "what": (f"fused_solve through the C ABI from page-locked host buffers: upload + validate "
                        f"{rows_local}x{COLS} per rank, init_col_sums, {args.steps} iterations, download "
                        f"plan + factors; wall {wall * 1e3:.1f} ms (max over ranks); per-step bytes = run bytes / steps")}
        pin.free()
        out.free()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(rows_global, args.cpu_steps or args.steps, args.warmup, w1_iters=args.cpu_w1_iters)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "w1", "same_config")}
    s.close()

    if rank != 0:
        return None
    xdesc = {"peer": ", column sums exchanged once per iteration inside the finalize kernels over peer memory "
                     "(NVLink): cols+1 f64 pushed to every rank, ascending-rank sum",
             "nccl": ", one NCCL allreduce of cols+N f64 per iteration", "none": ""}[exchange]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: gen_problem_t<float> SplitMix64 seed 42 bits, generated in HBM (value) / on the host (e2e)",
        "config": {
            "workload": f"{wname}, reg=0.1 reg_m=1.0 (fi=1/1.1), {args.steps} fused iterations",
            "rows_global": rows_global, "cols": COLS, "rows_per_gpu": rows_local, "storage": "f32",
            "arithmetic": "f64 products rounded once to f32, f64 sums (bit-compatible with the reference)",
            "parallelism": f"row-sharded x{world}" + xdesc,
            "schedule": {"weighted": "weighted static row blocks (weights calibrated once, untimed; "
                                     "deterministic: bit-reproducible for the given weights)",
                         "uniform": "uniform static row blocks, balanced_blocks (the default; bit-reproducible)",
                         "dynamic": "dynamic row batches (device counter; ~1e-12 run-to-run differences)"}[schedule],
            "l2": f"no flush: the resident matrix ({bytes_iter_local / 2 / 2**30:.1f} GiB/GPU) exceeds the 126 MB L2",
            "layout": {k: lay[k] for k in ("G", "groups", "slice", "threads", "nbuf", "rows_per_step", "smem_bytes",
                                           "dynamic", "schedule", "pinned")},
        },
        "schedules_value": schedules,
        "hbm_gbs": hbm_gbs,
        # the metric's own yardstick (report both): nominal 8 TB/s per GPU, and the measured copy peak
        "hbm_frac_of_8tbs": hbm_gbs / (8000.0 * world),
        "hbm_frac_of_measured_copy": hbm_gbs / (peak * world),
        "final_error": err,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(f"{rows_local}x{COLS}"),
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + "
                                       "dram__bytes_write.sum of one sweep launch of this shape)",
                     "peak_source": peak_src,
                     "kernel": "uotk::sweep_kernel (fused row pass)",
                     "bytes_per_launch": bytes_iter_local, "avg_launch_ms": sweep_avg_ms,
                     "finalize_avg_us": fin_avg_us},
        "sustained": sustained,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clk,
    }
    if world > 1:
        sw = [r["sweep_us"] for r in per_rank]
        line["per_rank"] = per_rank
        line["rank_skew_us"] = max(sw) - min(sw)
        line["exchange_finalize_us_max"] = max(r["exchange_finalize_us"] for r in per_rank)
        if t1_ms is not None:
            line["t1_ms_per_step"] = t1_ms / args.steps
            line["parallel_efficiency"] = t1_ms / (world * max_ms)
    return line


# ------------------------------------------------------------- launcher --

def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: one process per GPU via
    torch.distributed.run on this node (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default=os.environ.get("UOT_EXCHANGE", "peer"),
                    help="N>1: fused peer-memory exchange (default) or one NCCL allreduce per iteration")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-t1", action="store_true", help="N>1: skip the single-GPU T1 run (no parallel_efficiency)")
    ap.add_argument("--cpu-steps", type=int, default=0, help="cpu_baseline timed iterations (default: --steps)")
    ap.add_argument("--cpu-w1-iters", type=int, default=2, help="cpu_baseline W=1 iterations (0: skip)")
    ap.add_argument("--rows", type=int, default=0, help=argparse.SUPPRESS)  # tests: small stand-in workload
    ap.add_argument("--schedule", choices=["weighted", "uniform", "dynamic"], default="weighted",
                    help="row-batch schedule of the timed region (default: weighted, deterministic)")
    ap.add_argument("--no-schedule-ab", action="store_true", help="skip timing the other two schedules")
    ap.add_argument("--sustained-s", type=float, default=2.0,
                    help="seconds of back-to-back iterations for the `sustained` block (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    world = env_int("WORLD_SIZE", 1)
    if launched and world > 1 and world != args.gpus:
        sys.stderr.write(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using the launcher's world\n")
    if args.impl == "reference":
        # the reference's CPU path on rank 0 only; other ranks exit without work
        world = world if launched else args.gpus
        if env_int("RANK", 0) != 0:
            return 0
        print(json.dumps(run_reference_arm(args, world)), flush=True)
        return 0
    if not launched and args.gpus > 1:
        return relaunch_under_torchrun(args.gpus)
    grp = Group()
    line = run_ours(args, grp)
    grp.close()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
