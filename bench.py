#!/usr/bin/env python
"""bench.py — fused Sinkhorn-UOT iterations on B200 (MAP-UOT, arxiv 2412.11079).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one fused UOT iteration (fused_iterate_parallel, reference
include/uot/fused.hpp:197-250): one sm_100a sweep over the resident matrix plus
the O(cols) finalize (and, for N > 1, one NCCL allreduce of the column sums).

Workload (BASELINE.json metric): 32768 x 32768 fp32 per GPU, gen_problem_t seed
42, reg=0.1 reg_m=1.0 (fi = 1/1.1). N GPUs weak-scale: the global problem is
(32768*N) x 32768 row-sharded by RankPartition (N=4 is BASELINE config 5,
131072 x 32768). `value` counts 32768^2-equivalent iterations per second over
the whole job, so value(N) = N * value(1) is perfect scaling.

Under torchrun each rank drives its LOCAL_RANK GPU; torch.distributed (gloo)
carries only barriers, the NCCL id and the max-over-ranks of the timings.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "UOT iterations/s and HBM GB/s (% of ~8 TB/s) at 32768² fp32, 1/2/4/8 B200"
UNIT = "iterations/s (32768x32768 fp32-equivalent)"
ROWS_PER_GPU = 32768
COLS = 32768
SEED = 42
ER, EP = 1.0, 0.1  # reg_m = 1.0, reg = 0.1  ->  fi = 1/1.1
KNEVER = 1e-300    # positive but unreachable: fixed-length runs (acceptance.cpp:26)


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


# --------------------------------------------------------------- plumbing --

class Group:
    """rank / world / barrier / max-reduce over the torchrun job (gloo), or a no-op."""

    def __init__(self):
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        self.local_rank = env_int("LOCAL_RANK", self.rank)
        self.dist = None
        if self.world > 1:
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

    def close(self):
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join(HERE, "gpurun_out", f".clocks_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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
                "power_w_max": max(power) if power else None, "reasons": sorted(reasons)}


def peak_hbm():
    """MEASURED_PEAKS.json (driver-written) or the profiling guide's fallback."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per sweep launch from the
    committed ncu --set full summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(HERE, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------- CPU arms --

def cpu_reference(steps: int, warmup: int, sample_rows: int, kind_pref: str = "reference"):
    """Time the reference's fused_iterate_parallel (oracle/_ref: the unmodified
    reference compiled from its sources; else the C restatement) with every host
    thread on a row sample of the workload. Returns per-iteration ms list."""
    import oracle  # test/benchmark infrastructure only: the CPU baseline leg
    threads = os.cpu_count() or 1
    kind = "port"
    eng = None
    if kind_pref == "reference":
        try:
            eng = oracle.RefOracle()
            kind = "reference"
        except (OSError, FileNotFoundError):
            eng = None
    if eng is None:
        eng = oracle.Oracle()
    o = oracle.Oracle()
    a, rpd, cpd = o.gen_problem(SEED, sample_rows, COLS, threads=threads)
    if kind == "reference":
        ms = eng.time_fused_iterate(a, rpd, cpd, ER, EP, threads, warmup + steps)
    else:
        cs = o.init_col_sums(a, threads)
        fi = o.compute_fi(ER, EP)
        ms = []
        for _ in range(warmup + steps):
            t0 = time.perf_counter()
            o.fused_iterate(a, cs, rpd, cpd, fi, threads)
            ms.append((time.perf_counter() - t0) * 1e3)
    ms = list(ms[warmup:]) or list(ms)
    mean_ms = sum(ms) / len(ms)
    scale = (sample_rows * COLS) / (ROWS_PER_GPU * COLS)
    value = scale * 1e3 / mean_ms
    return {
        "value": value, "unit": UNIT, "cores": threads, "kind": kind,
        "sample": (f"rows 0..{sample_rows - 1} of gen_problem_t<float>(42, {sample_rows}, {COLS}); "
                   f"fused_iterate_parallel W={threads}, {len(ms)} timed iterations after {warmup} warm-up "
                   f"(mean {mean_ms:.1f} ms/iter, model {2 * sample_rows * COLS * 4 / mean_ms / 1e6:.1f} GB/s), "
                   f"scaled by rows to {ROWS_PER_GPU}x{COLS}"),
        "ms_per_iter": mean_ms,
    }


def run_reference_arm(args, grp: Group):
    if grp.rank != 0:
        return None
    sample_rows = args.cpu_sample_rows
    cb = cpu_reference(args.steps, args.warmup, sample_rows, "reference")
    return {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["ms_per_iter"] / ((sample_rows * COLS) / (ROWS_PER_GPU * COLS)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_problem_t SplitMix64 seed 42), host memory",
        "config": {"workload": f"{ROWS_PER_GPU}x{COLS} fp32 per GPU, fi=1/1.1 (reg=0.1, reg_m=1.0)",
                   "rows": ROWS_PER_GPU, "cols": COLS, "parallelism": "cpu threads",
                   "sample_rows": sample_rows},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------- our arm --

def run_ours(args, grp: Group):
    from paper_2412_11079_b200 import distributed as D
    from paper_2412_11079_b200 import uot

    world, rank = grp.world, grp.rank
    rows_global = ROWS_PER_GPU * world
    units = (rows_global * COLS) / (ROWS_PER_GPU * COLS)  # 32768^2-equivalents per iteration
    dev = int(os.environ.get("BENCH_DEVICE", grp.local_rank))  # BENCH_DEVICE: ranks sharing one GPU (smoke only)

    s = D.make_session(rows_global, COLS, dev, args.exchange)  # collective (peer handles / NCCL id)
    exchange = s.exchange  # "nccl" when the peer mappings could not be made (make_session falls back)
    lay = s.layout
    rows_local = s.rows

    # ---- device-resident throughput (the `value`) -------------------------
    s.generate_problem(SEED, ER, EP)  # gen_problem_t bits, generated in HBM
    s.init_col_sums()
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
    hbm_gbs = world * bytes_iter_local * args.steps / (max_ms / 1e3) / 1e9

    peak, peak_src = peak_hbm()
    sweep_avg_ms = sweep_ms / max(nsweeps, 1)
    achieved = bytes_iter_local / (sweep_avg_ms / 1e3) / 1e9
    traffic = ncu_traffic(f"{rows_local}x{COLS}")

    # ---- end to end through the public API with host buffers ---------------
    e2e = None
    if not args.no_e2e:
        pin = uot.PinnedBuffer((rows_local, COLS), np.float32)
        p = uot.gen_block(SEED, rows_global, COLS, s.row_offset, rows_local, out=pin.array)
        p.er, p.ep = ER, EP
        out = uot.PinnedBuffer((rows_local, COLS), np.float32)
        grp.barrier()
        t0 = time.perf_counter()
        res = D.distributed_solve(p, KNEVER, args.steps, session=s, global_rows=rows_global) \
            if world > 1 else None
        if world == 1:
            s.set_problem(p)              # H2D of A, rpd, cpd + validation (problem.hpp:64-103)
            s.init_col_sums()
            it2, _, _ = s.iterate(args.steps, KNEVER)
            f = s.factors()                # D2H alpha, beta
            s.plan(out=out.array)          # D2H plan
        else:
            it2 = res.report.iterations
            out.array[...] = res.plan
        wall = time.perf_counter() - t0
        wall = grp.max(wall)
        h2d = rows_local * COLS * 4 + rows_local * 8 + COLS * 8
        d2h = rows_local * COLS * 4 + rows_local * 8 + COLS * 8
        e2e = {"value": units * it2 / wall, "unit": UNIT,
               "h2d_bytes_per_step": h2d * world / args.steps, "d2h_bytes_per_step": d2h * world / args.steps,
               "what": (f"fused_solve through the C ABI from page-locked host buffers: upload + validate "
                        f"{rows_local}x{COLS} per rank, init_col_sums, {args.steps} iterations, download "
                        f"plan + factors; wall {wall * 1e3:.1f} ms (max over ranks); per-step bytes = run bytes / steps")}
        pin.free()
        out.free()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(args.cpu_steps, 1, args.cpu_sample_rows, "reference")
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    s.close()

    if rank != 0:
        return None
    xdesc = (", column sums exchanged once per iteration inside the finalize kernels over peer memory "
             "(CUDA IPC, NVLink): cols+1 f64 pushed to every rank, ascending-rank sum") \
        if exchange == "peer" else ", NCCL allreduce of cols+N f64 per iteration"
    return {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: gen_problem_t<float> SplitMix64 seed 42 bits, generated in HBM (value) / on the host (e2e)",
        "config": {
            "workload": f"{ROWS_PER_GPU}x{COLS} fp32 per GPU (global {rows_global}x{COLS}), reg=0.1 reg_m=1.0 "
                        f"(fi=1/1.1), {args.steps} fused iterations",
            "rows_global": rows_global, "cols": COLS, "rows_per_gpu": rows_local, "storage": "f32",
            "arithmetic": "f64 products rounded once to f32, f64 sums (bit-compatible with the reference)",
            "parallelism": f"row-sharded x{world}" + (xdesc if world > 1 else ""),
            "l2": f"no flush: the resident matrix ({bytes_iter_local / 2 / 2**30:.1f} GiB/GPU) exceeds the 126 MB L2",
            "layout": {k: lay[k] for k in ("G", "groups", "slice", "threads", "nbuf", "rows_per_step", "smem_bytes")},
        },
        "hbm_gbs": hbm_gbs,
        # the metric's own yardstick (report both): nominal 8 TB/s per GPU, and the measured copy peak
        "hbm_frac_of_8tbs": hbm_gbs / (8000.0 * world),
        "hbm_frac_of_measured_copy": hbm_gbs / (peak * world),
        "final_error": err,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "uotk::sweep_kernel (fused row pass)",
                     "bytes_per_launch": bytes_iter_local, "avg_launch_ms": sweep_avg_ms,
                     "finalize_avg_us": fin_ms / max(nsweeps, 1) * 1e3},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clk,
    }


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
    ap.add_argument("--cpu-sample-rows", type=int, default=8192)
    ap.add_argument("--cpu-steps", type=int, default=10)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    grp = Group()
    if grp.world != args.gpus and grp.world > 1:
        sys.stderr.write(f"note: --gpus {args.gpus} but WORLD_SIZE={grp.world}; using the launcher's world\n")
    args.gpus = grp.world if grp.world > 1 else args.gpus
    if args.gpus > 1 and grp.world == 1:
        ap.error("N > 1 runs under torchrun (one process per GPU)")
    if args.impl == "reference":
        line = run_reference_arm(args, grp)
    else:
        line = run_ours(args, grp)
    grp.close()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
