"""Sustained power / clock / throughput of the sweep against plain streaming.

Each case runs ~SECS seconds of back-to-back work while nvidia-smi samples
power and SM clock every 100 ms; the report is the median over the second half
(steady state). Cases: torch in-place scale (pure RMW streaming, the power floor
of moving the bytes), the fused sweep f32 / f64 on equal bytes.

python tools/power_study.py [SECS]
"""
import statistics
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

SECS = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
CASES = sys.argv[2].split(",") if len(sys.argv) > 2 else ["torch_rmw", "f32_32768", "f64_32768x16384", "f32_262144x4096"]


class Smi:
    def __enter__(self):
        self.p = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks.mem,temperature.gpu,clocks_event_reasons.active",
             "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        return self

    def __exit__(self, *a):
        self.p.terminate()
        out = self.p.communicate()[0]
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") == 4]
        rows = [r for r in rows if float(r[1]) > 1000]  # under load
        half = rows[len(rows) // 2:]
        self.power = statistics.median(float(r[0]) for r in half) if half else float("nan")
        self.sm = statistics.median(float(r[1]) for r in half) if half else float("nan")
        self.temp = max((float(r[3]) for r in half), default=float("nan"))
        self.reasons = sorted({r[4].strip() for r in half})


def cool():
    torch.cuda.synchronize()
    time.sleep(4.0)


def run_case(name):
    if name.startswith("torch_rmw"):
        # torch_rmw: constant data; torch_rmw_rand: uniform random bits (HBM power is data dependent)
        a = torch.rand(1 << 30, device="cuda") if name.endswith("rand") else torch.ones(1 << 30, device="cuda")
        for _ in range(3):
            a.mul_(1.0000001)
        torch.cuda.synchronize()
        per = []
        with Smi() as smi:
            t_end = time.time() + SECS
            while time.time() < t_end:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    a.mul_(1.0000001)
                e1.record()
                e1.synchronize()
                per.append(e0.elapsed_time(e1) / 20)
        nbytes = 2 * a.numel() * 4
        del a
    else:
        dt, shape = name.split("_")
        m, n = (int(x) for x in (shape.split("x") * 2)[:2])
        with uot.Session(m, n, dtype={"f32": "float32", "f64": "float64"}[dt]) as s:
            s.generate_problem(42, 1.0, 0.1)
            s.init_col_sums()
            s.iterate(3, 1e-300)
            per = []
            with Smi() as smi:
                t_end = time.time() + SECS
                while time.time() < t_end:
                    _, _, _, ms = s.iterate_timed(50, 1e-300)
                    per.append(ms / 50)
            nbytes = 2 * m * n * (8 if dt == "f64" else 4)
    first = per[0]
    steady = statistics.median(per[len(per) // 2:])
    print(f"{name:18s} first {nbytes / first / 1e6:6.0f} GB/s  steady {nbytes / steady / 1e6:6.0f} GB/s  "
          f"power {smi.power:6.1f} W  sm {smi.sm:6.0f} MHz  Tmax {smi.temp:.0f}  reasons {smi.reasons}", flush=True)


for c in CASES:
    cool()
    run_case(c)
