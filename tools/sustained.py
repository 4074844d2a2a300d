"""Sustained-load behaviour: device time per block of iterations over a long
run, with nvidia-smi power / clocks / temperatures sampled alongside.

python tools/sustained.py ROWS COLS BLOCKS ITERS_PER_BLOCK
"""
import subprocess
import sys
import time

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

m, n, blocks, per = (int(x) for x in sys.argv[1:5])
q = ("timestamp,power.draw,clocks.sm,clocks.mem,temperature.gpu,temperature.memory,"
     "clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown")
smi = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader", "-lms", "100"],
                       stdout=open("gpurun_out/sustained_smi.csv", "w"), stderr=subprocess.DEVNULL)
time.sleep(0.5)
with uot.Session(m, n) as s:
    s.generate_problem(42, 1.0, 0.1)
    s.init_col_sums()
    s.iterate(3, 1e-300)
    for b in range(blocks):
        it, err, conv, ms = s.iterate_timed(per, 1e-300)
        print(f"block {b:3d}: {ms / per * 1e3:8.1f} us/iter  {2 * m * n * 4 / (ms / per * 1e-3) / 1e9:6.0f} GB/s  t={time.time():.2f}",
              flush=True)
time.sleep(0.3)
smi.terminate()
