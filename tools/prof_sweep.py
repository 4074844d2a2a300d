"""Drive a few sweep launches of one configuration (for ncu / nvidia-smi runs).

python tools/prof_sweep.py ROWS COLS [ITERS] [--uniform]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 3
with uot.Session(m, n) as s:
    s.generate_problem(42, 1.0, 0.1)
    s.init_col_sums()
    if s.layout["pinned"] and "--uniform" not in sys.argv:
        s.calibrate_schedule(4)  # the bench's schedule: 4 scratch sweeps, then weighted row blocks
    s.set_timing(True)
    t0 = time.time()
    s.iterate(k, 1e-300)
    sw, fin, cnt = s.timing()
    print(f"{m}x{n}: {k} iterations, sweep {sw / cnt:.3f} ms, finalize {fin / cnt * 1e3:.1f} us, "
          f"{2 * m * n * 4 / (sw / cnt * 1e-3) / 1e9:.0f} GB/s, wall {time.time() - t0:.3f} s, layout {s.layout}")
