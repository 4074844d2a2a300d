"""Quick GPU sanity pass: parity on a few shapes vs the C oracle, then timing.

Scratch tool for development runs under gpurun; the real gates are tests/ and bench.py.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import Oracle  # noqa: E402
from paper_2412_11079_b200 import uot  # noqa: E402

o = Oracle()
ER, EP = 1.0, 0.1
shapes = [(2, 2, 3), (16, 16, 25), (10, 33, 25), (27, 6, 25), (1024, 1024, 100), (300, 20000, 10),
          (64, 32768, 10), (4096, 4096, 20), (2000, 513, 30)]
if len(sys.argv) > 1 and sys.argv[1] == "--quick":
    shapes = shapes[:5]
ok = True
for (m, n, k) in shapes:
    a, rpd, cpd = o.gen_problem(42, m, n)
    ref = o.fused_solve(a, rpd, cpd, ER, EP, 1e-300, k, workers=8)
    t = time.time()
    with uot.Session(m, n) as s:
        s.set_problem(uot.Problem(a, rpd, cpd, ER, EP))
        s.init_col_sums()
        it, err, conv = s.iterate(k, 1e-300)
        f = s.factors()
        plan = s.plan()
        cs = s.col_sums()
        lay = s.layout
    dt = time.time() - t
    rel = np.max(np.abs(plan.astype(np.float64) - ref.plan) / np.abs(ref.plan))
    bitw = np.mean(plan == ref.plan)
    ra = np.max(np.abs(f.alpha - ref.alpha) / np.abs(ref.alpha))
    rb = np.max(np.abs(f.beta - ref.beta) / np.abs(ref.beta))
    rc = np.max(np.abs(cs - ref.col_sums) / np.abs(ref.col_sums))
    good = it == k and rel <= 1e-5 and abs(err - ref.final_error) <= 1e-5 * max(1.0, ref.final_error)
    ok &= good
    print(f"{m}x{n} K={k}: it={it} plan maxrel={rel:.3e} bitwise={bitw:.6f} alpha={ra:.2e} beta={rb:.2e} "
          f"colsum={rc:.2e} err={err:.17g} ref_err={ref.final_error:.17g} G={lay['G']} groups={lay['groups']} "
          f"nt={lay['threads']} v={lay['chunks']} B={lay['rows_per_step']} ({dt:.2f}s) {'OK' if good else 'FAIL'}",
          flush=True)

for (m, n, k) in [(32768, 32768, 20), (262144, 4096, 20), (8192, 8192, 100), (1024, 1024, 200),
                  (131072, 32768, 5)]:
    with uot.Session(m, n) as s:
        s.generate_problem(42, ER, EP)
        s.init_col_sums()
        s.set_timing(True)
        s.iterate(3, 1e-300)
        t0 = time.time()
        s.iterate(k, 1e-300)
        wall = time.time() - t0
        sw, fin, n_ = s.timing()
        gbs = 2 * m * n * 4 / (sw / n_ * 1e-3) / 1e9
        print(f"{m}x{n}: sweep {sw / n_:.3f} ms/iter ({gbs:.0f} GB/s), finalize {fin / n_ * 1e3:.1f} us/iter, "
              f"wall {wall / k * 1e3:.3f} ms/iter, layout {s.layout}", flush=True)
print("ALL OK" if ok else "SOME FAILED")
