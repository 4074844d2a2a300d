"""Small solves through every device path, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck). Results are checked against the
oracle so a sanitizer-perturbed run that computes garbage also fails.

compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2412_11079_b200 import uot  # noqa: E402

o = oracle.Oracle()
KN = 1e-300


def check(name, plan, ref):
    rel = float(np.max(np.abs(plan.astype(np.float64) - ref) / ref))
    print(f"{name:40s} max rel err {rel:.2e}", flush=True)
    if rel > 1e-5:
        raise SystemExit(f"{name}: parity failed")


# streaming G=1 (34 rows per CTA: not resident), G=3, G=4 with TMEM column
# factors, resident, tiny
# streaming G=1 with wide slices (split sweep roles) and a problem past the 64 MiB
# L2-keep threshold (alternating sweep directions)
cases = [(5100, 1000, 3), (24, 20000, 3), (40, 32768, 3), (96, 1000, 5), (7, 9, 3), (400, 8192, 3),
         (2100, 8192, 3), (5000, 4096, 3)]
if "--only" in sys.argv:  # e.g. --only 2100x8192,5000x4096 (racecheck of single paths)
    want = {tuple(int(x) for x in c.split("x")) for c in sys.argv[sys.argv.index("--only") + 1].split(",")}
    cases = [c for c in cases if (c[0], c[1]) in want]
for m, n, k in cases:
    a, rpd, cpd = o.gen_problem(42, m, n)
    ref = o.fused_solve(a, rpd, cpd, 1.0, 0.1, KN, k, workers=2)
    res = uot.fused_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KN, k)
    with uot.Session(m, n) as s:
        lay = s.layout
    check(f"fused {m}x{n} G={lay['G']} resident={lay['resident']} v={lay['chunks']}", res.plan, ref.plan)
if "--only" in sys.argv:
    print("sanitize cases OK")
    raise SystemExit(0)
a, rpd, cpd = o.gen_problem(3, 50, 2500, dtype=np.float64)
ref = o.fused_solve(a, rpd, cpd, 1.0, 0.1, KN, 3, 2)
check("f64 50x2500", uot.fused_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KN, 3).plan, ref.plan)
for (m, n) in [(60, 1500), (64, 16384)]:  # group ranks at G=1 and G=2 (smid-addressed CTAs)
    a, rpd, cpd = o.gen_problem(5, m, n)
    ref = o.distributed_solve(a, rpd, cpd, 1.0, 0.1, KN, 3, 2)
    check(f"2-rank group {m}x{n}",
          uot.distributed_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KN, 3, 2, devices=[0, 0]).plan, ref.plan)
print("sanitize cases OK")
