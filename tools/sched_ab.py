"""A/B/C of the sweep's row-batch schedules on one B200, alternating runs on
the same box, K iterations each, device-timed (CUDA events around iterate):
uniform static blocks (default, balanced_blocks), weighted static blocks
(weights measured once by uot_calibrate_schedule) and the dynamic batch counter.

python tools/sched_ab.py [--k 200] [--reps 3] [--only 2,3,4,5] [--json OUT]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

SHAPES = {2: (8192, 8192), 3: (32768, 32768), 4: (262144, 4096), 5: (131072, 32768)}
MODES = ("weighted", "uniform", "dynamic")


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


k = int(arg("--k", 200))
reps = int(arg("--reps", 3))
only = [int(x) for x in arg("--only", "2,3,4,5").split(",")]
out = {"configs": []}
for c in only:
    m, n = SHAPES[c]
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        res = {mode: [] for mode in MODES}
        s.init_col_sums()
        w = s.calibrate_schedule(4)
        print(f"config {c}: calibrated weights min {w.min()} max {w.max()} (ratio {w.max() / w.min():.2f}) "
              f"over {w.size} groups", flush=True)
        for r in range(reps):
            for mode in MODES:
                s.set_schedule(mode)
                s.init_col_sums()
                s.iterate(3, 1e-300)
                it, err, conv, t = s.iterate_timed(k, 1e-300)
                res[mode].append(t * 1e3 / it)
                print(f"config {c} {m}x{n} {mode:15s}: {t * 1e3 / it:8.1f} us/iter", flush=True)
        med = {mode: sorted(v)[len(v) // 2] for mode, v in res.items()}
        print(f"config {c}: median us/iter " + ", ".join(f"{mode} {med[mode]:.1f}" for mode in MODES)
              + f"  (weighted vs dynamic {100 * (med['weighted'] / med['dynamic'] - 1):+.2f}%, "
                f"uniform vs dynamic {100 * (med['uniform'] / med['dynamic'] - 1):+.2f}%)", flush=True)
        out["configs"].append({"config": c, "rows": m, "cols": n, "k": k, "us_per_iter": res,
                               "weights": w.tolist()})
if "--json" in sys.argv:
    json.dump(out, open(arg("--json", ""), "w"), indent=1)
