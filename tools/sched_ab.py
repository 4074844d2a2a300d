"""A/B/C of the sweep's row-batch schedules on one B200, alternating runs on
the same box, K iterations each, device-timed (CUDA events around iterate):
class-weighted static blocks (default), uniform static blocks
(balanced_blocks) and the dynamic batch counter. Also prints the SM speed
classes (topology.cuh) and how many batches each class took under the dynamic
schedule — the fused sweep's own per-class rate.

python tools/sched_ab.py [--k 200] [--reps 3] [--only 2,3,4,5] [--json OUT]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

SHAPES = {2: (8192, 8192), 3: (32768, 32768), 4: (262144, 4096), 5: (131072, 32768)}
MODES = ("class_weighted", "uniform", "dynamic")


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


k = int(arg("--k", 200))
reps = int(arg("--reps", 3))
only = [int(x) for x in arg("--only", "2,3,4,5").split(",")]
cls, ms = uot.sm_classes(0)
ncls = int(cls.max()) + 1 if cls.size and cls.min() >= 0 else 0
print(f"SM speed classes: {ncls}; sizes {[int((cls == c).sum()) for c in range(ncls)]}; "
      f"probe ms {[round(float(np.median(ms[cls == c])), 3) for c in range(ncls)]}", flush=True)
out = {"classes": cls.tolist(), "probe_ms": ms.tolist(), "configs": []}
for c in only:
    m, n = SHAPES[c]
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        res = {mode: [] for mode in MODES}
        per_class = None
        for r in range(reps):
            for mode in MODES:
                s.set_schedule(mode)
                s.init_col_sums()
                s.iterate(3, 1e-300)
                it, err, conv, t = s.iterate_timed(k, 1e-300)
                res[mode].append(t * 1e3 / it)
                if mode == "dynamic" and ncls:
                    smid, nb, w = s.schedule_stats()
                    per_class = [float(nb[cls[smid] == q].mean()) if (cls[smid] == q).any() else 0.0
                                 for q in range(ncls)]
                print(f"config {c} {m}x{n} {mode:15s}: {t * 1e3 / it:8.1f} us/iter", flush=True)
        lay = s.layout
        _, _, w = s.schedule_stats()
        med = {mode: sorted(v)[len(v) // 2] for mode, v in res.items()}
        print(f"config {c}: median us/iter " + ", ".join(f"{mode} {med[mode]:.1f}" for mode in MODES)
              + f"  (class-weighted vs dynamic {100 * (med['class_weighted'] / med['dynamic'] - 1):+.2f}%, "
                f"uniform vs dynamic {100 * (med['uniform'] / med['dynamic'] - 1):+.2f}%)", flush=True)
        if per_class:
            slow = per_class[-1] or 1.0
            print(f"config {c}: dynamic batches per CTA by class {[round(x, 1) for x in per_class]} "
                  f"-> rate vs slowest {[round(x / slow, 3) for x in per_class]}; group weights used "
                  f"{sorted(set(int(x) for x in w))} /32; layout G={lay['G']} groups={lay['groups']} "
                  f"classes={lay['sm_classes']}", flush=True)
        out["configs"].append({"config": c, "rows": m, "cols": n, "k": k, "us_per_iter": res,
                               "dynamic_batches_per_class": per_class})
if "--json" in sys.argv:
    json.dump(out, open(arg("--json", ""), "w"), indent=1)
