"""A/B of the sweep's batch schedules on one B200: the dynamic batch counter vs
fixed row blocks (uot_set_deterministic), alternating runs on the same box,
K iterations each, device-timed (CUDA events around iterate).

python tools/sched_ab.py [--k 200] [--reps 3] [--only 3,4,5] [--json OUT]
"""
import json
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

SHAPES = {3: (32768, 32768), 4: (262144, 4096), 5: (131072, 32768), 2: (8192, 8192)}


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


k = int(arg("--k", 200))
reps = int(arg("--reps", 3))
only = [int(x) for x in arg("--only", "3,4,5").split(",")]
out = []
for c in only:
    m, n = SHAPES[c]
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        res = {"det": [], "dyn": []}
        for r in range(reps):
            for mode in ("dyn", "det"):
                s.set_deterministic(mode == "det")
                s.init_col_sums()
                s.iterate(3, 1e-300)
                it, err, conv, ms = s.iterate_timed(k, 1e-300)
                res[mode].append(ms * 1e3 / it)
                print(f"config {c} {m}x{n} {mode}: {ms * 1e3 / it:8.1f} us/iter", flush=True)
        d, y = min(res["det"]), min(res["dyn"])
        md, my = sorted(res["det"])[len(res["det"]) // 2], sorted(res["dyn"])[len(res["dyn"]) // 2]
        print(f"config {c}: best det {d:.1f} dyn {y:.1f} us/iter (det cost {100 * (d / y - 1):+.2f}%), "
              f"median det {md:.1f} dyn {my:.1f} ({100 * (md / my - 1):+.2f}%)", flush=True)
        out.append({"config": c, "rows": m, "cols": n, "k": k, "us_per_iter": res})
if "--json" in sys.argv:
    json.dump(out, open(arg("--json", ""), "w"), indent=1)
