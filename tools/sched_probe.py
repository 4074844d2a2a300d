"""Schedules interleaved in one session (scratch probe): uniform / weighted / dynamic.

python tools/sched_probe.py ROWSxCOLSxK [REPS]
"""
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1].split("x"))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
with uot.Session(m, n) as s:
    s.generate_problem(42, 1.0, 0.1)
    s.init_col_sums()
    s.iterate(3, 1e-300)
    w = s.calibrate_schedule(4)
    out = {"uniform": [], "weighted": [], "dynamic": []}
    for r in range(reps):
        for sc in out:
            if sc == "weighted":
                s.set_group_weights(w)
            s.set_schedule(sc)
            s.iterate(3, 1e-300)
            it, _, _, ms = s.iterate_timed(k, 1e-300)
            out[sc].append(ms / it * 1e3)
    print(sys.argv[1], " ".join(f"{sc} " + "/".join(f"{v:.1f}" for v in vals) for sc, vals in out.items()),
          "keep", s.layout.get("keep_batches"), flush=True)
