"""Weighted-schedule calibration length vs the dynamic schedule (scratch probe).

python tools/calib_probe.py ROWSxCOLSxK [...]
"""
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

for spec in sys.argv[1:]:
    m, n, k = (int(x) for x in spec.split("x"))
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        s.init_col_sums()
        s.iterate(3, 1e-300)
        res = {}
        for label in ("dyn", "cal4", "cal12", "cal32", "dyn2", "cal4b"):
            if label.startswith("dyn"):
                s.set_schedule("dynamic")
            else:
                s.calibrate_schedule(int(label[3:].rstrip("b")))
            s.iterate(3, 1e-300)
            it, _, _, ms = s.iterate_timed(k, 1e-300)
            res[label] = ms / it * 1e3
        print(spec, " ".join(f"{l} {v:7.1f}" for l, v in res.items()), flush=True)
