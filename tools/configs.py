"""Every BASELINE.json config on one B200 through the public Session API:
device-timed iterations/s and model HBM GB/s (2*R*C*4 bytes per iteration,
metrics.cpp:69-72) next to the measured copy peak (MEASURED_PEAKS.json).

python tools/configs.py [--json OUT] [--only 2,4] [--schedule uniform|weighted|dynamic]

--schedule: the row-batch schedule (default: the session default, uniform
static blocks; weighted calibrates its weights once, untimed).
"""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

CONFIGS = [  # BASELINE.json configs (config 5 on one GPU; its N-GPU form is bench.py --gpus N)
    ("1: 1024^2, K=100", 1024, 1024, 100),
    ("2: 8192^2, K=500", 8192, 8192, 500),
    ("3: 32768^2, K=200", 32768, 32768, 200),
    ("4: 262144x4096, K=200", 262144, 4096, 200),
    ("5: 131072x32768 (1 GPU), K=200", 131072, 32768, 200),
]
try:
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    peak = 6650.0
only = None  # --only 2,4: a subset of the configs
if "--only" in sys.argv:
    only = {int(x) for x in sys.argv[sys.argv.index("--only") + 1].split(",")}
rows = []
for idx, (name, m, n, k) in enumerate(CONFIGS, 1):
    if only and idx not in only:
        continue
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        s.init_col_sums()
        sched = sys.argv[sys.argv.index("--schedule") + 1] if "--schedule" in sys.argv else None
        if sched == "weighted" and not s.layout["pinned"]:
            sched = "uniform"
        if sched == "weighted":
            s.calibrate_schedule(4)
        if sched:
            s.set_schedule(sched)
        s.iterate(3, 1e-300)  # warm-up
        it, err, conv, ms = s.iterate_timed(k, 1e-300)
        lay = s.layout
    gbs = 2 * m * n * 4 * it / (ms * 1e-3) / 1e9
    mode = "resident" if lay["resident"] else f"streaming G={lay['G']} {sched or 'default'}"
    rows.append({"config": name, "iterations": it, "ms_total": ms, "us_per_iter": ms * 1e3 / it,
                 "it_per_s": it / (ms * 1e-3), "model_gbs": gbs, "frac_of_copy_peak": gbs / peak, "mode": mode})
    print(f"{name:34s} {ms * 1e3 / it:9.1f} us/iter {it / (ms * 1e-3):10.1f} it/s {gbs:7.0f} GB/s "
          f"({gbs / peak:.2f} of {peak:.0f})  [{mode}]", flush=True)
if "--json" in sys.argv:
    json.dump({"peak_gbs": peak, "rows": rows}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
