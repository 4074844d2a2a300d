"""Device time of the sweep per shape for one library build (scratch tool).

UOT_LIB_PATH=paper_2412_11079_b200/libuot_cuda_pipe.so python tools/time_shapes.py 32768x32768x20 ...
"""
import os
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

import numpy as np  # noqa: E402

tag = os.path.basename(os.environ.get("UOT_LIB_PATH", "libuot_cuda.so"))
f64 = "--f64" in sys.argv  # Problem<double>: 16 bytes per element per iteration
esz = 8 if f64 else 4
for spec in [a for a in sys.argv[1:] if not a.startswith("--")]:
    m, n, k = (int(x) for x in spec.split("x"))
    with uot.Session(m, n, dtype=np.float64 if f64 else np.float32) as s:
        s.set_deterministic("--dynamic" not in sys.argv)
        s.generate_problem(42, 1.0, 0.1)
        s.init_col_sums()
        s.set_timing(True)
        s.iterate(3, 1e-300)
        s.iterate(k, 1e-300)
        sw, fin, n_ = s.timing()
        gbs = 2 * m * n * esz / (sw / n_ * 1e-3) / 1e9
        lay = s.layout
        print(f"[{tag}{' f64' if f64 else ''}] {m}x{n}: sweep {sw / n_ * 1e3:.1f} us ({gbs:.0f} GB/s) finalize {fin / n_ * 1e3:.1f} us "
              f"G={lay["G"]} res={lay["resident"]} dyn={lay["dynamic"]} smid={lay["smid_map"]} groups={lay["groups"]} B={lay['rows_per_step']} thr={lay['threads']} v={lay['chunks']}",
              flush=True)
