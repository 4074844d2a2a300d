"""Phase timers of the sweep kernel (trace build): where do the cycles go?

python tools/trace_sweep.py ROWS COLS [ITERS]   (uses paper_2412_11079_b200/libuot_cuda_trace.so)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("UOT_LIB_PATH", os.path.abspath("paper_2412_11079_b200/libuot_cuda_trace.so"))
from paper_2412_11079_b200 import uot  # noqa: E402

NAMES = {0: "factor0 wait done1", 2: "factor0 exchange poll", 3: "factor0 pow+arrive", 9: "factor0 TOTAL",
         4: "producer wait done2", 8: "producer TOTAL",
         16: "warp0 wait full", 19: "warp0 wait alpha", 21: "warp0 TOTAL",
         24: "resident: beta load", 25: "resident: sweep 1", 26: "resident: factors (pow)",
         27: "resident: sweep 2 + partials", 28: "resident: barrier 1", 29: "resident: column reduction",
         30: "resident: barrier 2"}
L = uot.lib()
L.uot_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 32)()
for spec in sys.argv[1:]:
    m, n, k = (int(x) for x in spec.split("x"))
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        s.init_col_sums()
        s.iterate(2, 1e-300)
        L.uot_trace_read(buf, 1)
        s.set_timing(True)
        s.iterate(k, 1e-300)
        L.uot_trace_read(buf, 1)
        sw, fin, cnt = s.timing()
        lay = s.layout
        grid = lay["groups"] * lay["G"]
        nb = (m / lay["groups"]) / lay["rows_per_step"]
        nbf = {0: 2, 2: 2, 3: 2, 9: 1}  # factor warp 0 handles every NF-th batch (NF = 2 for these shapes)
        print(f"== {m}x{n} x{k}: sweep {sw / cnt:.3f} ms ({2 * m * n * 4 / (sw / cnt * 1e-3) / 1e9:.0f} GB/s) "
              f"G={lay['G']} groups={lay['groups']} B={lay['rows_per_step']} nbuf={lay['nbuf']} batches/CTA={nb:.0f}")
        for i, name in NAMES.items():
            if i >= 24:  # one CTA's per-iteration phase times
                if lay.get("resident"):
                    print(f"   {name:28s} {buf[i] / k / 1965:8.2f} us/iter")
                continue
            v = buf[i] / (grid * k)
            per = v / nb * (nbf.get(i, 1) if i != 9 else 1)
            print(f"   {name:28s} {v / 1e3:10.1f} kcyc/CTA/iter  {v / nb:8.0f} cyc/batch (all batches)")
