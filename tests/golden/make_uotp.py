"""Golden .uotp containers written by the UNMODIFIED reference (oracle/_ref:
uot::write_problem, problem_io.cpp:97-104). Run here, where /root/reference
exists; the files are committed and the tests only read them.

python tests/golden/make_uotp.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

ref = oracle.RefOracle()
cases = [("io_6x4_er2.5_ep0.5.uotp", 5, 6, 4, 2.5, 0.5),
         ("io_64x100.uotp", 11, 64, 100, 1.0, 0.1),
         ("io_37x1000.uotp", 3, 37, 1000, 1.0, 0.25)]
for name, seed, m, n, er, ep in cases:
    a, rpd, cpd = ref.gen_problem(seed, m, n)
    ref.write_problem(os.path.join(HERE, name), a, rpd, cpd, er, ep)
# a Problem<double> container (the product's kernels are f32-only: it must be rejected cleanly)
a, rpd, cpd = ref.gen_problem(5, 2, 2)
ref.write_problem(os.path.join(HERE, "io_2x2_f64.uotp"), a.astype(np.float64), rpd, cpd, 1.0, 0.25)
for f in sorted(os.listdir(HERE)):
    if f.endswith(".uotp"):
        print(f, os.path.getsize(os.path.join(HERE, f)))
