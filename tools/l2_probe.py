"""Does an earlier static sweep leave L2 state that speeds up the dynamic schedule? (scratch probe)"""
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1].split("x"))


def timed(s, sched, kk=k):
    s.set_schedule(sched)
    s.iterate(2, 1e-300)
    it, _, _, ms = s.iterate_timed(kk, 1e-300)
    return ms / it * 1e3


for case in ("dyn_fresh", "uni3_then_dyn", "dyn_uni_dyn"):
    with uot.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.1)
        s.init_col_sums()
        out = []
        if case == "dyn_fresh":
            out.append(timed(s, "dynamic"))
            out.append(timed(s, "dynamic"))
        elif case == "uni3_then_dyn":
            s.iterate(3, 1e-300)
            out.append(timed(s, "dynamic"))
            out.append(timed(s, "dynamic"))
        else:
            out.append(timed(s, "dynamic"))
            out.append(timed(s, "uniform"))
            out.append(timed(s, "dynamic"))
            out.append(timed(s, "uniform", 1))
            out.append(timed(s, "dynamic"))
        print(sys.argv[1], case, " ".join(f"{v:.1f}" for v in out), flush=True)
