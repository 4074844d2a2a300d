"""Bytes per iteration on real HBM: fused (8 B/elem) vs the paper's two-pass GPU
schedule (16 B/elem, tiled.hpp:210-229) vs the reference's four-sweep baseline
(24 B/elem, baseline.hpp:100-110) — the metrics.cpp:60-77 traffic model.

python tools/ablation.py [--json OUT] [RxCxK ...]
"""
import json
import sys

sys.path.insert(0, ".")
from paper_2412_11079_b200 import uot  # noqa: E402

MODEL = {"fused": 8, "two_pass": 16, "baseline": 24}
args = [x for x in sys.argv[1:] if "x" in x and not x.startswith("--")]
out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
shapes = [tuple(int(v) for v in s.split("x")) for s in args] or [(32768, 32768, 20), (262144, 4096, 20), (8192, 8192, 100)]
rows = []
for m, n, k in shapes:
    for var in ("fused", "two_pass", "baseline"):
        with uot.Session(m, n) as s:
            s.set_resident(False)
            s.generate_problem(42, 1.0, 0.1)
            s.init_col_sums()
            s.set_variant(var)
            s.iterate(3, 1e-300)
            it, err, conv, ms = s.iterate_timed(k, 1e-300)
        us = ms * 1e3 / it
        model_gbs = MODEL[var] * m * n / (us * 1e-6) / 1e9
        rows.append({"shape": f"{m}x{n}", "variant": var, "us_per_iter": us, "bytes_per_elem_model": MODEL[var],
                     "model_gbs": model_gbs, "speedup_vs_variant": None})
        print(f"{m}x{n} {var:9s} {us:9.1f} us/iter  {MODEL[var]:2d} B/elem model -> {model_gbs:6.0f} GB/s", flush=True)
    base = {r["variant"]: r["us_per_iter"] for r in rows if r["shape"] == f"{m}x{n}"}
    print(f"   fused speedup: {base['two_pass'] / base['fused']:.2f}x over two-pass, "
          f"{base['baseline'] / base['fused']:.2f}x over baseline", flush=True)
if out:
    json.dump(rows, open(out, "w"), indent=1)
