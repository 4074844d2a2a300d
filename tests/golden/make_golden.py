"""Generate tests/golden/ from the UNMODIFIED reference (oracle/_ref/libuot_ref.so,
compiled from /root/reference/proj/core by oracle/Makefile).

    python tests/golden/make_golden.py [--big]

small.npz : full outputs (plan, alpha, beta, col_sums, final_error) of the
            reference's fused_solve / fused_iterate_parallel on small problems,
            including the hand-checked known-answer cases of proj/tests.
big.npz   : anchors at the BASELINE.json sizes (sum/max of P, sampled rows and
            factors, final_error, sha256 of the plan) — the size-independent
            comparison points for the full-size GPU parity tests.

The inputs are never stored: gen_problem_t (problem_io.hpp:17-31) regenerates
them bit-exactly (pinned by tests/test_oracle.py::test_generator_*).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

KNEVER = 1e-300

# (seed, rows, cols, fi, iterations, workers)
SMALL = [
    (42, 1, 1, 1 / 1.1, 10, 1),
    (42, 1, 100, 1 / 1.1, 10, 1),
    (42, 100, 1, 1 / 1.1, 10, 1),
    (7, 7, 3, 0.5, 30, 1),
    (21, 16, 16, 0.5, 25, 1),      # test_fused.cpp:82
    (22, 10, 33, 1.0, 25, 1),      # test_fused.cpp:83 (shape)
    (24, 27, 6, 0.75, 25, 1),      # test_fused.cpp:85 (shape)
    (33, 128, 128, 0.5, 100, 4),   # test_fused.cpp:145-152 (shape)
    (123, 37, 21, 0.5, 20, 3),     # acceptance.cpp:116-139 (shape)
    (118, 33, 70, 0.5, 20, 2),     # acceptance.cpp:246 (shape)
    (42, 1024, 1024, 1 / 1.1, 100, 8),   # BASELINE config 1 (SURVEY 8c anchor)
    (5, 300, 20000, 1 / 1.1, 10, 8),     # rows spanning G > 1 CTAs on the GPU
    (9, 2000, 513, 0.9, 30, 8),          # ragged columns
]

# (seed, rows, cols, iterations) at BASELINE.json sizes, fi = 1/1.1, W = all cores
BIG = [
    (42, 8192, 8192, 10),
    (42, 32768, 32768, 4),
    (42, 262144, 4096, 4),
]  # 131072 x 32768 (16 GiB): the reference's matrix copies exceed this container's RAM


def er_ep(fi):
    return 1.0, (1.0 - fi) / fi  # oracle.hpp:61-67: er fixed at 1, fi = er/(er+ep)


def main():
    ref = oracle.RefOracle()
    o = oracle.Oracle()
    out = {}
    meta = []
    for (seed, m, n, fi, k, w) in SMALL:
        a, rpd, cpd = o.gen_problem(seed, m, n)
        er, ep = er_ep(fi)
        r = ref.fused_iterate_k(a, rpd, cpd, er, ep, w, k)
        key = f"s{seed}_{m}x{n}_k{k}_w{w}"
        if m * n <= 65536:
            out[key + "_plan"] = r.plan
        else:  # sampled rows + a digest of the whole plan keep the fixture small
            rows = np.unique(np.linspace(0, m - 1, 8).astype(np.int64))
            out[key + "_rows"] = rows
            out[key + "_plan_rows"] = r.plan[rows]
            out[key + "_plan_sum"] = np.array([float(np.sum(r.plan, dtype=np.float64))])
            out[key + "_plan_sha256"] = np.frombuffer(hashlib.sha256(r.plan.tobytes()).digest(), np.uint8)
        out[key + "_alpha"] = r.alpha
        out[key + "_beta"] = r.beta
        out[key + "_colsums"] = r.col_sums
        out[key + "_err"] = np.array([r.final_error])
        meta.append({"key": key, "seed": seed, "rows": m, "cols": n, "er": er, "ep": ep, "fi": fi,
                     "iterations": k, "workers": w})
    # Hand-checked KATs (test_fused.cpp:38-56, test_baseline.cpp:46-74), fp32.
    kat = {
        "kat_2x2": (np.ones((2, 2), np.float32), np.array([4.0, 2.0]), np.array([3.0, 3.0]), 1.0, 0.0, 1),
        "kat_1x1": (np.array([[2.0]], np.float32), np.array([4.0]), np.array([2.0]), 1.0, 0.0, 1),
        "kat_damped": (np.ones((1, 2), np.float32), np.array([8.0]), np.array([1.0, 1.0]), 1.0, 1.0, 1),
        "kat_fixed_point": (np.ones((6, 9), np.float32), np.full(6, 9.0), np.full(9, 6.0), 1.0, 1.0, 1),
    }
    for key, (a, rpd, cpd, er, ep, k) in kat.items():
        r = ref.fused_solve(a, rpd, cpd, er, ep, KNEVER, k, 1)
        out[key + "_a"] = a
        out[key + "_rpd"] = rpd
        out[key + "_cpd"] = cpd
        out[key + "_plan"] = r.plan
        out[key + "_alpha"] = r.alpha
        out[key + "_beta"] = r.beta
        out[key + "_err"] = np.array([r.final_error])
        meta.append({"key": key, "er": er, "ep": ep, "iterations": k, "kat": True})
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("small.npz:", len(meta), "cases")

    if "--big" not in sys.argv:
        return
    big = {}
    bmeta = []
    threads = os.cpu_count() or 1
    fi = 1 / 1.1
    er, ep = er_ep(fi)
    for (seed, m, n, k) in BIG:
        t0 = time.time()
        a, rpd, cpd = o.gen_problem(seed, m, n, threads=threads)
        r = ref.fused_iterate_k(a, rpd, cpd, er, ep, threads, k)
        del a
        key = f"b{seed}_{m}x{n}_k{k}"
        rows = np.array([0, 1, m // 2, m - 1])
        big[key + "_rows"] = rows
        big[key + "_plan_rows"] = r.plan[rows]
        stride = max(1, m // 4096)
        big[key + "_alpha_strided"] = r.alpha[::stride]
        big[key + "_alpha_stride"] = np.array([stride])
        cstride = max(1, n // 4096)
        big[key + "_beta_strided"] = r.beta[::cstride]
        big[key + "_colsums_strided"] = r.col_sums[::cstride]
        big[key + "_col_stride"] = np.array([cstride])
        big[key + "_sum"] = np.array([float(np.sum(r.plan, dtype=np.float64))])
        big[key + "_max"] = np.array([float(r.plan.max())])
        big[key + "_err"] = np.array([r.final_error])
        digest = hashlib.sha256(r.plan.tobytes()).hexdigest()
        bmeta.append({"key": key, "seed": seed, "rows": m, "cols": n, "iterations": k, "workers": threads,
                      "er": er, "ep": ep, "sha256_plan": digest,
                      "alpha0": float(r.alpha[0]), "beta0": float(r.beta[0]), "p00": float(r.plan[0, 0]),
                      "sum": float(big[key + "_sum"][0]), "final_error": r.final_error})
        print(key, f"{time.time() - t0:.1f}s", bmeta[-1], flush=True)
        del r
    np.savez_compressed(os.path.join(HERE, "big.npz"), **big)
    with open(os.path.join(HERE, "big.json"), "w") as f:
        json.dump(bmeta, f, indent=1)


if __name__ == "__main__":
    main()
