"""A/B of library builds on one B200: alternating runs, each build in its own
process (UOT_LIB_PATH), device-timed K iterations per shape.

python tools/lib_ab.py LIB_A.so LIB_B.so [...] [--shapes 32768x32768x200,...]
       [--reps 2] [--schedule weighted|uniform|dynamic] [--sustained-s S] [--json OUT]

--sustained-s S: after the K-iteration run, S seconds of back-to-back
iterations with nvidia-smi sampling (median SM clock and power under load).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def inner():
    sys.path.insert(0, ROOT)
    from paper_2412_11079_b200 import uot
    schedule = arg("--schedule", "weighted")
    out = []
    for spec in arg("--shapes", "").split(","):
        m, n, k = (int(x) for x in spec.split("x"))
        with uot.Session(m, n) as s:
            s.generate_problem(42, 1.0, 0.1)
            s.init_col_sums()
            sched = schedule
            if sched == "weighted":
                if s.layout.get("pinned"):
                    s.calibrate_schedule(4)
                else:
                    sched = "uniform"
            s.set_schedule(sched)
            s.iterate(5, 1e-300)
            it, _, _, ms = s.iterate_timed(k, 1e-300)  # whole-step time, no per-kernel events
            s.set_timing(True)  # per-kernel breakdown on a separate short run (events add gaps)
            s.iterate(min(k, 50), 1e-300)
            sw, fin, ns = s.timing()
            s.set_timing(False)
            row = {"shape": spec, "schedule": sched, "us_iter": ms / it * 1e3, "sweep_us": sw / ns * 1e3,
                   "fin_us": fin / ns * 1e3, "gbs": 2 * m * n * 4 / (ms / it * 1e-3) / 1e9}
            sus = float(arg("--sustained-s", 0))
            if sus > 0:
                import statistics
                import subprocess
                import time
                ks = max(k, int(sus / (ms / it * 1e-3)))
                smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                        "-lms", "100"], stdout=subprocess.PIPE, text=True)
                time.sleep(0.2)
                it2, _, _, ms2 = s.iterate_timed(ks, 1e-300)
                smi.terminate()
                vals = [ln.split(",") for ln in smi.communicate()[0].splitlines() if "," in ln]
                clk = [float(v[0]) for v in vals if v[0].strip().replace(".", "").isdigit()]
                pw = [float(v[1]) for v in vals if v[1].strip().replace(".", "").isdigit()]
                row.update({"sus_us_iter": ms2 / it2 * 1e3, "sus_gbs": 2 * m * n * 4 / (ms2 / it2 * 1e-3) / 1e9,
                            "sus_sm_mhz": statistics.median(clk) if clk else None,
                            "sus_power_w": statistics.median(pw) if pw else None})
            out.append(row)
    print("JSON" + json.dumps(out), flush=True)


def main():
    if "--inner" in sys.argv:
        return inner()
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    reps = int(arg("--reps", 2))
    passthru = []
    for k in ("--shapes", "--schedule", "--sustained-s"):
        if k in sys.argv:
            passthru += [k, arg(k, "")]
    if "--shapes" not in passthru:
        passthru += ["--shapes", "8192x8192x500,32768x32768x200,262144x4096x200,131072x32768x50"]
    res = {lib: [] for lib in libs}
    for r in range(reps):
        for lib in libs:
            env = dict(os.environ, UOT_LIB_PATH=os.path.abspath(lib), UOT_AUTOBUILD="0")
            p = subprocess.run([sys.executable, os.path.abspath(__file__), "--inner", *passthru], env=env,
                               capture_output=True, text=True, timeout=int(arg("--proc-timeout", 1200)))
            line = next((x for x in p.stdout.splitlines() if x.startswith("JSON")), None)
            if line is None:
                print(f"{lib}: failed\n{p.stdout[-2000:]}\n{p.stderr[-2000:]}", flush=True)
                continue
            rows = json.loads(line[4:])
            res[lib].append(rows)
            for x in rows:
                sus = (f"  | sustained {x['sus_us_iter']:8.1f} us/iter {x['sus_gbs']:6.0f} GB/s "
                       f"{x['sus_sm_mhz']} MHz {x['sus_power_w']} W") if "sus_us_iter" in x else ""
                print(f"rep {r} {os.path.basename(lib):28s} {x['shape']:20s} {x['schedule']:8s} "
                      f"{x['us_iter']:9.1f} us/iter  {x['gbs']:6.0f} GB/s  sweep {x['sweep_us']:9.1f}  "
                      f"fin {x['fin_us']:5.1f}{sus}", flush=True)
    if "--json" in sys.argv:
        with open(arg("--json", ""), "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
