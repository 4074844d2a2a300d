"""Assemble the judged evidence of one gpu_full.sh run into profiles/ (run here,
no GPU needed; ncu reports are read with `ncu -i`).

python tools/round_profiles.py TAG [ROUND]   e.g. tools/round_profiles.py r02z r02

Writes profiles/ROUND_{bench20,bench200,bench_ref}.json, _pytest_gpu.txt,
_facade.txt, _acceptance_gpu.txt, _configs.txt, _ablation.txt, _launches.csv,
_ncu.md (ncu --set full summaries of the sweep at 32768^2 and 8192^2 and of the
finalize, the per-opcode SASS profile, the launch-list shares) and
_sass_headline.md (static SASS histogram of the headline kernel), and refreshes
profiles/ncu_traffic.json from the captures.
"""
import csv
import collections
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else tag[:3]


def src(name):
    return os.path.join(OUT, f"{tag}_{name}")


def dst(name):
    return os.path.join(PROF, f"{rnd}_{name}")


for name in ("bench20.json", "bench200.json", "bench_ref.json", "pytest_gpu.txt", "facade.txt",
             "acceptance_gpu.txt", "configs.txt", "ablation.txt", "launches.csv", "gpu.txt"):
    if os.path.exists(src(name)):
        shutil.copy(src(name), dst(name))


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)


md = [f"# Round {rnd[1:]} ncu evidence (`tools/gpu_full.sh {tag}`, one B200)\n"]
traffic = {}
for rep, label, shape, elems in (("prof32", "sweep_kernel, 32768² (headline instance)", "32768x32768", 32768 * 32768),
                                 ("prof8k", "sweep_kernel, 8192² (config 2)", "8192x8192", 8192 * 8192),
                                 ("proffin", "finalize_kernel, 32768²", None, None)):
    path = src(f"{rep}.ncu-rep")
    if not os.path.exists(path):
        continue
    r = run([sys.executable, "tools/ncu_summary.py", path, label])
    md.append(r.stdout)
    try:
        t = json.loads(r.stderr.strip().splitlines()[-1])["traffic_bytes"]
        if shape:
            traffic[shape] = t
            md.append(f"Algorithmic bytes per launch (2·R·C·4): {2 * elems * 4 / 1e9:.3f} GB; "
                      f"DRAM/algorithmic = {t / (2 * elems * 4):.3f}\n")
    except (IndexError, KeyError, ValueError):
        pass
    if elems:
        p = run([sys.executable, "tools/ncu_sass_profile.py", path, str(elems), "--top", "25"])
        md.append("Per-opcode dynamic counts (`tools/ncu_sass_profile.py`, SASS source page):\n\n```\n"
                  + p.stdout.strip() + "\n```\n")

lc = src("launches.csv")
if os.path.exists(lc):
    rows = [r for r in csv.reader(open(lc)) if len(r) > 10]
    if rows:
        h = rows[0]
        ix = {k: i for i, k in enumerate(h)}
        dur = collections.defaultdict(list)
        for r in rows[1:]:
            if r[ix["Metric Name"]] == "gpu__time_duration.sum":
                dur[r[ix["Kernel Name"]].split("(")[0][:70]].append(float(r[ix["Metric Value"]].replace(",", "")))
        tot = sum(sum(v) for v in dur.values())
        md.append("## Launch list of a 20-step bench run (ncu `gpu__time_duration.sum`, serialised, cold caches)\n")
        md.append("| kernel | launches | mean µs | share of listed time |\n|---|---|---|---|")
        for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
        md.append("")

with open(dst("ncu.md"), "w") as f:
    f.write("\n".join(md) + "\n")

r = run([sys.executable, "tools/sass_histogram.py"])
with open(dst("sass_headline.md"), "w") as f:
    f.write(r.stdout)

if traffic:
    tj = os.path.join(PROF, "ncu_traffic.json")
    old = json.load(open(tj)) if os.path.exists(tj) else {}
    old.update(traffic)
    old["_source"] = (f"profiles/{rnd}_ncu.md (dram__bytes_read.sum + dram__bytes_write.sum, one sweep launch, "
                      f"ncu --set full, gpu_full.sh {tag})")
    json.dump(old, open(tj, "w"), indent=1)
print("wrote", sorted(x for x in os.listdir(PROF) if x.startswith(rnd)))
