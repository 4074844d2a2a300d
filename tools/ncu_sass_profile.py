"""Per-opcode dynamic instruction counts and stall samples of one kernel in an
ncu --set full report (source page, SASS view). Run here, no GPU needed.

python tools/ncu_sass_profile.py REPORT.ncu-rep ELEMENTS [--top N]
ELEMENTS: matrix elements one launch processes (per-element instruction rates).
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, elems = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops, stall, total, tstall = collections.Counter(), collections.Counter(), 0, 0
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", src)
    if not m:
        continue
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    op = m.group(2)
    ops[op] += n
    stall[op] += s
    total += n
    tstall += s
    lines.append((s, n, r[ix["Address"]], src))
print(f"warp instructions executed: {total:.4g}  = {total * 32 / elems:.2f} thread instructions per element")
print(f"{'opcode':28s} {'per elem':>9s} {'share':>7s} {'stall%':>7s}")
for op, n in ops.most_common(top):
    print(f"{op:28s} {n * 32 / elems:9.3f} {n / total:7.1%} {stall[op] / max(tstall, 1):7.1%}")
print("\nhottest instructions by stall samples:")
for s, n, a, src in sorted(lines, reverse=True)[:top]:
    print(f"{s / max(tstall, 1):6.1%} {n * 32 / elems:7.3f}/elem  {src[:90]}")
