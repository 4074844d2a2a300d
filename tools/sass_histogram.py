"""Static SASS evidence for one kernel of libuot_cuda.so: opcode histogram
(UBLKCP = cp.async.bulk / TMA engine, LDTM/STTM = tcgen05.ld/st Tensor Memory,
SYNCS = mbarrier), registers and spills from ptxas (-Xptxas -v, build.log).

python tools/sass_histogram.py [MANGLED_NAME] > profiles/rNN_sass_headline.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2412_11079_b200", "libuot_cuda.so")
LOG = os.path.join(ROOT, "paper_2412_11079_b200", "build.log")
HEADLINE = "_ZN4uotk12sweep_kernelILi512ELi4ELi1ELi7ELi2ELb1ELi3ELb1ELb0EfLb1EEEvNS_9SweepArgsE"

name = sys.argv[1] if len(sys.argv) > 1 else HEADLINE
sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
block = next(b for b in sass.split("Function : ") if b.startswith(name))
ops = collections.Counter()
total = 0
for line in block.splitlines():
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
    if m:
        ops[m.group(2)] += 1
        total += 1
props = ""
if os.path.exists(LOG):
    text = open(LOG).read()
    i = text.find(f"Function properties for {name}")
    if i >= 0:
        props = " ".join(text[i:i + 600].splitlines()[1:4])
regs = re.search(r"Used (\d+) registers", props or "")
print(f"# SASS of `{name}`\n")
print(f"- instructions (static): {total}")
print(f"- ptxas: {props.strip() or 'n/a'}")
print()
groups = {
    "TMA bulk copies (UBLKCP)": ("UBLKCP",),
    "Tensor Memory (LDTM / STTM)": ("LDTM", "STTM"),
    "mbarrier / async sync (SYNCS*)": ("SYNCS",),
    "f64 products / sums (DMUL / DADD / DFMA)": ("DMUL", "DADD", "DFMA"),
    "conversions (F2F*)": ("F2F",),
    "shared memory (LDS / STS)": ("LDS", "STS"),
}
print("| class | opcodes | static count |\n|---|---|---|")
for g, prefixes in groups.items():
    keys = sorted(k for k in ops if k.split(".")[0] in prefixes or any(k.startswith(p + ".") for p in prefixes))
    print(f"| {g} | {', '.join(keys)} | {sum(ops[k] for k in keys)} |")
print("\n## Full opcode histogram\n\n| opcode | count |\n|---|---|")
for k, v in ops.most_common():
    print(f"| {k} | {v} |")
