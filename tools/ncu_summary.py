"""Summarise an ncu --set full report of the sweep kernel (run here, no GPU needed).

python tools/ncu_summary.py REPORT.ncu-rep LABEL  -> markdown on stdout, traffic json line on stderr
"""
import csv
import io
import json
import subprocess
import sys

rep, label = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def f(k):
    v = d.get(k, ("", ""))[0].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return None


keys = [
    ("Kernel", "Kernel Name"), ("Grid", "launch__grid_size"), ("Block", "launch__block_size"),
    ("Registers/thread", "launch__registers_per_thread"), ("Dynamic smem/block (B)", "launch__shared_mem_per_block_dynamic"),
    ("Duration (ns)", "gpu__time_duration.sum"), ("SM clock (Hz)", "sm__cycles_elapsed.avg.per_second"),
    ("DRAM read (B)", "dram__bytes_read.sum"), ("DRAM write (B)", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Issue active % (SMSP)", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("ALU pipe %", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("XU pipe % (F2F)", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("Tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("Warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
]
out = [f"### {label}", "", "| metric | value |", "|---|---|"]
for name, k in keys:
    v = d.get(k, ("n/a", ""))
    out.append(f"| {name} | {v[0]} {v[1]} |")
st = [(k, f(k)) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
st = [(k, v) for k, v in st if v]
st.sort(key=lambda x: -x[1])
tot = sum(v for _, v in st) or 1
out += ["", "Top warp stall reasons (pc sampling):", ""]
out += [f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%" for k, v in st[:8]]
dur = f("gpu__time_duration.sum")
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
if dur and rd is not None:
    unit_mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    rdb = rd * unit_mult.get(d["dram__bytes_read.sum"][1], 1)
    wrb = wr * unit_mult.get(d["dram__bytes_write.sum"][1], 1)
    dur_s = dur * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                   "s": 1.0}.get(d["gpu__time_duration.sum"][1], 1e-9)
    out += ["", f"DRAM traffic per launch: {(rdb + wrb) / 1e9:.3f} GB "
                f"({(rdb + wrb) / dur_s / 1e9:.0f} GB/s under ncu replay, cold cache)"]
    sys.stderr.write(json.dumps({"label": label, "traffic_bytes": rdb + wrb}) + "\n")
print("\n".join(out))
