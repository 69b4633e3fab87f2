"""Summarise an ncu --set full capture of k_sweep (with --import-source): the
headline throughputs (DRAM, issue, fp64 pipe), the stall reasons per issue,
and the source lines with the most warp-stall samples (SASS addresses mapped
to lines with nvdisasm --print-line-info of the same build's cubin).
  python tools/ncu_hotlines.py REPORT.ncu-rep KERNEL_MANGLED_NAME OBJ.o [N]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

rep, name, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum"]
for i, n in enumerate(h):
    if n in want or (n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")):
        print(f"{n} [{u[i]}] = {v[i]}")
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True,
                          text=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text." + name + ":")][0]
m, cur = {}, "?"
for l in sass[start + 1:]:
    if l.startswith(".text.") or ".section" in l:
        break
    mm = re.search(r'## File "([^"]*)", line (\d+)', l)
    if mm:
        cur = mm.group(1).split("/")[-1] + ":" + mm.group(2)
        continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo:
        m[int(mo.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, data = rows[1], rows[2:]
ia, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
ci, cs = Counter(), Counter()
for r in data:
    k = m.get(int(r[0], 16) - base, "?")
    ci[k] += int(r[ia] or 0)
    cs[k] += int(r[isamp] or 0)
ti, ts = sum(ci.values()), sum(cs.values())
here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2406_13191_b200", "csrc")
files = {}
print(f"\nsource lines by warp-stall samples (of {ts} samples, {ti} warp instructions; "
      f"{len(data)} SASS instructions mapped {sum(1 for r in data if int(r[0], 16) - base in m)})")
for k, n in cs.most_common(top):
    text = ""
    if ":" in k:
        f, ln = k.split(":")
        p = os.path.join(here, f)
        if p not in files and os.path.exists(p):
            files[p] = open(p).read().split("\n")
        text = files.get(p, [""] * int(ln))[int(ln) - 1].strip()[:90]
    print(f"{n / ts * 100:5.1f}% samples {ci[k] / ti * 100:5.1f}% inst  {k:24s} {text}")
