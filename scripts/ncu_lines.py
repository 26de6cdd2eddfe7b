"""Attribute an ncu source-page capture (SASS level) to CUDA source lines.

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep KERNEL_REGEX [csrc/file.cu] [N]

Recompiles nothing: it disassembles the in-tree build/csrc/<file>.o with
nvdisasm -g (line info) and joins on the instruction offset."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
srcfile = sys.argv[3] if len(sys.argv) > 3 else "paper_2305_17408_b200/csrc/ag_fused.cu"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors.sum", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread"]:
    print(k, d.get(k))
for k in r[0]:
    if "smsp__average_warps_issue_stalled" in k and float(d[k] or 0) > 0.1:
        print("  stall", k[34:].replace("_per_issue_active.ratio", ""), d[k])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
rows = rows[2:]
ii = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
import os
obj = os.path.abspath("build/csrc/" + srcfile.split("/")[-1] + ".o")
subprocess.run(["cuobjdump", "-xelf", "all", obj], capture_output=True, cwd="/tmp")
cub = "/tmp/" + srcfile.split("/")[-1].replace(".cu", ".sm_100a.cubin")
txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
# the profiled kernel's own (mangled) name, so template instances do not mix
mangled = ""
rawm = subprocess.run(["ncu", "-i", rep, "--print-kernel-base", "mangled", "--page", "raw", "--csv"],
                      capture_output=True, text=True).stdout
rm = list(csv.reader(io.StringIO(rawm)))
if len(rm) > 2:
    mangled = dict(zip(rm[0], rm[2])).get("Kernel Name", "")
starts = [i for i, l in enumerate(txt) if l.strip().startswith(".section") and ".text." in l
          and (mangled and (".text." + mangled) in l)]
if not starts:
    starts = [i for i, l in enumerate(txt) if l.strip().startswith(".section") and ".text." in l
              and re.search(kre, l)]
m = {}
line = None
for l in txt[starts[0] + 1:]:
    if l.strip().startswith(".section"):
        break
    mm = re.search(r'//## File ".*", line (\d+)', l)
    if mm:
        line = int(mm.group(1))
        continue
    mm = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mm and line is not None:
        m[int(mm.group(1), 16)] = line
base = int(rows[0][0], 16)
agg = defaultdict(lambda: [0, 0])
for x in rows:
    ln = m.get(int(x[0], 16) - base, -1)
    agg[ln][0] += int(x[ii])
    agg[ln][1] += int(x[si])
lines = open(srcfile).read().split("\n")
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
print("instructions", tot, "samples", tots)
print("line  %instr  %stall  source")
ORDER = os.environ.get("ORDER")
items = sorted(agg.items(), key=lambda kv: -kv[1][0] - kv[1][1] * tot / max(tots, 1))[:N]
if ORDER: items.sort()
for ln, (n, s) in items:
    print(f"{ln:5d} {n / tot * 100:6.1f} {s / tots * 100:6.1f}  " + (lines[ln - 1].strip()[:90] if ln > 0 else "?"))
