"""Summarise an ncu report: key metrics per kernel + SASS opcode mix (for profiles/)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
KEYS = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
        "Theoretical Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
        "Block Limit Shared Mem", "Block Limit Registers", "Grid Size", "Block Size", "Executed Instructions")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
iK, iID, iM, iU, iV = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"),
                      h.index("Metric Value"))
seen = collections.OrderedDict()
for r in rows[1:]:
    key = (r[iID], r[iK][:70])
    seen.setdefault(key, {})
    if r[iM] in KEYS:
        seen[key][r[iM]] = f"{r[iV]} {r[iU]}".strip()
for (i, k), m in seen.items():
    print(f"== launch {i}: {k}")
    for kk in KEYS:
        if kk in m:
            print(f"   {kk}: {m[kk]}")
# opcode mix + dram bytes
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
want = [c for c in hh if c.startswith("dram__bytes_read.sum") or c.startswith("dram__bytes_write.sum")
        or c.startswith("sm__inst_executed_pipe_fp64") or c.startswith("sm__pipe_fp64_cycles_active")
        or c.startswith("smsp__inst_executed_op_dmma") or "pipe_fp64" in c and "pct" in c]
for r in rr[2:]:
    print("   raw:", r[hh.index("Kernel Name")][:40], {c: r[hh.index(c)] for c in want[:12]})
