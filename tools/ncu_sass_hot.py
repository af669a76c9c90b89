"""Hottest SASS instructions of an ncu report (source page, SASS view) with their dominant stall reasons:
python tools/ncu_sass_hot.py <report.ncu-rep> [top] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = rows[1:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot}, instructions {len(data)}")
for i in order[:top]:
    r = data[i]
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{i:6d} {100*smp/tot:5.2f}%  {r[ix['Source']].strip()[:60]:60s} " + " ".join(f"{k}={v}" for v, k in st if v))
