"""Per-CUDA-source-line hot spots of an ncu report (instructions executed, stall samples)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None
hdr = None
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((samp, inst, fname, r[0], r[1].strip()[:90]))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"total samples {ts}  instructions {ti}")
for samp, inst, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*samp/ts:5.1f}% smp {100*inst/ti:5.1f}% ins  {f}:{ln}  {src}")
