"""Shared-memory instructions of an ncu report ranked by excessive (bank-conflict) wavefronts:
python tools/ncu_smem_conflicts.py <report.ncu-rep> [top] [kernel index]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
# one section per profiled kernel, each starting with a "Kernel Name" line; argv[3] picks one (default 0)
secs = [s for s in out.split('"Kernel Name"') if s.strip()]
sec = secs[int(sys.argv[3]) if len(sys.argv) > 3 else 0]
rows = list(csv.reader(io.StringIO("\n".join(sec.splitlines()[1:]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = rows[1:]
num = lambda r, k: float(r[ix[k]] or 0) if r[ix[k]] not in ("-", "") else 0.0
tot_ex = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
tot = sum(num(r, "L1 Wavefronts Shared") for r in data)
print(f"shared wavefronts {tot:.3e}, excessive {tot_ex:.3e}")
order = sorted(range(len(data)), key=lambda i: -num(data[i], "L1 Wavefronts Shared Excessive"))
for i in order[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    r = data[i]
    print(f"{i:6d} ex {num(r, 'L1 Wavefronts Shared Excessive'):.3e} all {num(r, 'L1 Wavefronts Shared'):.3e} ideal {num(r, 'L1 Wavefronts Shared Ideal'):.3e}  {r[ix['Source']].strip()[:70]}")
