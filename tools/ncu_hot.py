"""Per-opcode instruction/stall breakdown of the hottest code in an ncu report."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

path = sys.argv[1]
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
ci = {c: hdr.index(c) for c in cols}
tot_inst = sum(int(r[iE] or 0) for r in data)
byop, stall = Counter(), defaultdict(Counter)
for r in data:
    s = r[iS].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0] if s else "?"
    byop[op] += int(r[iE] or 0)
    for c in cols:
        stall[c][op] += int(r[ci[c]] or 0)
T = sum(sum(v.values()) for v in stall.values()) or 1
print("total warp instructions", tot_inst)
for op, n in byop.most_common(16):
    print(f"  {op:10s} {n / tot_inst * 100:5.1f}%")
for c in sorted(cols, key=lambda c: -sum(stall[c].values()))[:8]:
    print(f"{c:24s} {sum(stall[c].values()) / T * 100:5.1f}%  {stall[c].most_common(4)}")
cnt = Counter(int(r[iE] or 0) for r in data)
print("execution-count classes (count x #instrs):", sorted(cnt.items(), key=lambda kv: -kv[0] * kv[1])[:6])
