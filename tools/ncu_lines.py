"""Instructions executed per CUDA source line of one kernel in an ncu report
(run here, no GPU):  python tools/ncu_lines.py REP KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and r[0].isdigit() and r[iE] not in ("", "-"):
        try:
            out.append((int(r[iE]), int(r[iS] or 0), cur, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
samp = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot}")
for n, s, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{n / tot * 100:5.1f}% inst {s / samp * 100:5.1f}% samples  {f}:{ln}  {src}")
