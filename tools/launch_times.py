"""Per-kernel device times from an ncu --metrics gpu__time_duration.sum --csv log
(run here):  python tools/launch_times.py LOG [last_n | --group]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
if len(sys.argv) > 2 and sys.argv[2] == "--group":
    acc = defaultdict(list)
    for r in rows:
        name = re.sub(r"\(hth::\w+\)$", "", r[4].replace("void ", ""))
        acc[name].append(float(r[-1]) / 1e3)
    for k, v in sorted(acc.items()):
        print(f"{sum(v) / len(v):9.2f} us x{len(v):<4d} {k[:80]}")
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for r in rows[-n:]:
        print(f"{float(r[-1]):10.2f} {r[-2]:>6s}  {r[4][:90]}")
