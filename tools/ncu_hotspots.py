"""Top stall instructions of one ncu report (SASS source page), grouped with their stall
reasons: python tools/ncu_hotspots.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
R = rows[2:]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
s = [int(r[2] or 0) for r in R]
print("total samples", sum(s), "instructions", len(R))
for i in sorted(range(len(R)), key=lambda i: -s[i])[:top]:
    reasons = {c[6:]: int(float(R[i][idx[c]] or 0)) for c in cols if R[i][idx[c]] not in ("", "0")}
    reasons = dict(sorted(reasons.items(), key=lambda x: -x[1])[:3])
    ctx = " | ".join(R[j][1].strip()[:38] for j in range(max(0, i - 3), i))
    print(f"{s[i]:6d} {i:5d} {R[i][1].strip()[:50]:50s} {reasons}  <- {ctx}")
