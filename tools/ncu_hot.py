"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iall, inot = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Warp Stall Sampling (Not-issued Samples)")
iex = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iall] or 0), int(r[inot] or 0), r[ia], r[isrc], r[iex]))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{d[0]:7d} {100*d[0]/tot:5.1f}% {d[2]} ex={d[4]:>10} {d[3][:90]}")
