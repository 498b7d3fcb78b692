"""Print the SASS lines of an ncu source-page CSV (--print-source sass) with the
most warp-stall samples, with +-N lines of context.
  python tools/sass_hot.py page.csv [top] [ctx]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
src = h.index("Source")
tot = sum(int(r[si] or 0) for r in data)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
order = sorted(range(len(data)), key=lambda i: -int(data[i][si] or 0))[:top]
print("total samples", tot)
for i in sorted(order) if ctx == 0 else order:
    r = data[i]
    print(f"{i:5d} {100*int(r[si])/tot:5.1f}% ex={r[ei]:>8} {r[src].strip()}")
    if ctx:
        for j in range(max(0, i - ctx), min(len(data), i + ctx + 1)):
            if j != i:
                print(f"      {j:5d} {100*int(data[j][si])/tot:5.1f}% {data[j][src].strip()}")
        print()


def by_reason(path, reason, top=15):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    d = rows[2:]
    ri = h.index(reason)
    tot = sum(float(r[ri] or 0) for r in d)
    print(f"== {reason}: {tot:.0f} samples")
    for i in sorted(range(len(d)), key=lambda i: -float(d[i][ri] or 0))[:top]:
        print(f"{i:5d} {float(d[i][ri] or 0):7.0f} {d[i][h.index('Source')].strip()}")
