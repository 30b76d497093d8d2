"""Summarise an ncu SASS source page (csv): stall totals and the hottest instructions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 45
h = rows[1]; data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
f = lambda x: float(x) if x not in ("", "-") else 0.0
si = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
stalls = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot = sum(f(r[si]) for r in data)
print("total samples", tot, "n instr", len(data))
agg = {c: sum(f(r[h.index(c)]) for r in data) for c in stalls}
for c, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"{c:28s} {v:10.0f} {100*v/max(tot,1):5.1f}%")
top = sorted(enumerate(data), key=lambda x: -f(x[1][si]))[:ntop]
for i, r in sorted(top):
    st = sorted(((f(r[h.index(c)]), c) for c in stalls), reverse=True)[:2]
    print(f"{i:5d} {f(r[si]):7.0f} ex={r[ie]:>9s} {r[1].strip()[:58]:58s} {st[0][1][6:]}:{st[0][0]:.0f} {st[1][1][6:]}:{st[1][0]:.0f}")
