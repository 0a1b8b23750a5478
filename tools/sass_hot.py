"""Hot SASS instructions of one ncu source-page export (--page source --csv --print-source sass):
stall samples per instruction with the top stall reasons, plus per-region totals."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
h = r[1]
rows = [x for x in r[2:] if x and x[0].startswith("0x")]
si = h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
num = lambda v: float(v) if v not in ("", "-") else 0.0
tot = sum(num(x[si]) for x in rows)
agg = {h[c]: sum(num(x[c]) for x in rows) for c in sc}
print(f"samples {tot:.0f} over {len(rows)} instructions;",
      ", ".join(f"{k[6:]} {v:.0f}" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(rows)), key=lambda i: -num(rows[i][si]))[:n]
for i in sorted(top):
    x = rows[i]
    rs = sorted(((h[c][6:], num(x[c])) for c in sc), key=lambda t: -t[1])[:2]
    print(f"{i:6d} {num(x[si]):5.0f}  {x[1].strip()[:70]:70s} {rs}")
