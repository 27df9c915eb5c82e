"""Summarise an ncu `--page source --csv --print-source sass` dump: total warp
instructions, the hottest instructions, and opcode mix weighted by execution count."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iE, iSm = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iE: continue
    try: n = int(r[iE]); s = int(r[iSm])
    except ValueError: continue
    data.append((r[iA], r[iS].strip(), n, s))
tot = sum(d[2] for d in data); tots = sum(d[3] for d in data)
print("total warp instructions", tot, "stall samples", tots)
mix = collections.Counter()
for a, s, n, _ in data:
    op = s.split()[0] if s else "?"
    if op.startswith("@"): op = s.split()[1]
    mix[op.split(".")[0]] += n
for op, n in mix.most_common(30): print(f"  {op:10s} {n/tot*100:5.1f}%")
if len(sys.argv) > 2:
    lo = int(sys.argv[2]); 
    for i, (a, s, n, sm) in enumerate(data):
        if n >= lo: print(i, a[-5:], n, sm, s)
