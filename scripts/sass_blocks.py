"""Basic-block view of an ncu SASS source dump (csv or csv.gz): blocks (runs of equal
execution count) ranked by executed warp instructions, with opcode mix and stalls."""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
iA, iS, iE, iW = (h.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iA], 16), r[iS].strip(), int(r[iE]), int(r[iW])))
    except (ValueError, IndexError):
        pass
blocks, cur = [], None
for a, s, n, w in data:
    if cur and cur["n"] == n and a == cur["end"] + 16:
        cur["ins"].append(s); cur["end"] = a; cur["w"] += w
    else:
        cur = {"start": a, "end": a, "n": n, "ins": [s], "w": w}
        blocks.append(cur)
tot = sum(b["n"] * len(b["ins"]) for b in blocks)
totw = sum(b["w"] for b in blocks)
print(f"total warp instructions {tot}, stall samples {totw}")
for b in sorted(blocks, key=lambda b: -b["n"] * len(b["ins"]))[:top]:
    ops = [x.split()[1] if x.startswith("@") else x.split()[0] for x in b["ins"] if x]
    c = collections.Counter(o.split(".")[0] for o in ops)
    print(f"{b['start'] & 0xfffff:05x} n={b['n']:>10d} len={len(b['ins']):>4d} "
          f"instr={100 * b['n'] * len(b['ins']) / tot:5.1f}% stall={100 * b['w'] / max(totw, 1):5.1f}% "
          + " ".join(f"{k}:{v}" for k, v in c.most_common(7)))
