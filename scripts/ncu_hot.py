"""Summarise an ncu source page (SASS) CSV: top stall instructions and per-opcode totals."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia = hdr.index("Address"); isrc = hdr.index("Source"); ist = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ist]), r[ia], r[isrc].strip(), int(r[iex])))
    except Exception:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = {d[1]: i for i, d in enumerate(data)}
for s, a, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{s:8d} {100*s/tot:5.1f}% {ex:10d} {a[-5:]} {src[:90]}")
ops = collections.Counter()
exs = collections.Counter()
for s, a, src, ex in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += s
    exs[op] += ex
print("--- by opcode (samples, executed)")
for op, s in ops.most_common(25):
    print(f"{op:12s} {s:8d} {100*s/tot:5.1f}%  exec {exs[op]}")
