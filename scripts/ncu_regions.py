"""Stall reasons per SASS region of an ncu source page CSV (dev aid).
usage: ncu_regions.py src.csv  -> regions = runs of instructions with similar execution counts."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, iex, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), int(r[iex]), int(r[ist]), [int(r[i] or 0) for i in sc]))
    except Exception:
        pass
data.sort()
tot = sum(d[2] for d in data)
segs, cur = [], None
for a, e, s, st in data:
    if cur is None or (e != cur[2] and abs(e - cur[2]) > 0.05 * max(cur[2], 1)):
        cur = [a, a, e, 0, [0] * len(sc), 0]
        segs.append(cur)
    cur[1] = a; cur[3] += s; cur[5] += 1
    cur[4] = [x + y for x, y in zip(cur[4], st)]
for a0, a1, e, s, st, n in segs:
    if s > float(sys.argv[2] if len(sys.argv) > 2 else 0.01) * tot:
        top = sorted(zip(st, [h[i][6:] for i in sc]), reverse=True)[:4]
        print(f"{a0 & 0xfffff:05x}-{a1 & 0xfffff:05x} n={n:4d} exec={e:8d} {100 * s / tot:5.1f}%  " +
              " ".join(f"{k}:{100 * v / max(s, 1):.0f}%" for v, k in top))
