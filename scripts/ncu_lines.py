"""Per-source-line warp-stall samples from an ncu report (cuda,sass source page).
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
cur = None
agg = collections.Counter()
stalls = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else cur
        src[cur] = r[1]
    try:
        n = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    agg[cur] += n
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and r[i] and r[i] != "0":
            try:
                stalls[cur][h[6:]] += int(float(r[i]))
            except ValueError:
                pass
tot = sum(agg.values())
print(f"total samples {tot}")
for ln, n in agg.most_common(top):
    s = ", ".join(f"{k} {v}" for k, v in stalls[ln].most_common(3))
    print(f"{ln:5d} {100*n/tot:5.1f}%  {src.get(ln,'')[:70]:70s} | {s}")
