"""Table of the configs[3] sweep under ncu: per (S, N) point the encode_tc launches' summed duration and
their duration-weighted tensor-pipe activity (sm__pipe_tensor_cycles_active, % of peak over elapsed)."""
import csv, sys
points = [tuple(map(int, l.split()[1:])) for l in open(sys.argv[1]) if l.startswith("POINT")]
rows = [r for r in csv.reader(l for l in open(sys.argv[2]) if not l.startswith("==")) if r]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
launch = {}
for r in rows[1:]:
    d = launch.setdefault(int(r[ki]), {})
    v = float(r[vi].replace(",", ""))
    if r[ui] in ("nsecond", "ns"):
        v /= 1e6
    elif r[ui] in ("usecond", "us"):
        v /= 1e3
    d[r[mi]] = v
ids = sorted(launch)
print("| S | N | encode_tc launches | ncu ms (sum) | TFLOP/s (ncu time) | tensor pipe active (% of elapsed, duration-weighted) |")
print("|---|---|---|---|---|---|")
i = 0
for S, N, n in points:
    ls = [launch[k] for k in ids[i:i + n]]
    i += n
    t = sum(l["gpu__time_duration.sum"] for l in ls)
    tp = sum(l["gpu__time_duration.sum"] * l["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"] for l in ls) / t
    fl = 2 * 128 * S * N * (1 << 20)
    print(f"| {S} | {N} | {n} | {t:.3f} | {fl / t / 1e9:.0f} | {tp:.1f} |")
