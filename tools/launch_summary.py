"""Summarise an ncu launch list (gpu__time_duration.sum per launch): per-kernel totals and shares."""
import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
seq = []
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].split("<")[0].split("::")[-1]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * 1e3 if r[ui] in ("msecond", "ms") else v
    seq.append((name, v))
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in seq:
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{len(seq)} launches, {tot:.1f} us total (serialised, cold-cache ncu timing)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:28s} n={n:5d} total={t:9.1f}us avg={t / n:7.2f}us share={t / tot:.3f}")
if len(sys.argv) > 2:
    for n, v in seq:
        if sys.argv[2] in n:
            print(f"{n} {v:.1f}")
