"""Group an ncu launch list (gpu__time_duration.sum [+ launch__grid_size]) by full kernel name
(template arguments included): count, total and mean time per group, in launch order of first use."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("(anonymous namespace)::", "")})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * 1e3 if r[ui] in ("msecond", "ms") else v
        d["us"] = v
    else:
        d[r[mi]] = v
agg = collections.OrderedDict()
for d in launch.values():
    key = (d["name"], int(d.get("launch__grid_size", 0)))
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += d.get("us", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{len(launch)} launches, {tot:.1f} us")
for (n, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n[:60]:60s} grid={g:5d} n={c:4d} total={t:8.1f}us avg={t / c:6.2f}us")
