"""Per-launch table from an ncu --csv launch list with several metrics per launch.

Groups launches by (kernel, grid) — the grid identifies the layer shape class — and prints
count, mean time, DRAM MB and GB/s, tensor-pipe %.  Usage: launch_table.py launches.csv [steps]
"""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
I = {k: h.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value")}
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= I["Metric Value"]:
        continue
    lid = r[I["ID"]]
    d = launch.setdefault(lid, {"name": r[I["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1],
                                "grid": r[I["Grid Size"]]})
    v = float(r[I["Metric Value"]].replace(",", ""))
    u = r[I["Metric Unit"]]
    m = r[I["Metric Name"]]
    if m == "gpu__time_duration.sum":
        v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
        d["us"] = v
    elif m.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        d["bytes"] = d.get("bytes", 0.0) + v * scale
    elif "tensor" in m:
        d["tensor"] = v
agg = collections.OrderedDict()
for d in launch.values():
    k = (d["name"], d["grid"])
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("us", 0.0)
    a[2] += d.get("bytes", 0.0)
    a[3] += d.get("tensor", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{len(launch)} launches, {tot:.1f} us total ({tot / steps:.1f} us/step over {steps:g} steps)")
print(f"{'kernel':34s} {'grid':16s} {'n':>5s} {'avg_us':>8s} {'tot_us':>9s} {'share':>6s} {'MB':>7s} {'GB/s':>7s} {'tc%':>5s}")
for (n, g), (c, t, b, tc) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:34]:34s} {g:16s} {c:5d} {t / c:8.2f} {t:9.1f} {t / tot:6.3f} {b / c / 1e6:7.2f} "
          f"{(b / c) / (t / c * 1e3) if t else 0:7.0f} {tc / c:5.1f}")
