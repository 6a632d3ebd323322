"""Per-kernel-class summary of an ncu launch list taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
over whole eager steps (PST_GRAPHS=0).  Prints per-class launches / time share / DRAM
bytes per launch and writes profiles/traffic.json ({class: mean DRAM bytes per launch}),
the `roofline.traffic` figure bench.py reports for its dominant kernel class.

usage: python tools/ncu_traffic.py gpurun_out/traffic.csv [profiles/traffic.json]
"""
import collections
import csv
import json
import re
import sys


def kernel_class(name):
    if "conv_fwd_kernel" in name:
        m = re.search(r"conv_fwd_kernel<([^>]*)>", name)
        dg = m and m.group(1).replace(" ", "").split(",")[-1] in ("true", "1", "(bool)1")
        return "conv_dgrad" if dg else "conv_fwd"
    if "conv_ts_kernel" in name:   # template <KC, EPI, TPS>; EPI 3 = EPI_DGRAD
        m = re.search(r"conv_ts_kernel<([^>]*)>", name)
        epi = m.group(1).replace(" ", "").split(",")[1] if m else "0"
        return "conv_dgrad" if epi == "3" else "conv_fwd"
    if "conv_wgrad" in name:
        return "conv_wgrad"
    for key, cls in (("bn_apply", "bn_apply"), ("bwd_pre", "bwd_pre"), ("bn_bwd", "bn_bwd"), ("maxpool", "pool"),
                     ("gap_kernel", "pool"), ("sgd_kernel", "sgd"), ("softmax_ce", "loss")):
        if key in name:
            return cls
    return "misc"


def scale(v, unit):
    u = unit.lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
            "ns": 1e-3, "us": 1, "ms": 1e3}
    return v * mult.get(u, 1)


def main():
    path = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else None
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ii, ki, mi, vi, ui = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = scale(float(r[vi].replace(",", "")), r[ui])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in launches.values():
        a = agg[kernel_class(d["name"])]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{len(launches)} launches, {tot:.1f} us (serialised, cold-cache ncu timing)")
    print(f"  {'class':12s} {'n':>6s} {'time_us':>10s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>8s}")
    res = {}
    for cls, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {cls:12s} {n:6d} {t:10.1f} {t / tot:6.3f} {b / n / 1e6:10.3f} {b / (t * 1e3) if t else 0:8.1f}")
        res[cls] = b / n
    if out:
        json.dump(res, open(out, "w"), indent=1)
        print("wrote", out)


if __name__ == "__main__":
    main()
