"""Top source lines by warp-stall samples from an .ncu-rep (needs -lineinfo).  usage: stall_lines.py rep [n]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"; agg = collections.defaultdict(lambda: [0.0, collections.Counter(), ""]); hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or r[0] == "Function Name": continue
    try: v = float(r[4])
    except ValueError: continue
    k = (fname, r[0]); a = agg[k]; a[0] += v; a[2] = r[1][:90]
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try: a[1][name[6:]] += float(r[i])
            except ValueError: pass
tot = sum(a[0] for a in agg.values()) or 1
for (f, ln), (v, c, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    top = ",".join(f"{k}:{int(x)}" for k, x in c.most_common(3) if x)
    print(f"{v / tot:6.3f} {f}:{ln:>4} {s:90s} {top}")
