"""Copy one evidence run (tools/_job_final.sh output) into profiles/ under a tag:
bench lines, reference arm, pytest/smoke logs, the launch list (gpu__time_duration.sum rows of the
ncu capture), per-class DRAM traffic (profiles/traffic.json for bench.py's roofline.traffic), and
summaries of the full ncu captures.   usage: python tools/make_profiles.py gpurun_out/f3 r1d"""
import csv, os, shutil, subprocess, sys

run, tag = sys.argv[1], sys.argv[2]
P = "profiles"
for src, dst in [("bench.json", "bench.json"), ("bench2.json", "bench_repeat.json"), ("bench_repeat.json", "bench_repeat.json"),
                 ("bench_ref.json", "bench_reference.json"), ("bench_reference.json", "bench_reference.json"),
                 ("bench_n2_shared_gpu.json", "bench_n2_shared_gpu.json"), ("stage_times.jsonl", "stage_times.jsonl"),
                 ("tg.log", "pytest_gpu.log"), ("smoke.log", "smoke.log")]:
    if os.path.exists(os.path.join(run, src)):
        shutil.copy(os.path.join(run, src), os.path.join(P, f"{tag}_{dst}"))
rows = list(csv.reader(open(os.path.join(run, "traffic.csv"))))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
mi = rows[h].index("Metric Name")
with open(os.path.join(P, f"{tag}_launches.csv"), "w") as f:
    csv.writer(f).writerows([rows[h]] + [r for r in rows[h + 1:] if len(r) > mi and r[mi] == "gpu__time_duration.sum"])
with open(os.path.join(P, f"{tag}_launch_list_summary.txt"), "w") as f:
    f.write(subprocess.run([sys.executable, "tools/launch_summary.py", os.path.join(P, f"{tag}_launches.csv")],
                           capture_output=True, text=True).stdout)
with open(os.path.join(P, f"{tag}_traffic_by_class.txt"), "w") as f:
    f.write(subprocess.run([sys.executable, "tools/ncu_traffic.py", os.path.join(run, "traffic.csv"),
                            os.path.join(P, "traffic.json")], capture_output=True, text=True).stdout)
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.sum", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for name in ("wgrad", "ts", "bn_apply"):
    rep = os.path.join(run, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hd, units, v = r[0], r[1], r[2] if len(r) > 2 else r[1]
    lines = [f"ncu --set full capture (one launch, cold cache, --clock-control none): {rep}"]
    lines += [f"  {k} = {v[hd.index(k)]} ({units[hd.index(k)]})" for k in KEYS if k in hd]
    st = [(float(v[i]), hd[i]) for i in range(len(hd)) if hd[i].startswith("smsp__pcsamp_warps_issue_stalled")
          and not hd[i].endswith("not_issued") and v[i].replace(".", "").isdigit()]
    st.sort(reverse=True)
    tot = sum(x for x, _ in st) or 1.0
    lines.append("  warp stall samples (top):")
    lines += [f"   {100 * x / tot:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}" for x, k in st[:8]]
    open(os.path.join(P, f"{tag}_ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
print("wrote profiles for", tag)
