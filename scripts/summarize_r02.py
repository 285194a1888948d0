"""Round-2 profile summaries into profiles/: per-kernel launch-list shares of the
configs[2] bench (ncu gpu__time_duration, cold/serialised), ncu --set full
details of the node-block kernels (configs[2] scene batch, configs[3] and
configs[4] single systems) and the DRAM traffic of the configs[2] capture.
usage: python scripts/summarize_r02.py <tag of the gpurun_out files, e.g. r2j> <profile prefix, e.g. r02>"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, pre = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out, prof = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")

rows = list(csv.reader(open(os.path.join(out, f"{tag}_launches.csv"))))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())
lines = [f"# ncu launch list, configs[2] bench.py --steps 1 --warmup 0 --e2e-steps 1 (timed run + e2e run)",
         f"# {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.1f} ms of kernel time (cold, serialised)",
         f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k[:70]:70s} {n:8d} {t / 1e3:10.2f} {t / tot:7.1%}")
open(os.path.join(prof, f"{pre}_cfg2_launches_summary.txt"), "w").write("\n".join(lines) + "\n")

want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__grid_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__pcsamp_sample_count",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_membar",
        "local_load_bytes", "local_store_bytes"]
for cfg in ("cfg2", "cfg3", "cfg4"):
    rep = os.path.join(out, f"{tag}_{cfg}_nodes.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(prof, f"{pre}_{cfg}_nodes_ncu.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, one launch of {d['Kernel Name'][0]}\n")
        for w in want:
            if w in d:
                f.write(f"{w} = {d[w][0]} {d[w][1]}\n")
        f.write("\n" + det)
    if cfg == "cfg2":
        rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6}[d["dram__bytes_read.sum"][1]]
        wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6}[d["dram__bytes_write.sum"][1]]
        lb = json.load(open(os.path.join(out, f"{tag}_cfg2_launch_bytes.json"))) if os.path.exists(
            os.path.join(out, f"{tag}_cfg2_launch_bytes.json")) else None
        step = lb["steps"][150] if lb else {}
        json.dump({"kernel": d["Kernel Name"][0], "launch": "node-block kernel launch 150 (configs[2] step 150)",
                   "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "algorithmic_bytes_same_launch": step.get("algorithmic_bytes"),
                   "layout_bytes_same_launch": step.get("layout_bytes"),
                   "note": "dram = ncu dram__bytes_read.sum + dram__bytes_write.sum of one capture; algorithmic = "
                           "SURVEY 8(d) 12 B/entry rule for that launch's iterations; layout = the node-block "
                           "layout's streamed bytes (vfpi_fem_layout_info: 72 B of values per 3x3 block, "
                           "block columns from the template, + row operands)",
                   "gpu_time_ms_under_ncu": float(d["gpu__time_duration.sum"][0].replace(",", "")),
                   "live_loop_ms_same_launch": step.get("loop_ms")},
                  open(os.path.join(prof, f"{pre}_cfg2_traffic.json"), "w"), indent=1)
print(open(os.path.join(prof, f"{pre}_cfg2_launches_summary.txt")).read()[:2500])
