"""Copy the judged profile summaries from gpurun_out/ (scratch) into profiles/:
launch list share table, ncu --set full details of the iteration kernel, its
DRAM traffic per launch (bench.py's roofline "traffic"), and the bench line.
usage: python scripts/summarize_profiles.py <round tag, e.g. r01>"""
import collections
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")

# launch list (gpu__time_duration.sum per launch, cold/serialised)
rows = list(csv.reader(open(os.path.join(out, "launches.csv"))))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"]
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += v
tot = sum(v[1] for v in agg.values())
with open(os.path.join(prof, f"{tag}_launches_summary.txt"), "w") as f:
    f.write("# ncu launch list summary (gpu__time_duration.sum, --clock-control none, cold/serialised)\n")
    f.write("# command: python bench.py --steps 2 --warmup 1 --no-cpu-baseline (scripts/gpu_round.sh)\n")
    f.write("launches    total_us  share  kernel\n")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{n:8d} {v:11.1f} {100 * v / tot:5.1f}%  {k[:100]}\n")

# ncu --set full details of the iteration kernel
rep = os.path.join(out, "prof_iter.ncu-rep")
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
with open(os.path.join(prof, f"{tag}_k_iterate_res_full.txt"), "w") as f:
    f.write(det)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units, vals = rr[0], rr[1], rr[2]
m = dict(zip(h, vals))
u = dict(zip(h, units))


def num(key):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(key, "byte"), 1)
    return float(m[key].replace(",", "")) * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
traffic = {
    "kernel": m.get("Kernel Name", "k_iterate_res"),
    "source": f"ncu --set full --clock-control none, profiles/{tag}_k_iterate_res_full.txt",
    "dram_bytes_read_per_launch": int(rd),
    "dram_bytes_write_per_launch": int(wr),
    "dram_bytes_per_launch": int(rd + wr),
    "duration_us": float(m["gpu__time_duration.sum"].replace(",", "")) * {
        "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(u.get("gpu__time_duration.sum"), 1.0),
    "note": "after the L2 flush the partition is read once from HBM into shared memory; the iterations then run "
            "from SMEM/L2",
}
json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
bl = [ln for ln in open(os.path.join(out, "bench_default.log")) if ln.startswith("{")]
if bl:
    open(os.path.join(prof, f"{tag}_bench_line.json"), "w").write(bl[-1])
print(open(os.path.join(prof, f"{tag}_launches_summary.txt")).read()[:1500])
print(json.dumps(traffic, indent=1))
