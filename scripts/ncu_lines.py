"""Per-source-line warp-stall summary of an ncu report (tuning aid).
usage: python scripts/ncu_lines.py report.ncu-rep [file-substring] [top] [metric]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else "vfpi_resident.cu"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
metric = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
hdr = None
lines = []
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "" or row[0] == "Function Name":
        continue
    if want not in (cur or ""):
        continue
    d = dict(zip(hdr[2:], row[2:]))
    try:
        smp = float(d.get(metric, 0) or 0)
    except ValueError:
        continue
    reasons = {k: float(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
               and v not in ("", "-")}
    lines.append((smp, int(row[0]), row[1].strip()[:70], sorted(reasons.items(), key=lambda x: -x[1])[:3]))
tot = sum(x[0] for x in lines) or 1
for smp, ln, src, rs in sorted(lines, reverse=True)[:top]:
    print(f"{ln:5d} {smp / tot * 100:5.1f}% {smp:12.0f}  {src:70s} "
          + " ".join(f"{k[6:]}={v / tot * 100:.1f}" for k, v in rs))
