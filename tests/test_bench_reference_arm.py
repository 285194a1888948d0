"""bench.py's CPU-side contracts: the reference arm keeps the driver's JSON
line and runs without a GPU; ``--gpus N`` outside torchrun launches N ranks,
each bound to its own device with its own contiguous scene block."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "contact-iter/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    assert d["config"]["workload"].startswith("configs[2]")
    assert d["higher_is_better"] is True and d["scaling"] == "strong"


def test_gpus_2_launches_two_ranks_on_distinct_devices():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "VFPI_DEVICE")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and len(d["ranks"]) == 2
    r0, r1 = sorted(d["ranks"], key=lambda r: r["rank"])
    assert (r0["device"], r1["device"]) == (0, 1)
    assert (r0["local_rank"], r1["local_rank"]) == (0, 1)
    assert r0["pid"] != r1["pid"]
    assert r0["scenes"] == [0, 512] and r1["scenes"] == [512, 1024]
