"""bench.py keeps the driver's contract: the reference arm (CPU, the oracle port) prints
ONE JSON line with the keys the driver reads.  Runs on CPU (config 1, a few ms)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("port", "reference")


def test_bench_defines_gpu_arm():
    src = open(os.path.join(ROOT, "bench.py")).read()
    compile(src, "bench.py", "exec")
    for name in ("def main", "def run_e2e", "def run_e2e_sharded", "roofline", "cpu_baseline", "gpu_launches"):
        assert name in src, name
