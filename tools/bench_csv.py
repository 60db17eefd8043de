"""CSV ingest throughput: native host parse vs parse straight into HBM (tableio.read_table)."""
import os, sys, time, tempfile
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_23385_b200 as P
from paper_2503_23385_b200 import tableio
m, n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000, int(sys.argv[2]) if len(sys.argv) > 2 else 16
rng = np.random.default_rng(0)
keys = np.sort(rng.integers(0, m // 100, m))
data = rng.random((m, n))
d = tempfile.mkdtemp()
p = os.path.join(d, "t.csv")
t0 = time.perf_counter(); tableio.write_table(P.Table(data, keys), p); tw = time.perf_counter() - t0
size = os.path.getsize(p)
for dev in (None, "cuda"):
    tableio.read_table(p, key_col=0, device=dev)
    t0 = time.perf_counter()
    t = tableio.read_table(p, key_col=0, device=dev)
    if dev:
        import torch; torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"read_table device={dev}: {m} rows x {n + 1} cells, {size / 1e6:.0f} MB in {dt * 1e3:.0f} ms = "
          f"{size / dt / 1e9:.2f} GB/s of text, {m * n / dt / 1e6:.0f} M values/s (threads {os.cpu_count()})")
print(f"(write_table python: {tw:.1f} s)")
