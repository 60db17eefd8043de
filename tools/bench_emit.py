"""HBM throughput of the reduced-matrix API kernels (head_tail, reduce_cartesian,
reduce_join with keys): bytes read + written per call / device time."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2503_23385_b200 as P
from paper_2503_23385_b200 import datagen


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m, n = 20_000_000, 64
X = torch.empty((m, n), dtype=torch.float64, device="cuda"); datagen.uniform(5, m, n, out=X)
ms = timeit(lambda: P.head_tail(X))
print(f"head_tail {m}x{n}: {ms:.2f} ms, {2 * 8 * m * n / ms / 1e6:.0f} GB/s (read + write)")
A = torch.empty((m // 2, n), dtype=torch.float64, device="cuda"); datagen.uniform(6, m // 2, n, out=A)
B = torch.empty((m // 2, n), dtype=torch.float64, device="cuda"); datagen.uniform(7, m // 2, n, out=B)
ms = timeit(lambda: P.reduce_cartesian(A, B))
byt = 8 * (A.numel() + B.numel()) + 8 * (A.shape[0] + B.shape[0] - 1) * 2 * n
print(f"reduce_cartesian {m // 2}x{n} |x| {m // 2}x{n}: {ms:.2f} ms, {byt / ms / 1e6:.0f} GB/s (read + write)")
k = torch.arange(m // 2, device="cuda", dtype=torch.int64) // 100
ms = timeit(lambda: P.reduce_join(P.Table(A, k), P.Table(B, k)))
print(f"reduce_join 1e5 keys x 100: {ms:.2f} ms, {byt / ms / 1e6:.0f} GB/s (read + write, approx)")
