"""Figaro vs brute force on one B200 (the paper's Fig. 1/2 comparison):
time-to-R of figaro_r against join_r_bruteforce (TSQR over the join rows, generated
on the fly) for Cartesian products m x n |x| m x n, inputs resident in HBM, CUDA
events, mean of 3 after 1 warm-up.

python tools/figaro_vs_bruteforce.py > profiles/r01_figaro_vs_bruteforce.txt
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_23385_b200 as P
from paper_2503_23385_b200 import datagen


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


print("# figaro_r vs join_r_bruteforce, Cartesian m x n |x| m x n, f64, one B200")
print(f"{'m':>7} {'n':>4} {'join rows':>10} {'figaro ms':>10} {'brute ms':>10} {'speed-up':>9} {'brute TF/s':>10} {'rel Gram diff':>13}")
for m, n in [(100, 2), (1000, 2), (3000, 2), (10000, 2), (1000, 8), (3000, 8), (10000, 8),
             (1000, 32), (3000, 32), (1000, 64), (3000, 64)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((m, n), dtype=torch.float64, device="cuda")
    datagen.uniform(11, m, n, out=A)
    datagen.uniform(12, m, n, out=B)
    ta, tb = P.Table(A), P.Table(B)
    tf, rf = timed(lambda: P.figaro_r(ta, tb))
    tb_ms, rb = timed(lambda: P.join_r_bruteforce(ta, tb))
    rf, rb = rf.cpu().numpy(), rb.cpu().numpy()
    g = rb.T @ rb
    diff = np.linalg.norm(rf.T @ rf - g) / np.linalg.norm(g)
    rows, N = m * m, 2 * n
    tflops = (2.0 * rows * N * N) / (tb_ms / 1e3) / 1e12
    print(f"{m:7d} {n:4d} {rows:10.2e} {tf:10.3f} {tb_ms:10.3f} {tb_ms / tf:9.1f} {tflops:10.2f} {diff:13.2e}")
