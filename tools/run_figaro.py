"""Run figaro_r / figaro_svd once on device-resident synthetic data (profiling helper).

python tools/run_figaro.py --m 2000000 --n 64 [--keys groups|zipf] [--svd] [--reps 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_23385_b200 as P  # noqa: E402
from paper_2503_23385_b200 import _native as N, datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--keys", default=None)
ap.add_argument("--svd", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--all", action="store_true", help="print min tsqr/total ms over the reps after the first")
a = ap.parse_args()
A = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
B = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
datagen.uniform(4001, a.m, a.n, out=A)
datagen.uniform(4002, a.m, a.n, out=B)
ka = kb = None
if a.keys == "groups":
    ka = torch.from_numpy(datagen.near_equal_keys(a.m, max(1, a.m // 100))).cuda()
    kb = ka.clone()
elif a.keys == "zipf":
    ka = torch.from_numpy(datagen.zipf_sorted_keys(3003, a.m)).cuda()
    kb = torch.from_numpy(datagen.zipf_sorted_keys(3004, a.m)).cuda()
tims = []
for _ in range(a.reps):
    if a.svd:
        P.figaro_svd(P.Table(A, ka), P.Table(B, kb), want_vectors=True)
    else:
        P.figaro_r(P.Table(A, ka), P.Table(B, kb))
    tims.append(N.last_timing())
torch.cuda.synchronize()
if a.all:
    rest = tims[1:] or tims
    print(f"tsqr_ms min {min(t['tsqr_ms'] for t in rest):.3f} total_ms min {min(t['total_ms'] for t in rest):.3f} "
          f"ctas {tims[-1]['tsqr_ctas']}")
else:
    print("timing", N.last_timing())
