"""Time svd_of_r on an n x n upper-triangular R (CUDA events) -- A/B of the Jacobi kernels.

JQ_SVD_IMPL=coop python tools/svd_probe.py --n 256
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_23385_b200 import svd
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--vectors", type=int, default=1)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand((4 * a.n, a.n), dtype=torch.float64, device="cuda", generator=g)
r = torch.linalg.qr(x, mode="r")[1].contiguous()
for _ in range(2):
    res = svd.svd_of_r(r, want_vectors=bool(a.vectors))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    res = svd.svd_of_r(r, want_vectors=bool(a.vectors))
e1.record()
torch.cuda.synchronize()
ref = torch.linalg.svdvals(r)
err = ((res.values if hasattr(res, "values") else res[0]) - ref).abs().max().item() / ref[0].item()
print(f"n={a.n} impl={os.environ.get('JQ_SVD_IMPL', 'default')} ms={e0.elapsed_time(e1) / a.reps:.3f} max_rel_err={err:.2e}")
