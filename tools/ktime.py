"""Per-warp phase breakdown of tsqr_kernel (needs lib/libjoinqr_ktime.so: make -C csrc ktime).

JOINQR_LIB=.../libjoinqr_ktime.so python tools/ktime.py --m 2000000 --n 64 [--variant footnote]
"""
import argparse, ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2503_23385_b200 as P
from paper_2503_23385_b200 import _native as N, datagen
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--variant", default="dense")
a = ap.parse_args()
P.set_variant(a.variant)
A = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
B = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
datagen.uniform(1, a.m, a.n, out=A); datagen.uniform(2, a.m, a.n, out=B)
P.figaro_r(P.Table(A), P.Table(B))
lib = N.lib(); fn = lib.jq_debug_ktime; fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
fn(buf, 1)
P.figaro_r(P.Table(A), P.Table(B))
torch.cuda.synchronize()
fn(buf, 1)
ctas = buf[15]
t = N.last_timing()
names = ["load: TMA wait", "Gram/Z partials + sync", "panel chain + sync", "W tiles + apply", "chunk-end barrier", "load: prep", "load: registers / direct: transform", "direct: coefs + issue", "direct: loads + scan", "direct: carry-ins"]
tot = sum(buf[i] for i in range(10))
print(f"variant={a.variant} ctas(launches incl. tree)={ctas} tsqr_ms={t['tsqr_ms']:.2f}")
for i, nm in enumerate(names):
    print(f"  {nm:34s} {buf[i] / tot:6.1%}  {buf[i] / 1e6:12.1f} Mcycles (sum over warps)")
