"""Timeline of tsqr_ws2_kernel (CTA 0: chain warp, data warp 0, loader) and Gram-panel rejections (lib/libjoinqr_ktime.so: make -C csrc ktime).

JOINQR_LIB=.../libjoinqr_ktime.so python tools/ktime_ws.py --m 2000000 --n 64 [--variant footnote]
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
ap.add_argument("--variant", default="footnote")
ap.add_argument("--keys", default=None, choices=[None, "zipf"])
a = ap.parse_args()
P.set_variant(a.variant)
A = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
B = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
datagen.uniform(1, a.m, a.n, out=A); datagen.uniform(2, a.m, a.n, out=B)
ka = kb = None
if a.keys == "zipf":
    ka = torch.from_numpy(datagen.zipf_sorted_keys(3003, a.m)).cuda()
    kb = torch.from_numpy(datagen.zipf_sorted_keys(3004, a.m)).cuda()
P.figaro_r(P.Table(A, ka), P.Table(B, kb))
t = N.last_timing()
print(f"variant={a.variant} tsqr_ms={t['tsqr_ms']:.2f} ctas={t['tsqr_ctas']}")
ff = N.lib().jq_debug_gram_fail; ff.argtypes = [ctypes.c_void_p, ctypes.c_int]
fb = (ctypes.c_ulonglong * 16)()
ff(fb, 1)
print("Gram panels rejected (explicit fallback):", fb[0])
tf = N.lib().jq_debug_trace; tf.argtypes = [ctypes.c_void_p, ctypes.c_int]; tf.restype = ctypes.c_int
tb = (ctypes.c_longlong * 4096)()
tf(tb, 1)
P.figaro_r(P.Table(A, ka), P.Table(B, kb))
torch.cuda.synchronize()
tf(tb, 1)
ev = sorted([(tb[w * 1365 + 2 * k + 1], w, tb[w * 1365 + 2 * k]) for w in (0, 1, 2) for k in range(600)
             if tb[w * 1365 + 2 * k + 1] != 0])
evnames = {(0, 1): "chain start", (0, 2): "chain done", (0, 3): "chain B pass", (0, 4): "chain VREADY",
           (0, 5): "chain Gnext", (1, 1): "d0 V ok", (1, 2): "d0 reduce done", (1, 3): "d0 BAR_DATA pass",
           (1, 4): "d0 applies done", (1, 5): "d0 step4 done", (1, 6): "d0 B pass", (1, 7): "d0 wait READY / load start",
           (1, 8): "d0 READY ok / load done",
           (1, 15): "d0 load: coefs", (1, 17): "d0 load: loads issued + barrier", (1, 18): "d0 load: scan", (1, 19): "d0 load: carry-ins", (2, 1): "loader FREE ok", (2, 2): "loader TMA done", (2, 3): "loader prep done",
           (2, 4): "loader BAR raw", (2, 5): "loader coeffs done", (2, 6): "loader pass1 done", (2, 7): "loader BAR seg"}
t0 = ev[0][0] if ev else 0
prev = t0
for ts, who, e in ev[:int(os.environ.get('KT_N', '160'))]:
    print(f"{ts - t0:9d} +{ts - prev:6d}  {evnames.get((who, e), (who, e))}")
    prev = ts
