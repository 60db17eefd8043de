"""One keyed footnote figaro_r at a C3-like shape (Zipf keys), for profiling the N=32 leaf."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_23385_b200 as P
from paper_2503_23385_b200 import datagen
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
P.set_variant("footnote")
A = torch.empty((m, n), dtype=torch.float64, device="cuda"); B = torch.empty((m, n), dtype=torch.float64, device="cuda")
datagen.uniform(3001, m, n, out=A); datagen.uniform(3002, m, n, out=B)
ka = torch.from_numpy(datagen.zipf_sorted_keys(3003, m)).cuda(); kb = torch.from_numpy(datagen.zipf_sorted_keys(3004, m)).cuda()
for _ in range(2):
    P.figaro_r(P.Table(A, ka), P.Table(B, kb))
torch.cuda.synchronize()
print("ok")
