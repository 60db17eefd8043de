import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_23385_b200 as P, oracle as O
P.set_variant(sys.argv[1] if len(sys.argv) > 1 else "footnote")
rng = np.random.default_rng(1)
for m, n in [(300, 33), (300, 64), (2500, 20), (2500, 40), (2500, 64), (200, 64), (129, 64), (128, 64)]:
    A, B = rng.random((m, n)), rng.random((m + 5, n))
    r = np.asarray(P.figaro_r(P.Table(A), P.Table(B)))
    ref = O.figaro_r(O.Table(A), O.Table(B), lapack=True)
    print(m, n, 'nan' if np.isnan(r).any() else f'{np.linalg.norm(np.abs(r)-np.abs(ref))/np.linalg.norm(ref):.2e}', flush=True)
