import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_23385_b200 as P
rng = np.random.default_rng(0)
step = sys.argv[1]
if step == 'hh':
    for rows, cols in [(7,3),(64,16),(1000,31),(3000,128),(1500,256)]:
        r = P.householder_r(rng.random((rows, cols))); print('hh', rows, cols, 'ok', flush=True)
elif step == 'fig':
    for m, n in [(2,1),(1000,4),(4000,32),(2500,64)]:
        r = P.figaro_r(P.Table(rng.random((m, n))), P.Table(rng.random((m+3, n)))); print('fig', m, n, 'ok', flush=True)
