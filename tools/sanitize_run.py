"""Small C1/C2-shaped calls of every kernel family of libjoinqr.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck): tools/sanitize.sh.

Host numpy inputs only (no torch kernels in the process, so every report is ours).
Each call's result is checked loosely (finite, right shape) -- parity is the job of
tests/; this script exists to drive the kernels under the sanitizer.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_23385_b200 as P  # noqa: E402
from paper_2503_23385_b200 import _native as N  # noqa: E402
from paper_2503_23385_b200 import datagen  # noqa: E402


def ok(name, x):
    x = np.asarray(x)
    assert np.all(np.isfinite(x)), name
    print(f"  {name}: {x.shape}", flush=True)


def main(which):
    rng = np.random.default_rng(0)
    N.set_device(0)
    fams = which.split(",")
    if "gen" in fams or "all" in fams:
        ok("gen_uniform", datagen.uniform(11, 3000, 7))
        ok("zipf_keys", datagen.zipf_sorted_keys(12, 5000, universe=1000))
    if "group" in fams or "all" in fams:
        ka, kb = np.sort(rng.integers(0, 40, 3000)), np.sort(rng.integers(10, 60, 2000))
        g = P.group_keys(ka, kb)
        ok("group_keys", g[0])
        try:
            P.group_keys(ka[::-1].copy(), kb)
        except ValueError:
            print("  unsorted keys -> ValueError", flush=True)
    if "headtail" in fams or "all" in fams:
        ok("head_tail", P.head_tail(rng.random((3000, 9))))
        ok("reduce_cartesian", P.reduce_cartesian(rng.random((1000, 4)), rng.random((1000, 4))).matrix)
        ka, kb = np.sort(rng.integers(0, 30, 2000)), np.sort(rng.integers(0, 30, 1500))
        ok("reduce_natural_join",
           P.reduce_natural_join(P.Table(rng.random((2000, 5)), ka), P.Table(rng.random((1500, 6)), kb)).matrix)
    if "qr" in fams or "all" in fams:
        for cols in (8, 40, 100, 200):
            ok(f"householder_r n={cols}", P.householder_r(rng.random((5000, cols))))
        for variant in ("dense", "footnote"):
            P.set_variant(variant)
            a, b = rng.random((1000, 4)), rng.random((1000, 4))
            ok(f"figaro_r C1 {variant}", P.figaro_r(P.Table(a), P.Table(b)))
            ka = np.repeat(np.arange(100), 100)
            a, b = rng.random((10000, 16)), rng.random((10000, 16))
            ok(f"figaro_r C2-shaped {variant}", P.figaro_r(P.Table(a, ka), P.Table(b, ka)))
            a, b = rng.random((20000, 64)), rng.random((20000, 64))
            ok(f"figaro_r n=64+64 {variant}", P.figaro_r(P.Table(a), P.Table(b)))
        P.set_variant("auto")
    if "stream" in fams or "all" in fams:
        os.environ["JQ_STREAM_MIN_BYTES"] = "1"
        os.environ["JQ_PIECE_BYTES"] = str(8 * 16 * 1024)
        for variant in ("dense", "footnote"):
            P.set_variant(variant)
            ok(f"figaro_r streamed {variant}", P.figaro_r(P.Table(rng.random((3500, 16))),
                                                        P.Table(rng.random((2100, 16)))))
        del os.environ["JQ_STREAM_MIN_BYTES"], os.environ["JQ_PIECE_BYTES"]
        P.set_variant("auto")
    if "svd" in fams or "all" in fams:
        for n in (6, 40, 130):
            r = np.triu(rng.random((n, n))) + np.eye(n)
            s = P.svd_of_r(r, True)
            ok(f"svd_of_r n={n}", s.right_vectors)
        s = P.figaro_svd(P.Table(rng.random((2000, 20))), P.Table(rng.random((2000, 20))), want_vectors=True)
        ok("figaro_svd", s.values)
    if "brute" in fams or "all" in fams:
        ka = np.sort(rng.integers(0, 10, 300))
        ok("materialize_natural_join", P.materialize_natural_join(P.Table(rng.random((300, 3)), ka),
                                                                  P.Table(rng.random((300, 2)), ka)))
        ok("join_r_bruteforce", P.join_r_bruteforce(P.Table(rng.random((200, 3))), P.Table(rng.random((150, 4)))))
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
