"""Large-configuration oracle: factorised Gram of the join + Cholesky.

J^T J = [[sum_g m2g A_g^T A_g,          sum_g (1^T A_g)^T (1^T B_g)],
         [   (sym)          ,           sum_g m1g B_g^T B_g        ]]
computed in O(m1 n1^2 + m2 n2^2) without touching the join; R_oracle =
chol(J^T J)^T (positive diagonal = canonical R for a full-rank join, SPEC.md:289,
PAPER.md "constitutes a Cholesky decomposition"), sigma_oracle = sqrt(eig(J^T J)).
Accuracy ~ kappa(J)^2 * eps, ample for uniform(0,1) data at the 1e-10 bar.
Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from .joins import Table, group_keys


def factorised_gram(a: Table, b: Table) -> np.ndarray:
    n1, n2 = a.data.shape[1], b.data.shape[1]
    g = np.zeros((n1 + n2, n1 + n2))
    if a.keys is None:
        groups = [(0, a.data.shape[0], 0, b.data.shape[0])]
    else:
        _, a_s, a_c, b_s, b_c, _ = group_keys(a.keys, b.keys)
        groups = list(zip(a_s, a_c, b_s, b_c))
    if len(groups) > 64 and a.keys is not None:
        # vectorised per-group sums: weights m2g on A rows, m1g on B rows
        _, a_s, a_c, b_s, b_c, _ = group_keys(a.keys, b.keys)
        wa = np.zeros(a.data.shape[0]); wb = np.zeros(b.data.shape[0])
        ga = np.full(a.data.shape[0], -1); gb = np.full(b.data.shape[0], -1)
        for gi, (s, c) in enumerate(zip(a_s, a_c)):
            ga[s:s + c] = gi
        for gi, (s, c) in enumerate(zip(b_s, b_c)):
            gb[s:s + c] = gi
        ma, mb = ga >= 0, gb >= 0
        wa[ma] = b_c[ga[ma]]
        wb[mb] = a_c[gb[mb]]
        g[:n1, :n1] = (a.data * wa[:, None]).T @ a.data
        g[n1:, n1:] = (b.data * wb[:, None]).T @ b.data
        sa = np.zeros((len(a_s), n1)); sb = np.zeros((len(b_s), n2))
        np.add.at(sa, ga[ma], a.data[ma])
        np.add.at(sb, gb[mb], b.data[mb])
        g[:n1, n1:] = sa.T @ sb
    else:
        for s1, c1, s2, c2 in groups:
            ag = a.data[s1:s1 + c1]
            bg = b.data[s2:s2 + c2]
            g[:n1, :n1] += c2 * (ag.T @ ag)
            g[n1:, n1:] += c1 * (bg.T @ bg)
            g[:n1, n1:] += np.outer(ag.sum(axis=0), bg.sum(axis=0))
    g[n1:, :n1] = g[:n1, n1:].T
    return g


def gram_r(g: np.ndarray) -> np.ndarray:
    """Canonical (positive-diagonal) R with R^T R = g."""
    return np.linalg.cholesky(g).T


def gram_sigma(g: np.ndarray) -> np.ndarray:
    w = np.linalg.eigvalsh(g)
    return np.sqrt(np.clip(w, 0.0, None))[::-1]
