"""Restatement of jq_split_group_rows (multi-GPU co-partition) for the
gloo orchestration tests.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Per group (parts contiguous, in shard order) with m1g = sum of the parts' A rows and
m2g of the B rows: the head row [sqrt(m2g) SA / sqrt(m1g) | sqrt(m1g) SB / sqrt(m2g)]
(the footnote head, PAPER.md:59 footnote) and per side one row per part k >= 1,
  v_k = scale sqrt(W m_k / (W + m_k)) (s_k / m_k - S / W),   scale = sqrt(m_other)
(W, S: rows and column sums of the parts before k) -- the pairwise update of the
centred Gram, which is what the carry-free part factors miss (SPEC.md:125-150 tails
restarted per part)."""
import numpy as np


def split_group_rows(part_sums, part_rows, part_group, n1, n2):
    sums = np.asarray(part_sums, dtype=np.float64)
    pr = np.asarray(part_rows, dtype=np.int64).reshape(-1, 2)
    pg = list(np.asarray(part_group).reshape(-1))
    n = n1 + n2
    out = []
    k = 0
    while k < len(pg):
        k1 = k
        while k1 < len(pg) and pg[k1] == pg[k]:
            k1 += 1
        m1g, m2g = float(pr[k:k1, 0].sum()), float(pr[k:k1, 1].sum())
        head = np.zeros(n)
        side_rows = []
        for side, cols, scale, mx in ((0, slice(0, n1), np.sqrt(m2g), m1g), (1, slice(n1, n), np.sqrt(m1g), m2g)):
            W, S = 0.0, np.zeros(cols.stop - cols.start)
            for j in range(k, k1):
                mk = float(pr[j, side])
                if mk <= 0:
                    continue
                sk = sums[j, cols]
                if W > 0:
                    row = np.zeros(n)
                    row[cols] = scale * np.sqrt(W * mk / (W + mk)) * (sk / mk - S / W)
                    side_rows.append(row)
                W += mk
                S = S + sk
            head[cols] = scale * S / np.sqrt(mx) if mx > 0 else 0.0
        out.append(head)
        out.extend(side_rows)
        k = k1
    return np.array(out).reshape(-1, n)
