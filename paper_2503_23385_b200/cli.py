"""`joinqr` command line on the GPU backend (the reference's cli-bench module,
SPEC.md:487-547; console script `joinqr = "joinqr.cli:run"`, pyproject.toml:16).

  joinqr gen    --rows R --cols C --seed S [--key-groups K] --out t.csv
  joinqr qr     --left a.csv --right b.csv [--key-col k] [--has-header] [--method figaro|baseline] --out r.csv
  joinqr svd    --left a.csv --right b.csv [--key-col k] [--values-only | --with-v] --out s.csv
  joinqr verify --left a.csv --right b.csv [--key-col k] [--tol t]
  joinqr bench  --rows-list 100,200 --cols-list 4,8 [--repeats 4] [--target qr|svd]
                [--format csv|md] [--skip-baseline-above J] [--out report]

Exit codes: 0 success, 1 verification failure, 2 usage / IO errors.  `baseline`
is the GPU brute force (join_r_bruteforce: the join's own rows through the same
TSQR, never written); the bench reports it next to figaro_r the way the paper's
Figures 1-2 do (an absent baseline cell = above the join-size cutoff).  Timings
exclude file IO: device-synchronised wall clock, one warm-up, mean
of `repeats`.
"""

from __future__ import annotations

import argparse
import sys
import time
from typing import List, Optional

import numpy as np


class _Usage(Exception):
    pass


def _load_pair(args):
    from .tableio import read_table
    a = read_table(args.left, args.has_header, args.key_col)
    b = read_table(args.right, args.has_header, args.key_col)
    return a, b


def _baseline_r(a, b):
    from .bruteforce import join_r_bruteforce
    return join_r_bruteforce(a, b)


def cmd_gen(args) -> int:
    from .datagen import GenSpec, gen_uniform
    from .tableio import write_table
    if args.rows < 1 or args.cols < 1:
        raise _Usage("gen needs --rows >= 1 and --cols >= 1")
    if args.key_groups is not None and not 1 <= args.key_groups <= args.rows:
        raise _Usage("--key-groups must lie in 1..rows")
    write_table(gen_uniform(GenSpec(args.rows, args.cols, args.seed, args.key_groups)), args.out)
    return 0


def cmd_qr(args) -> int:
    from .qr import figaro_r
    from .tableio import write_matrix
    a, b = _load_pair(args)
    r = figaro_r(a, b) if args.method == "figaro" else _baseline_r(a, b)
    write_matrix(r, args.out)
    return 0


def cmd_svd(args) -> int:
    from .svd import figaro_svd
    from .tableio import write_svd
    a, b = _load_pair(args)
    res = figaro_svd(a, b, want_vectors=args.with_v)
    if args.with_v:
        v = np.asarray(res.right_vectors)
        if np.abs(v.T @ v - np.eye(v.shape[0])).max() > 1e-10:
            print("svd: V^T V check failed", file=sys.stderr)
            return 1
    write_svd(res, args.out, args.out + ".v.csv" if args.with_v else None)
    return 0


def cmd_verify(args) -> int:
    from .qr import figaro_r
    from .svd import svd_of_r
    a, b = _load_pair(args)
    rf = np.asarray(figaro_r(a, b))
    rb = np.asarray(_baseline_r(a, b))
    dr = float(np.abs(rf - rb).max()) if rf.size else 0.0
    sf = np.asarray(svd_of_r(rf).values)
    sb = np.asarray(svd_of_r(rb).values)
    ds = float((np.abs(sf - sb) / max(1.0, float(sb[0]) if sb.size else 1.0)).max()) if sb.size else 0.0
    print(f"max |R_figaro - R_baseline| = {dr:.3e}   max relative sigma difference = {ds:.3e}")
    return 0 if (dr <= args.tol and ds <= args.tol) else 1


def _ints(s: str) -> List[int]:
    try:
        v = [int(x) for x in s.split(",") if x.strip()]
    except ValueError:
        raise _Usage(f"not a comma-separated integer list: {s!r}") from None
    if not v or min(v) < 1:
        raise _Usage(f"list entries must be >= 1: {s!r}")
    return v


def _timed(f, repeats: int) -> float:
    import torch
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(repeats):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / repeats


def cmd_bench(args) -> int:
    import torch
    from . import datagen
    from .joins import Table
    from .qr import figaro_r
    from .svd import figaro_svd, svd_of_r
    rows_l, cols_l = _ints(args.rows_list), _ints(args.cols_list)
    if args.repeats < 1:
        raise _Usage("--repeats must be >= 1")
    cells = []
    for m in rows_l:
        for n in cols_l:
            A = torch.empty((m, n), dtype=torch.float64, device="cuda")
            B = torch.empty((m, n), dtype=torch.float64, device="cuda")
            datagen.uniform(1, m, n, out=A)
            datagen.uniform(2, m, n, out=B)
            ta, tb = Table(A), Table(B)
            if args.target == "qr":
                fig = lambda: figaro_r(ta, tb)
                base = lambda: _baseline_r(ta, tb)
            else:
                fig = lambda: figaro_svd(ta, tb)
                base = lambda: svd_of_r(_baseline_r(ta, tb))
            f_ms = _timed(fig, args.repeats)
            join_rows = m * m
            b_ms: Optional[float] = None
            if join_rows * 2 * n <= args.skip_baseline_above:
                b_ms = _timed(base, args.repeats)
            cells.append(dict(rows=m, cols=n, figaro_ms=f_ms, baseline_ms=b_ms,
                              speedup=(b_ms / f_ms) if b_ms is not None else None, repeats=args.repeats,
                              join_rows=join_rows, reduced_rows=2 * m - 1))
    fields = ["rows", "cols", "figaro_ms", "baseline_ms", "speedup", "repeats", "join_rows", "reduced_rows"]

    def cell(v):
        if v is None:
            return ""
        return f"{v:.4f}" if isinstance(v, float) else str(v)

    if args.format == "csv":
        text = ",".join(fields) + "\n" + "".join(",".join(cell(c[k]) for k in fields) + "\n" for c in cells)
    else:
        table = [fields] + [[cell(c[k]) for k in fields] for c in cells]
        w = [max(len(r[i]) for r in table) for i in range(len(fields))]
        line = lambda r: "| " + " | ".join(r[i].rjust(w[i]) for i in range(len(r))) + " |"
        text = "\n".join([line(table[0]), "|" + "|".join("-" * (x + 2) for x in w) + "|"] +
                         [line(r) for r in table[1:]]) + "\n"
    if args.out:
        with open(args.out, "w", encoding="utf-8") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="joinqr", description="Figaro QR / SVD of two-table joins on a B200")
    p.add_argument("--threads", type=int, default=None, help="accepted for compatibility (GPU build)")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen")
    g.add_argument("--rows", type=int, required=True)
    g.add_argument("--cols", type=int, required=True)
    g.add_argument("--seed", type=int, required=True)
    g.add_argument("--key-groups", type=int, default=None)
    g.add_argument("--out", required=True)
    g.set_defaults(func=cmd_gen)

    def pair(sp):
        sp.add_argument("--left", required=True)
        sp.add_argument("--right", required=True)
        sp.add_argument("--key-col", type=int, default=None)
        sp.add_argument("--has-header", action="store_true")

    q = sub.add_parser("qr")
    pair(q)
    q.add_argument("--method", choices=["figaro", "baseline"], default="figaro")
    q.add_argument("--out", required=True)
    q.set_defaults(func=cmd_qr)
    s = sub.add_parser("svd")
    pair(s)
    mode = s.add_mutually_exclusive_group()
    mode.add_argument("--values-only", action="store_true")
    mode.add_argument("--with-v", action="store_true")
    s.add_argument("--out", required=True)
    s.set_defaults(func=cmd_svd)
    v = sub.add_parser("verify")
    pair(v)
    v.add_argument("--tol", type=float, default=1e-8)
    v.set_defaults(func=cmd_verify)
    b = sub.add_parser("bench")
    b.add_argument("--rows-list", required=True)
    b.add_argument("--cols-list", required=True)
    b.add_argument("--repeats", type=int, default=4)
    b.add_argument("--target", choices=["qr", "svd"], default="qr")
    b.add_argument("--format", choices=["csv", "md"], default="md")
    b.add_argument("--skip-baseline-above", type=float, default=2e8)
    b.add_argument("--out", default=None)
    b.set_defaults(func=cmd_bench)
    return p


def run(argv: Optional[List[str]] = None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:  # argparse: usage errors exit 2, --help exits 0
        return int(e.code or 0)
    try:
        return args.func(args)
    except _Usage as e:
        print(f"joinqr {args.cmd}: {e}", file=sys.stderr)
        return 2
    except (OSError, ValueError) as e:
        print(f"joinqr {args.cmd}: {e}", file=sys.stderr)
        return 2


def main() -> None:
    sys.exit(run())


if __name__ == "__main__":
    main()
