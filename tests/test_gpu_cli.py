"""`joinqr` CLI end to end on the GPU: gen -> qr (figaro and
baseline) -> svd -> verify, and the bench report shape / baseline cutoff."""

import numpy as np
import pytest

from paper_2503_23385_b200 import tableio
from paper_2503_23385_b200.cli import run

pytestmark = pytest.mark.gpu


def test_cli_fixture_qr_svd_verify(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    a.write_text("1\n2\n")
    b.write_text("3\n4\n")
    for method in ("figaro", "baseline"):
        out = tmp_path / f"r_{method}.csv"
        assert run(["qr", "--left", str(a), "--right", str(b), "--method", method, "--out", str(out)]) == 0
        r = tableio.read_matrix(str(out))
        assert np.abs(r - [[3.162278, 6.640783], [0, 2.428992]]).max() < 1e-6
    s = tmp_path / "s.csv"
    assert run(["svd", "--left", str(a), "--right", str(b), "--with-v", "--out", str(s)]) == 0
    vals = tableio.read_matrix(str(s)).ravel()
    assert np.abs(vals - [7.681146, 1.0]).max() < 1e-6
    v = tableio.read_matrix(str(s) + ".v.csv")
    assert np.abs(v.T @ v - np.eye(2)).max() < 1e-10
    assert run(["verify", "--left", str(a), "--right", str(b), "--tol", "1e-8"]) == 0


def test_cli_gen_keyed_join_verify(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert run(["gen", "--rows", "300", "--cols", "3", "--seed", "1", "--key-groups", "7", "--out", str(a)]) == 0
    assert run(["gen", "--rows", "200", "--cols", "4", "--seed", "2", "--key-groups", "7", "--out", str(b)]) == 0
    t = tableio.read_table(str(a), key_col=0)
    assert t.data.shape == (300, 3) and np.all((t.data > 0) & (t.data < 1))
    assert run(["verify", "--left", str(a), "--right", str(b), "--key-col", "0", "--tol", "1e-8"]) == 0
    assert run(["verify", "--left", str(a), "--right", str(b), "--key-col", "0", "--tol", "0"]) in (0, 1)


def test_cli_bench_report(tmp_path):
    out = tmp_path / "bench.csv"
    assert run(["bench", "--rows-list", "100,200", "--cols-list", "4,8", "--repeats", "2", "--format", "csv",
                "--skip-baseline-above", "1e6", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "rows,cols,figaro_ms,baseline_ms,speedup,repeats,join_rows,reduced_rows"
    cells = [l.split(",") for l in lines[1:]]
    assert len(cells) == 4
    for c in cells:
        rows, cols = int(c[0]), int(c[1])
        assert float(c[2]) > 0 and int(c[6]) == rows * rows and int(c[7]) == 2 * rows - 1
        if rows * rows * 2 * cols <= 1e6:
            assert float(c[3]) > 0 and float(c[4]) > 0
        else:
            assert c[3] == "" and c[4] == ""                 # baseline cell absent above the cutoff
    md = tmp_path / "bench.md"
    assert run(["bench", "--rows-list", "100", "--cols-list", "4", "--repeats", "1", "--target", "svd",
                "--format", "md", "--out", str(md)]) == 0
    assert md.read_text().startswith("| ")
