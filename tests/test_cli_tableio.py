"""CSV data-io and the `joinqr` command line:
host-side parsing, round trips and the usage / IO exit codes (no GPU needed)."""

import os

import numpy as np
import pytest

from paper_2503_23385_b200 import tableio
from paper_2503_23385_b200.cli import run


def test_read_spec_example_and_round_trip(tmp_path):
    p = tmp_path / "m.csv"
    p.write_text("1.5,2.0\n3.0,4.0\n")
    t = tableio.read_table(str(p))
    assert np.array_equal(t.data, [[1.5, 2.0], [3.0, 4.0]]) and t.keys is None
    rng = np.random.default_rng(1)
    m = rng.random((7, 3)) * 10.0 ** rng.integers(-5, 5, (7, 3))
    q = tmp_path / "r.csv"
    tableio.write_matrix(m, str(q))
    assert np.array_equal(tableio.read_matrix(str(q)), m)        # exact round trip (repr)
    first = q.read_text()
    tableio.write_matrix(tableio.read_matrix(str(q)), str(q))
    assert q.read_text() == first                                   # byte-equivalent


def test_keys_header_and_errors(tmp_path):
    p = tmp_path / "k.csv"
    p.write_text("key,x,y\n1,0.5,0.25\n1,1.5,2.5\n3,4.0,5.0\n")
    t = tableio.read_table(str(p), has_header=True, key_col=0)
    assert t.keys.tolist() == [1, 1, 3] and np.array_equal(t.data, [[0.5, 0.25], [1.5, 2.5], [4.0, 5.0]])
    out = tmp_path / "t.csv"
    tableio.write_table(t, str(out))
    t2 = tableio.read_table(str(out), key_col=0)
    assert np.array_equal(t2.data, t.data) and t2.keys.tolist() == [1, 1, 3]
    (tmp_path / "rag.csv").write_text("1,2\n3\n")
    with pytest.raises(ValueError, match=":2"):
        tableio.read_table(str(tmp_path / "rag.csv"))            # ragged row names its line
    (tmp_path / "bad.csv").write_text("1,x\n")
    with pytest.raises(ValueError, match="column 1"):
        tableio.read_table(str(tmp_path / "bad.csv"))
    (tmp_path / "uns.csv").write_text("2,1.0\n1,2.0\n")
    with pytest.raises(ValueError):
        tableio.read_table(str(tmp_path / "uns.csv"), key_col=0)   # unsorted keys


def test_cli_usage_and_io_exit_codes(tmp_path):
    assert run([]) == 2
    assert run(["gen", "--rows", "0", "--cols", "2", "--seed", "1", "--out", str(tmp_path / "g.csv")]) == 2
    assert run(["bench", "--rows-list", "a,b", "--cols-list", "4"]) == 2
    missing = str(tmp_path / "nope.csv")
    assert run(["qr", "--left", missing, "--right", missing, "--out", str(tmp_path / "r.csv")]) == 2
    assert run(["verify", "--left", missing, "--right", missing]) == 2
    assert run(["svd", "--left", missing, "--right", missing, "--values-only", "--with-v",
                "--out", "x"]) == 2                                     # mutually exclusive flags


def test_native_csv_edge_cases(tmp_path):
    p = tmp_path / "e.csv"
    p.write_text("h1,h2\r\n\r\n 1.5 , +2.0\r\n\n3e-3,-4\r\n")     # CRLF, blank lines, spaces, signs
    t = tableio.read_table(str(p), has_header=True)
    assert np.array_equal(t.data, [[1.5, 2.0], [3e-3, -4.0]])
    (tmp_path / "empty.csv").write_text("")
    assert tableio.read_table(str(tmp_path / "empty.csv")).data.shape[0] == 0
    (tmp_path / "inf.csv").write_text("1,2\n3,inf\n")
    with pytest.raises(ValueError, match=":2: non-finite"):
        tableio.read_table(str(tmp_path / "inf.csv"))
    (tmp_path / "wide.csv").write_text("1,2\n3,4,5\n")
    with pytest.raises(ValueError, match=":2: ragged"):
        tableio.read_table(str(tmp_path / "wide.csv"))
    with pytest.raises(ValueError):
        tableio.read_table(str(tmp_path / "nope.csv"))


def test_native_csv_multi_chunk_round_trip_and_line_numbers(tmp_path):
    """> 4 MB files are parsed by several threads in newline-aligned chunks: values,
    keys and error line numbers must not depend on the chunking."""
    rng = np.random.default_rng(2)
    m = 120_000
    keys = np.sort(rng.integers(-50, 5000, m))
    data = rng.random((m, 4)) * 10.0 ** rng.integers(-8, 8, (m, 4))
    p = tmp_path / "big.csv"
    tableio.write_table(tableio.Table(data, keys), str(p))
    assert p.stat().st_size > (8 << 20)
    t = tableio.read_table(str(p), key_col=0)
    assert np.array_equal(t.data, data) and np.array_equal(t.keys, keys)
    lines = p.read_text().splitlines()
    bad = 100_001
    lines[bad - 1] = lines[bad - 1].replace(",", ",x", 1)
    q = tmp_path / "bad.csv"
    q.write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError, match=f":{bad}: cannot parse"):
        tableio.read_table(str(q), key_col=0)
    lines = p.read_text().splitlines()
    lines[bad - 1] = "-100," + lines[bad - 1].split(",", 1)[1]   # unsorted key deep in the file
    q.write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError, match=f":{bad}: keys are not sorted"):
        tableio.read_table(str(q), key_col=0)
