"""CSV ingest straight into HBM (jq_csv_parse with device outputs: pinned staging
slots, H2D overlapped with the parse) equals the host parse bit for bit, and feeds
figaro_r directly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_csv_to_device_matches_host(tmp_path):
    import torch
    import paper_2503_23385_b200 as P
    from paper_2503_23385_b200 import tableio
    rng = np.random.default_rng(3)
    m = 400_000
    keys = np.sort(rng.integers(0, 2000, m))
    data = rng.random((m, 6))
    p = tmp_path / "t.csv"
    tableio.write_table(P.Table(data, keys), str(p))
    th = tableio.read_table(str(p), key_col=0)
    td = tableio.read_table(str(p), key_col=0, device="cuda")
    assert td.data.is_cuda and td.keys.is_cuda
    assert np.array_equal(td.data.cpu().numpy(), th.data) and np.array_equal(td.keys.cpu().numpy(), th.keys)
    assert np.array_equal(th.data, data)
    r_dev = P.figaro_r(td, td).cpu().numpy()
    r_host = np.asarray(P.figaro_r(th, th))
    assert np.linalg.norm(r_dev - r_host) <= 1e-12 * np.linalg.norm(r_host)
    (tmp_path / "bad.csv").write_text("1,2\n3,x\n")
    with pytest.raises(ValueError, match=":2"):
        tableio.read_table(str(tmp_path / "bad.csv"), device="cuda")
