"""History / sweep / Matrix Market formats: byte-compatible
with the reference's writers (fixtures from the unmodified reference)."""

import io

import numpy as np
import pytest

from conftest import golden
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import cli, harness, mmio
from paper_1706_05988_b200.solvers import IterationRecord


@pytest.fixture(scope="module")
def gold():
    return golden("formats")


def records(h):
    opt = lambda v: None if np.isnan(v) else float(v)
    return [IterationRecord(int(r[0]), *map(float, r[1:6]), rnorm_true=opt(r[6]), gap_f=opt(r[7]),
                            gap_g=opt(r[8]), gap_h=opt(r[9]), gap_j=opt(r[10])) for r in h]


@pytest.mark.parametrize("tag", ["gaps", "plain"])
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_emit_history_bytes(gold, tag, fmt):
    recs = records(gold[f"{tag}_hist"])
    sink = io.StringIO()
    harness.emit_history(recs, fmt, sink)
    assert sink.getvalue().encode("ascii") == gold[f"{tag}_{fmt}"].tobytes()
    back = harness.load_history(io.StringIO(sink.getvalue()))
    assert [(r.iter, r.alpha, r.gap_f, r.rnorm_true) for r in back] == \
           [(r.iter, r.alpha, r.gap_f, r.rnorm_true) for r in recs]


@pytest.mark.parametrize("tag", ["lap5x4", "rspd6"])
def test_matrix_market_bytes_and_roundtrip(gold, tag, tmp_path):
    g = gold
    A = K.SparseMatrix(int(g[f"mmA_{tag}_n"]), g[f"mmA_{tag}_row_ptr"], g[f"mmA_{tag}_col_idx"],
                       g[f"mmA_{tag}_values"])
    sink = io.BytesIO()
    mmio.write_matrix_market(A, sink)
    assert sink.getvalue() == g[f"mm_{tag}"].tobytes()
    B = mmio.read_matrix_market(sink.getvalue())
    assert np.array_equal(B.row_ptr, A.row_ptr) and np.array_equal(B.col_idx, A.col_idx)
    assert B.values.tobytes() == A.values.tobytes()
    import gzip
    path = tmp_path / "m.mtx.gz"
    path.write_bytes(gzip.compress(sink.getvalue()))
    assert mmio.read_matrix_market(path).values.tobytes() == A.values.tobytes()


def test_matrix_market_errors():
    with pytest.raises(mmio.MatrixMarketError):
        mmio.read_matrix_market(b"%%MatrixMarket matrix array real general\n2 2\n")
    with pytest.raises(mmio.MatrixMarketError):
        mmio.read_matrix_market(b"%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n")
    with pytest.raises(mmio.MatrixMarketError):
        mmio.read_matrix_market(b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n")


def test_run_configs_and_sources():
    with pytest.raises(ValueError):
        harness.RunConfig("lapl:4x4", rhs_mode="bad")
    with pytest.raises(ValueError):
        harness.load_matrix("lapl:4")
    assert harness.load_matrix("lapl:4x3").n == 12
    assert harness.load_matrix("stencil3:4x3x2").n == 24
    assert np.array_equal(harness.parse_sigma_grid("0:0.5:2"), [0.0, 0.5, 1.0, 1.5, 2.0])


def test_analyze_shift_from_history_file(gold, tmp_path):
    recs = records(gold["plain_hist"])
    h = tmp_path / "h.csv"
    harness.emit_history(recs, "csv", h)
    out = tmp_path / "sweep.csv"
    sw = harness.run_analyze_shift(h, 500, "0:0.5:2", output=out)
    assert sw.iter == 25                                    # truncated to the records available
    lines = out.read_text().splitlines()
    assert lines[0] == "sigma,psi" and len(lines) == 6


def test_cli_gen_and_usage(tmp_path, capsys):
    out = tmp_path / "lap.mtx"
    assert cli.main(["gen", "--matrix", "lapl:5x4", "--out", str(out)]) == 0
    assert mmio.read_matrix_market(out).n == 20
    assert cli.main(["analyze-shift", "--history", str(out), "--iter", "3"]) == 2
    assert cli.main(["gen", "--matrix", "nosuchfile.mtx", "--out", str(out)]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_solve_on_device(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    h = tmp_path / "h.csv"
    assert cli.main(["solve", "--matrix", "stencil:200x200", "--method", "pcg-sh", "--shift", "4",
                     "--maxit", "500", "--rhs", "ones-rhs", "--history", str(h)]) == 0
    outp = capsys.readouterr().out
    assert "n-iterations=500" in outp and "true residual norm" in outp
    recs = harness.load_history(h)
    assert len(recs) == 501 and recs[-1].rnorm_true <= 6.8e-11
    assert cli.main(["analyze-shift", "--history", str(h), "--iter", "500", "--sigma-grid", "0:1:8"]) == 0
