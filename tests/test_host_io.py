"""File formats and persistence (reference data_io.py):
byte-identical writers (golden bytes from the reference), exact round trips,
the five ingestion formats, and their error messages."""

import io

import numpy as np
import pytest

import paper_2304_13724_b200 as bm


def _io(golden):
    return golden["io"]


def test_writers_byte_identical(golden):
    g = _io(golden)
    model = bm.FactorModel(np.array(g["u"]), np.array(g["v"]))
    buf = io.StringIO()
    bm.save_model(model, buf)
    assert buf.getvalue() == g["model"]
    trace = bm.ConvergenceTrace()
    for i, (tr, te) in enumerate(zip(g["train"], g["test"]), start=1):
        trace.append(bm.TraceStep(i, tr, te, 0.0, 1))
    buf = io.StringIO()
    bm.write_trace(trace, buf, config={"k": 3, "grid": "2x2", "schedule": "const:1"})
    assert buf.getvalue() == g["trace"]
    d = bm.gen_synthetic(bm.SyntheticSpec(7, 5, 1, 5, seed=2, density=0.6))
    buf = io.StringIO()
    bm.save_dataset(d, buf)
    assert buf.getvalue() == g["dataset"]


def test_round_trips(tmp_path, golden):
    g = _io(golden)
    p = tmp_path / "model.txt"
    p.write_text(g["model"])
    m = bm.load_model(str(p))
    assert np.array_equal(m.u, np.array(g["u"])) and np.array_equal(m.v, np.array(g["v"]))
    p = tmp_path / "trace.csv"
    p.write_text(g["trace"])
    cfg, tr = bm.read_trace(str(p))
    assert cfg == {"k": "3", "grid": "2x2", "schedule": "const:1"}
    assert [s.train_rmse for s in tr] == g["train"]
    assert [s.test_rmse for s in tr] == g["test"]
    p = tmp_path / "d.csv"
    p.write_text(g["dataset"])
    d = bm.load(str(p), "csv")
    assert (d.n, d.m) == (7, 5)
    assert d.rows.tolist() == g["rows"] and d.values.tolist() == g["values"]


def test_formats(tmp_path):
    (tmp_path / "u.data").write_text("1\t2\t3\t881250949\n3\t1\t5\t1\n")
    d = bm.load(str(tmp_path / "u.data"), "ml-100k")
    assert (d.n, d.m) == (3, 2) and d.rows.tolist() == [0, 2] and d.cols.tolist() == [1, 0]
    (tmp_path / "r.dat").write_text("1::1::4::0\n2::3::2::0\n")
    d = bm.load(str(tmp_path / "r.dat"), "ml-1m")
    assert (d.n, d.m) == (2, 3) and d.values.tolist() == [4.0, 2.0]
    (tmp_path / "ratings.csv").write_text("userId,movieId,rating,timestamp\n1,2,3.5,0\n")
    d = bm.load(str(tmp_path / "ratings.csv"), "ml-20m")
    assert d.values.tolist() == [3.5]
    (tmp_path / "jester.csv").write_text("1.5,99,-2\n99,3,4\n")
    d = bm.load(str(tmp_path / "jester.csv"), "jester")
    assert (d.n, d.m) == (2, 3) and len(d) == 4
    (tmp_path / "t.csv").write_text("# shape: 10 12\n0,1,2.0\n3,4,1.0\n")
    d = bm.load(str(tmp_path / "t.csv"), "csv")
    assert (d.n, d.m) == (10, 12)


def test_format_errors(tmp_path):
    with pytest.raises(bm.DataError, match="unknown format"):
        bm.load("x", "parquet")
    (tmp_path / "e.csv").write_text("")
    with pytest.raises(bm.DataError, match="empty"):
        bm.load(str(tmp_path / "e.csv"), "csv")
    (tmp_path / "b.csv").write_text("1,2\n")
    with pytest.raises(bm.DataError, match="expected at least 3 fields"):
        bm.load(str(tmp_path / "b.csv"), "csv")
    (tmp_path / "d.csv").write_text("0,0,1\n0,0,2\n")
    with pytest.raises(bm.DataError, match="duplicate"):
        bm.load(str(tmp_path / "d.csv"), "csv")
    (tmp_path / "m.txt").write_text("2 2\n")
    with pytest.raises(bm.DataError, match="malformed header"):
        bm.load_model(str(tmp_path / "m.txt"))
    (tmp_path / "m2.txt").write_text("1 1 2\n1.0 2.0\n")
    with pytest.raises(bm.DataError, match="expected 2 factor rows"):
        bm.load_model(str(tmp_path / "m2.txt"))
