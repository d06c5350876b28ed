"""Graph ingestion — the reference's test_graph.cpp cases against the product
(R:proj/tests/test_graph.cpp), plus the RMAT generator."""
import numpy as np
import pytest


def test_from_edges_kats(mgg):
    g = mgg.from_edges(3, [(0, 1), (0, 2), (1, 2)])
    assert g.row_ptr.tolist() == [0, 2, 3, 3] and g.col_idx.tolist() == [1, 2, 2]
    g = mgg.from_edges(2, np.zeros((0, 2), np.uint64))
    assert g.row_ptr.tolist() == [0, 0, 0] and g.num_edges == 0
    g = mgg.from_edges(4, [(3, 0), (0, 3)])
    assert g.row_ptr.tolist() == [0, 1, 1, 1, 2] and g.col_idx.tolist() == [3, 0]
    g = mgg.from_edges(3, [(0, 2), (0, 1), (0, 2)])
    assert g.col_idx.tolist() == [1, 2, 2]
    with pytest.raises(mgg.InputError, match="out of range"):
        mgg.from_edges(3, [(0, 5)])


def test_load_edge_list(mgg, tmp_path):
    def load(text):
        p = tmp_path / "g.txt"
        p.write_text(text)
        return mgg.load_edge_list(str(p))
    g = load("0 1\n1 0\n")
    assert g.num_nodes == 2 and g.row_ptr.tolist() == [0, 1, 2] and g.col_idx.tolist() == [1, 0]
    g = load("# c\n2 0\n")
    assert g.num_nodes == 3 and g.num_edges == 1
    assert load("% header\n\n0 1\n").num_edges == 1
    assert load("  0\t1  \r\n").num_edges == 1
    for bad in ["", "# nothing\n% here\n"]:
        with pytest.raises(mgg.ParseError):
            load(bad)
    with pytest.raises(mgg.ParseError, match=r"line 2"):
        load("0 1\n1 x\n")
    with pytest.raises(mgg.ParseError):
        load("0 1 7\n")
    with pytest.raises(mgg.ParseError):
        load("0\n")
    with pytest.raises(mgg.ParseError):
        load("99999999999999999999999 1\n")  # u64 overflow


def test_generators(mgg):
    a = mgg.gen_synthetic(mgg.UNIFORM, 100, 8, 42)
    b = mgg.gen_synthetic(mgg.UNIFORM, 100, 8, 42)
    c = mgg.gen_synthetic(mgg.UNIFORM, 100, 8, 43)
    assert np.array_equal(a.col_idx, b.col_idx) and not np.array_equal(a.col_idx, c.col_idx)
    assert a.num_edges == 800
    h = mgg.gen_synthetic(mgg.UNIFORM, 100, 8.5, 42)
    assert 800 <= h.num_edges <= 900
    p = mgg.gen_synthetic(mgg.POWERLAW, 1000, 10, 7)
    d = p.degrees()
    assert d.max() > 3 * d.mean() and d.min() >= 1
    with pytest.raises(mgg.InputError):
        mgg.gen_synthetic(mgg.UNIFORM, 0, 1, 0)
    with pytest.raises(mgg.InputError):
        mgg.gen_synthetic(mgg.UNIFORM, 10, -1, 0)


def test_rmat(mgg):
    g = mgg.gen_rmat(100_000, 1_600_000, seed=0)
    assert g.num_nodes == 100_000 and g.num_edges == 1_600_000
    assert g.col_idx.max() < 100_000
    g2 = mgg.gen_rmat(100_000, 1_600_000, seed=0)
    assert np.array_equal(g.col_idx, g2.col_idx)
    d = g.degrees()
    # skewed, low ids dense (unshuffled R-MAT keeps the core at low ids)
    assert d[:1000].mean() > 5 * d.mean()
    rows = np.split(g.col_idx, g.row_ptr[1:-1].astype(np.int64))
    assert all(np.all(np.diff(r.astype(np.int64)) >= 0) for r in rows[:2000])


def test_csr_round_trip(mgg, tmp_path):
    g = mgg.gen_synthetic(mgg.POWERLAW, 200, 6, 3)
    p = str(tmp_path / "g.bin")
    g.save_csr(p)
    h = mgg.load_csr(p)
    assert np.array_equal(g.row_ptr, h.row_ptr) and np.array_equal(g.col_idx, h.col_idx)
    # byte layout is the reference's: LE u64 N, E, row_ptr, col_idx
    raw = np.fromfile(p, dtype="<u8")
    assert raw[0] == 200 and raw[1] == g.num_edges
    assert np.array_equal(raw[2:203], g.row_ptr)
    (tmp_path / "short.bin").write_bytes(b"short")
    with pytest.raises(mgg.ParseError):
        mgg.load_csr(str(tmp_path / "short.bin"))


def test_validate_csr(mgg):
    with pytest.raises(mgg.InputError):
        mgg.CsrGraph.from_csr([0, 2, 1], [0])
    with pytest.raises(mgg.InputError):
        mgg.CsrGraph.from_csr([0, 1], [5])
    with pytest.raises(mgg.InputError):
        mgg.CsrGraph.from_csr([1, 1], [0])


def test_csr_round_trip_through_edges(mgg):
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = 1 + int(rng.integers(0, 200))
        e = rng.integers(0, n, size=(int(rng.integers(0, 8 * n)), 2), dtype=np.uint64)
        g = mgg.from_edges(n, e)
        src = np.repeat(np.arange(n, dtype=np.uint64), g.degrees().astype(np.int64))
        h = mgg.from_edges(n, np.stack([src, g.col_idx], 1))
        assert np.array_equal(g.row_ptr, h.row_ptr) and np.array_equal(g.col_idx, h.col_idx)
        assert int(g.degrees().sum()) == g.num_edges
