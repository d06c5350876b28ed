"""Partition metadata is bit-exact to the reference library (oracle/_ref).

Mirrors the reference's own suites (R:proj/tests/test_placement.cpp,
test_workload.cpp, acceptance.cpp criteria 1-2) but compares the product's
builder against the compiled reference on the same inputs.
"""
import json

import numpy as np
import pytest

from oracle import RefGraph, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _random_graph(rng, max_nodes=200, max_avg=8.0):
    # same distribution as R:proj/tests/test_util.hpp:57-68 (numpy stream)
    n = 1 + int(rng.integers(0, max_nodes))
    m = int(rng.integers(0, max(1, int(n * max_avg)) + 1))
    edges = rng.integers(0, n, size=(m, 2), dtype=np.uint64)
    return n, edges


def _both(mgg, n, edges):
    return mgg.from_edges(n, edges), RefGraph.from_edges(n, edges)


def test_generators_bit_identical(mgg):
    for kind in (0, 1):
        for n, avg, seed in [(1, 0, 0), (7, 3.5, 1), (1000, 8, 42), (5000, 16.25, 7),
                             (20000, 31.7, 9)]:
            g = mgg.gen_synthetic(kind, n, avg, seed)
            r = RefGraph.gen(kind, n, avg, seed)
            rp, cl = r.csr()
            assert np.array_equal(g.row_ptr, rp)
            assert np.array_equal(g.col_idx, cl)


def test_from_edges_identical(mgg):
    rng = np.random.default_rng(5)
    for _ in range(100):
        n, e = _random_graph(rng)
        g, r = _both(mgg, n, e)
        rp, cl = r.csr()
        assert np.array_equal(g.row_ptr, rp) and np.array_equal(g.col_idx, cl)


def test_split_matches_reference_1000_graphs(mgg):
    # acceptance criterion 1 (R:proj/tests/acceptance.cpp:54-70) vs the ref lib
    rng = np.random.default_rng(1001)
    for _ in range(1000):
        n, e = _random_graph(rng)
        gpus = 1 + int(rng.integers(0, 8))
        g, r = _both(mgg, n, e)
        assert np.array_equal(mgg.split_by_edges(g, gpus), r.split(gpus))


def test_placement_translate_footprint(mgg):
    rng = np.random.default_rng(33)
    for _ in range(100):
        n, e = _random_graph(rng)
        gpus = 1 + int(rng.integers(0, 6))
        mode = int(rng.integers(0, 2))
        dim = int(rng.integers(1, 700))
        g, r = _both(mgg, n, e)
        assert np.array_equal(mgg.plan_ne_placement(g, gpus, mode, dim),
                              r.placement(gpus, mode, dim))
        ids = np.arange(n, dtype=np.uint64)
        a, b = mgg.translate(g, gpus, mode, ids), r.translate(gpus, mode, ids)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        mem = int(rng.integers(0, 1 << 16))
        pa, fa = mgg.memory_footprint(g, gpus, mode, dim, mem)
        pb, fb = r.footprint(gpus, mode, dim, mem)
        assert np.array_equal(pa, pb) and fa == fb


def _expand_ref(rp):
    out = {}
    for kind in (0, 1):
        t, s, nb = rp.parts(kind)
        out[kind] = (t, s, nb)
    return out


def _expand_flat(fp, ranges):
    """FlatPlan -> (targets, sizes, global neighbor ids) per kind."""
    out = {}
    for kind in (0, 1):
        meta = fp.meta(kind).astype(np.int64)
        cols = fp.cols(kind).astype(np.uint64)
        targets = fp.first_target + meta[:-1, 0]
        sizes = np.diff(meta[:, 1])
        owner = cols >> np.uint64(28)
        off = cols & np.uint64((1 << 28) - 1)
        glob = ranges[owner.astype(np.int64), 0] + off if len(cols) else cols
        out[kind] = (targets.astype(np.uint64), sizes.astype(np.uint64), glob)
    return out


CFGS = [(1, 1, 1), (2, 1, 2), (16, 1, 2), (32, 16, 16), (3, 5, 7), (7, 2, 1)]


@pytest.mark.parametrize("mapping,granularity", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_flat_plan_expands_to_reference_plan(mgg, mapping, granularity):
    """Every partition (target, kind, neighbor ids), every warp's task list,
    the block tiling and smem equal the reference KernelLaunchPlan; the
    canonical JSON is byte-identical (R:proj/src/workload.cpp:276-305)."""
    rng = np.random.default_rng(2002 + 10 * mapping + granularity)
    for it in range(60):
        n, e = _random_graph(rng, 120)
        gpus = 1 + int(rng.integers(0, 6))
        mode = int(rng.integers(0, 2))
        gpu = int(rng.integers(0, gpus))
        ps, dist, wpb = CFGS[it % len(CFGS)]
        dim = int(rng.integers(1, 64))
        g, r = _both(mgg, n, e)
        fp = mgg.build_flat_plan(g, gpus, gpu, ps, dist, wpb, dim, mode, mapping, granularity)
        rp = r.plan(gpus, mode, gpu, ps, dist, wpb, dim, mapping, granularity)
        ranges = mgg.plan_ne_placement(g, gpus, mode, dim).astype(np.uint64)
        a, b = _expand_flat(fp, ranges), _expand_ref(rp)
        for kind in (0, 1):
            for x, y in zip(a[kind], b[kind]):
                assert np.array_equal(x, y), (kind, it)
        assert fp.num_warps == rp.n_warps and fp.num_blocks == rp.n_blocks
        assert fp.smem_bytes_per_block == rp.smem
        off, kind, idx = fp.tasks()
        roff, _, rkind, ridx, bf, bc = rp.warps()
        assert np.array_equal(off, roff)
        assert np.array_equal(kind, rkind) and np.array_equal(idx, ridx)
        assert list(bc) == [min(wpb, rp.n_warps - f) for f in bf]
        assert fp.to_json() == rp.json()


def test_plan_at_config1_scale(mgg):
    """Config-1 shape (RMAT 100K / 1.6M, 2 logical partitions): the device
    plan of both gpus equals the reference's."""
    g = mgg.gen_rmat(100_000, 1_600_000, seed=0)
    r = RefGraph.from_csr(g.row_ptr, g.col_idx)
    ranges = mgg.plan_ne_placement(g, 2, 1, 16).astype(np.uint64)
    for gpu in (0, 1):
        fp = mgg.build_flat_plan(g, 2, gpu, 16, 1, 2, 16)
        rp = r.plan(2, 1, gpu, 16, 1, 2, 16)
        a, b = _expand_flat(fp, ranges), _expand_ref(rp)
        for kind in (0, 1):
            for x, y in zip(a[kind], b[kind]):
                assert np.array_equal(x, y)
        assert fp.num_warps == rp.n_warps and fp.num_blocks == rp.n_blocks


def test_local_remote_conservation(mgg):
    """acceptance criterion 2: local+remote = chunk edges as multisets."""
    rng = np.random.default_rng(44)
    for _ in range(200):
        n, e = _random_graph(rng, 80)
        gpus = 1 + int(rng.integers(0, 4))
        mode = int(rng.integers(0, 2))
        ps = 1 + int(rng.integers(0, 32))
        g, r = _both(mgg, n, e)
        ranges = mgg.plan_ne_placement(g, gpus, mode, 4).astype(np.uint64)
        chunks = mgg.chunk_ranges(g, gpus)
        for gpu in range(gpus):
            fp = mgg.build_flat_plan(g, gpus, gpu, ps, 1, 1, 4, mode)
            exp = _expand_flat(fp, ranges)
            lo, hi = (int(x) for x in chunks[gpu])
            rp_, cl_ = g.row_ptr, g.col_idx
            want = sorted((v, int(u)) for v in range(lo, hi) for u in cl_[rp_[v]:rp_[v + 1]])
            got = []
            for kind in (0, 1):
                t, s, nb = exp[kind]
                tt = np.repeat(t, s.astype(np.int64))
                got += list(zip(tt.tolist(), nb.tolist()))
                owner = mgg.translate(g, gpus, mode, nb)[0] if len(nb) else np.zeros(0)
                assert np.all((owner == gpu) == (kind == 0))
                assert np.all(s <= ps) and np.all(s >= 1)
            assert sorted(got) == want


def test_reference_known_answers(mgg):
    """Hand cases from R:proj/tests/test_placement.cpp / test_workload.cpp."""
    deg = lambda ds: mgg.from_edges(len(ds), [(v, 0) for v, d in enumerate(ds) for _ in range(d)])  # noqa: E731
    assert list(mgg.split_by_edges(deg([2, 2, 2, 2]), 2)) == [2]
    assert list(mgg.split_by_edges(deg([5, 1, 1, 1]), 2)) == [1]
    assert list(mgg.split_by_edges(deg([3, 3, 2]), 1)) == []
    ch = mgg.chunk_ranges(deg([4, 4]), 5)
    assert ch.shape == (5, 2) and int((ch[:, 1] - ch[:, 0]).sum()) == 2
    g10 = mgg.from_edges(10, [])
    assert mgg.plan_ne_placement(g10, 4, 0, 8).tolist() == [[0, 3], [3, 6], [6, 9], [9, 10]]
    g6 = mgg.from_edges(6, [])
    gpu, off = mgg.translate(g6, 2, 0, [4, 0])
    assert list(zip(gpu.tolist(), off.tolist())) == [(1, 1), (0, 0)]
    with pytest.raises(mgg.InputError):
        mgg.translate(g6, 2, 0, [6])
    # partition slicing: degrees [5,2], ps=2 -> sizes [2,2,1,2]
    g = mgg.from_edges(6, [(0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (1, 1), (1, 2)])
    fp = mgg.build_flat_plan(g, 1, 0, 2, 1, 1, 4, 0)
    assert np.diff(fp.meta(0)[:, 1]).tolist() == [2, 2, 1, 2]
    # smem: (16,1,2) D=16 -> 384 ; (4,1,1) D=602 -> 16 + 4816 ; acceptance 79104
    assert mgg.smem(16, 1, 2, 16) == 384
    assert mgg.smem(4, 1, 1, 602) == 4 * 4 + 4816
    assert mgg.smem(32, 16, 16, 602) == 79104
    # footprint at Reddit scale (R:proj/tests/test_placement.cpp:177-186)
    rp = np.zeros(232965 + 1, np.uint64)
    big = mgg.CsrGraph.from_csr(rp, np.zeros(0, np.uint64))
    per, fits = mgg.memory_footprint(big, 4, 0, 602, 40 << 30)
    assert int(per[:, 0].sum()) == 232965 * 602 * 4 and fits


def test_plan_json_roundtrip_shape(mgg):
    g = mgg.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 0), (1, 2)])
    fp = mgg.build_flat_plan(g, 2, 0, 2, 1, 2, 8)
    j = json.loads(fp.to_json())
    assert set(j) == {"cfg", "dim", "smemBytesPerBlock", "localParts", "remoteParts", "warps"}
    assert j["cfg"] == {"dist": 1, "ps": 2, "wpb": 2}


@pytest.mark.parametrize("workload", ["reddit-gcn", "products-gcn", "orkut-gcn"])
def test_plan_at_baseline_scale_8_parts(mgg, workload):
    """BASELINE configs[1..3] graphs at full size, 8 parts, the bench's tuned
    (ps, dist, wpb): every part's device plan expands to the reference's
    KernelLaunchPlan — partitions, warp task lists, block tiling, smem
    (R:proj/tests/acceptance.cpp:54-116 criteria, at scale)."""
    import bench
    _, g, model, _ = bench.build(mgg, workload)
    ps, dist, wpb = bench.WORKLOADS[workload][3][:3]
    dim = model.in_dim
    r = RefGraph.from_csr(g.row_ptr, g.col_idx)
    assert np.array_equal(mgg.split_by_edges(g, 8), r.split(8))
    ranges = mgg.plan_ne_placement(g, 8, 1, dim).astype(np.uint64)
    for gpu in range(8):
        fp = mgg.build_flat_plan(g, 8, gpu, ps, dist, wpb, dim)
        rp = r.plan(8, 1, gpu, ps, dist, wpb, dim)
        a, b = _expand_flat(fp, ranges), _expand_ref(rp)
        for kind in (0, 1):
            for x, y in zip(a[kind], b[kind]):
                assert np.array_equal(x, y), (workload, gpu, kind)
        assert fp.num_warps == rp.n_warps and fp.num_blocks == rp.n_blocks
        assert fp.smem_bytes_per_block == rp.smem
        off, kind, idx = fp.tasks()
        roff, _, rkind, ridx, bf, bc = rp.warps()
        assert np.array_equal(off, roff)
        assert np.array_equal(kind, rkind) and np.array_equal(idx, ridx)
        del fp, rp, a, b
