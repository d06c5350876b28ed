"""Pins the oracle before anything is checked against it.

Metadata restatement (oracle.c) vs the reference's golden fixtures
(tests/golden/reference_metadata.json, generated from oracle/_ref) and the
reference's own known-answer tests. Layer arithmetic (parity unpinned by
reference code) vs hand-computed known answers from the paper's equations
and an fp64-vs-fp32 cross-check.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "reference_metadata.json")))


def test_split_restatement_vs_golden():
    for case in GOLD["splits"]:
        rp = np.array(case["row_ptr"], np.uint64)
        assert oracle.split_points(rp, case["gpus"]).tolist() == case["split"]
        assert oracle.placement(rp, case["gpus"], 0).tolist() == case["equal_nodes"]


def test_split_restatement_reference_kats():
    # R:proj/tests/test_placement.cpp:39-61
    assert oracle.split_points(np.array([0, 2, 4, 6, 8], np.uint64), 2).tolist() == [2]
    assert oracle.split_points(np.array([0, 5, 6, 7, 8], np.uint64), 2).tolist() == [1]
    assert oracle.split_points(np.array([0, 3, 6, 8], np.uint64), 1).tolist() == []
    # equal_nodes on 10 nodes / 4 gpus (test_placement.cpp:104-108)
    assert oracle.placement(np.zeros(11, np.uint64), 4, 0).tolist() == [
        [0, 3], [3, 6], [6, 9], [9, 10]]


def test_partition_counts_and_interleave_vs_golden_plans():
    for case in GOLD["plans"]:
        plan = json.loads(case["plan_json"])
        rp = np.array(case["row_ptr"], np.uint64)
        cl = np.array(case["col_idx"], np.uint64)
        gpus, gpu = case["gpus"], case["gpu"]
        ranges = oracle.placement(rp, gpus, case["mode"])
        chunk = oracle.placement(rp, gpus, 1)[gpu]
        if case["granularity"] == 0:
            lp, rp_, le, re_ = oracle.partition_counts(rp, cl, gpus, ranges, chunk, gpu,
                                                       case["ps"])
            assert lp == len(plan["localParts"]) and rp_ == len(plan["remoteParts"])
            assert le == sum(len(p["neighbors"]) for p in plan["localParts"])
            assert re_ == sum(len(p["neighbors"]) for p in plan["remoteParts"])
        if case["mapping"] == 0:
            nl, nr = len(plan["localParts"]), len(plan["remoteParts"])
            for w in plan["warps"]:
                want = [(0 if k == "local" else 1, i) for k, i in w["tasks"]]
                assert oracle.warp_tasks(nl, nr, case["dist"], w["warp"]) == want


def test_interleave_reference_kats():
    # R:proj/tests/test_workload.cpp:153-186: dist 1 -> [L,R] x4, dist 2 -> [L,L,R,R] x2
    for w in range(4):
        assert oracle.warp_tasks(4, 4, 1, w) == [(0, w), (1, w)]
    assert oracle.warp_tasks(4, 4, 2, 0) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert oracle.warp_tasks(4, 4, 2, 1) == [(0, 2), (0, 3), (1, 2), (1, 3)]
    assert oracle.warp_tasks(3, 0, 1, 2) == [(0, 2)]


def test_product_builder_vs_golden_plans(mgg):
    """The product's device plan, expanded, is byte-identical to the
    reference plan JSON stored in the fixture (no oracle/_ref needed)."""
    for case in GOLD["plans"]:
        g = mgg.CsrGraph.from_csr(case["row_ptr"], case["col_idx"])
        fp = mgg.build_flat_plan(g, case["gpus"], case["gpu"], case["ps"], case["dist"],
                                 case["wpb"], case["dim"], case["mode"], case["mapping"],
                                 case["granularity"])
        assert fp.to_json() == case["plan_json"]


def test_product_generators_vs_golden(mgg):
    for case in GOLD["generators"]:
        g = mgg.gen_synthetic(case["kind"], case["n"], case["avg"], case["seed"])
        assert g.row_ptr.tolist() == case["row_ptr"]
        assert g.col_idx.tolist() == case["col_idx"]


def test_product_tuner_vs_golden(mgg):
    import math

    def convex(c):
        ps, dist, wpb = c
        return 1000 + int(round(30.0 * (math.log2(ps) - 2) ** 2 + 20.0 *
                                (math.log2(dist) - 1) ** 2 + 10.0 * (math.log2(wpb) - 1) ** 2))
    for key, cap in (("convex", 164 * 1024), ("convex_capped", 1000)):
        trace, best = mgg.optimize(convex, mgg.HardwareProfile("a100", 108, 64, cap), 16)
        gt, gb = GOLD["tuner"][key]
        assert [list(t) for t in trace] == gt and list(best) == gb


# ---------------------------------------------------------------------------
# layer arithmetic (paper equations; hand known answers)


def _py_aggregate(rows, x, self_scale=1.0, relu=False):
    f = (lambda v: max(v, 0.0)) if relu else (lambda v: v)
    out = []
    for v, nb in enumerate(rows):
        acc = [self_scale * f(x[v][j]) for j in range(len(x[0]))]
        for u in nb:
            for j in range(len(x[0])):
                acc[j] += f(x[u][j])
        out.append(acc)
    return np.array(out)


def test_aggregate_hand_example():
    # 3 nodes: 0 <- {1, 2}, 1 <- {0}, 2 <- {} ; a_v = h_v + Σ h_u (R:PAPER.md:33-38)
    rp = np.array([0, 2, 3, 3], np.uint64)
    cl = np.array([1, 2, 0], np.uint64)
    x = np.array([[1, -2], [3, 4], [-5, 6]], np.float32)
    got = oracle.aggregate(rp, cl, x)
    assert got.tolist() == [[-1, 8], [4, 2], [-5, 6]]
    got = oracle.aggregate(rp, cl, x, relu_in=True, self_scale=2.0)
    assert got.tolist() == [[5, 10], [7, 8], [0, 12]]
    # sym norm: d = deg+1 = [3, 2, 1]; a_0 = 1/3 h0 + h1/sqrt(6) + h2/sqrt(3)
    got = oracle.aggregate(rp, cl, x, norm=1)
    want0 = x[0] / 3 + x[1] / np.sqrt(6) + x[2] / np.sqrt(3)
    assert np.allclose(got[0], want0, rtol=1e-6)


def test_aggregate_matches_python_loops():
    rng = np.random.default_rng(3)
    n = 40
    rows = [sorted(rng.integers(0, n, rng.integers(0, 9)).tolist()) for _ in range(n)]
    rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.uint64)
    cl = np.array([u for r in rows for u in r], np.uint64)
    x = rng.uniform(-1, 1, (n, 5)).astype(np.float32)
    for relu in (False, True):
        want = _py_aggregate(rows, x.astype(np.float64).tolist(), 1.5, relu)
        got = oracle.aggregate(rp, cl, x, self_scale=1.5, relu_in=relu)
        assert np.allclose(got, want, rtol=1e-6, atol=1e-6)


def test_gcn2_hand_example(mgg):
    # path 0 <- 1 <- 2 with identity-ish weights: checks Â·ReLU(Â X W1)·W2
    rp = np.array([0, 1, 2, 2], np.uint64)
    cl = np.array([1, 2], np.uint64)
    x = np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, 2.0]], np.float32)
    w1 = np.array([[1.0, -1.0], [1.0, 1.0]], np.float32)
    w2 = np.array([[1.0], [0.5]], np.float32)
    model = mgg.Model(0, 2, 2, 2, 1, np.concatenate([w1.ravel(), w2.ravel()]))
    h1, logits, z = oracle.gcn2_forward(rp, cl, x, model)
    xw = x @ w1                                  # [[1,-1],[1,1],[1,3]]
    a1 = np.array([xw[0] + xw[1], xw[1] + xw[2], xw[2]])
    assert np.array_equal(h1, np.maximum(a1, 0))
    a2 = np.array([h1[0] + h1[1], h1[1] + h1[2], h1[2]])
    assert np.allclose(logits, a2 @ w2)
    assert np.allclose(z, 1.0)  # one class -> softmax 1


def test_fp64_vs_fp32_cross_check(mgg):
    g = mgg.gen_rmat(5000, 80000, seed=3)
    x = mgg.random_features(g.num_nodes, 24, seed=4)
    a64 = oracle.aggregate(g.row_ptr, g.col_idx, x, acc64=True)
    a32 = oracle.aggregate(g.row_ptr, g.col_idx, x, acc64=False)
    scale = np.maximum(np.abs(a64).max(axis=1, keepdims=True), 1e-6)
    assert (np.abs(a64 - a32) / scale).max() < 1e-5
    model = mgg.make_gin(24, 16, 5, layers=3)
    l64, _ = oracle.gin_forward(g.row_ptr, g.col_idx, x, model, acc64=True)
    l32, _ = oracle.gin_forward(g.row_ptr, g.col_idx, x, model, acc64=False)
    scale = np.maximum(np.abs(l64).max(axis=1, keepdims=True), 1e-6)
    assert (np.abs(l64 - l32) / scale).max() < 1e-4


def test_partition_independence_of_layer_output(mgg):
    """A property the kernels must share: the forward does not depend on how
    many parts the graph is split into (checked here on the oracle's input
    side: every plan of every part covers each edge exactly once)."""
    g = mgg.gen_rmat(2000, 20000, seed=8)
    rp = g.row_ptr
    for gpus in (1, 2, 3, 8):
        ranges = oracle.placement(rp, gpus, 1)
        tot = 0
        for gpu in range(gpus):
            c = oracle.partition_counts(rp, g.col_idx, gpus, ranges, ranges[gpu], gpu, 7)
            tot += c[2] + c[3]
        assert tot == g.num_edges


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_restatement_vs_reference_library_fuzz():
    rng = np.random.default_rng(99)
    for _ in range(300):
        n = 1 + int(rng.integers(0, 150))
        e = rng.integers(0, n, size=(int(rng.integers(0, 6 * n + 1)), 2), dtype=np.uint64)
        r = oracle.RefGraph.from_edges(n, e)
        rp, cl = r.csr()
        gpus = 1 + int(rng.integers(0, 8))
        assert np.array_equal(oracle.split_points(rp, gpus), r.split(gpus))
        for mode in (0, 1):
            assert np.array_equal(oracle.placement(rp, gpus, mode), r.placement(gpus, mode))


def _scipy_adj(rp, cl, n, self_loops):
    import scipy.sparse as sp
    rp = np.asarray(rp, np.int64)
    cl = np.asarray(cl, np.int64)
    a = sp.csr_matrix((np.ones(len(cl)), cl, rp), shape=(n, n))  # row = target, duplicates summed
    return a + sp.identity(n, format="csr") if self_loops else a


@pytest.mark.parametrize("norm", [0, 1])
def test_gcn2_vs_independent_scipy_restatement(mgg, norm):
    """The oracle's GCN-2L (R:PAPER.md:504-508: Z = softmax(Â·ReLU(Â·X·W1)·W2),
    Â = A + I, optionally D^-1/2 (A+I) D^-1/2 with d = |N(v)| + 1) against an
    independent fp64 restatement with scipy.sparse matrix products — two
    implementations of the paper's formula agreeing to fp32 output rounding
    (the layer arithmetic has no reference code to pin it, R:SPEC.md:121-124)."""
    g = mgg.gen_rmat(3000, 40000, seed=11)
    n = g.num_nodes
    x = mgg.random_features(n, 20, seed=12)
    model = mgg.make_gcn(20, 12, 7, seed=13)
    w1 = model.w1[: 20 * 12].reshape(20, 12).astype(np.float64)
    w2 = model.w1[20 * 12:].reshape(12, 7).astype(np.float64)
    ahat = _scipy_adj(g.row_ptr, g.col_idx, n, True)
    if norm:
        d = np.diff(np.asarray(g.row_ptr, np.int64)).astype(np.float64) + 1.0
        import scipy.sparse as sp
        s = sp.diags(1.0 / np.sqrt(d))
        ahat = s @ ahat @ s
    h1 = np.maximum(ahat @ (x.astype(np.float64) @ w1), 0)
    logits = ahat @ h1 @ w2
    z = np.exp(logits - logits.max(axis=1, keepdims=True))
    z /= z.sum(axis=1, keepdims=True)
    _, lg, zo = oracle.gcn2_forward(g.row_ptr, g.col_idx, x, model, norm=norm)
    scale = np.maximum(np.abs(logits).max(axis=1, keepdims=True), 1e-6)
    assert (np.abs(lg - logits) / scale).max() < 2e-6
    # the oracle's softmax reads its fp32 logits: |dp| <= 2 |dlogit| ~ 2 |l| 2^-24
    assert np.abs(zo - z).max() < 2e-6 + 4 * np.abs(logits).max() * 2.0 ** -24


def test_gin_vs_independent_scipy_restatement(mgg):
    """The oracle's GIN (R:PAPER.md:511-517: h' = MLP((1+eps) h_v + Σ h_u),
    MLP = Linear-ReLU-Linear, ReLU between layers, softmax head) against the
    same independent scipy.sparse fp64 restatement."""
    g = mgg.gen_synthetic(mgg.POWERLAW, 2500, 9.0, 5)
    n = g.num_nodes
    x = mgg.random_features(n, 18, seed=6)
    model = mgg.make_gin(18, 10, 6, layers=3, seed=7, eps=0.3)
    adj = _scipy_adj(g.row_ptr, g.col_idx, n, False)
    dims = model.gin_dims()
    h = x.astype(np.float64)
    o1 = ob1 = o2 = ob2 = 0
    for l in range(model.layers):
        din, dout = dims[l], dims[l + 1]
        w1 = model.w1[o1:o1 + din * 10].reshape(din, 10).astype(np.float64)
        b1 = model.b1[ob1:ob1 + 10].astype(np.float64)
        w2 = model.w2[o2:o2 + 10 * dout].reshape(10, dout).astype(np.float64)
        b2 = model.b2[ob2:ob2 + dout].astype(np.float64)
        o1, ob1, o2, ob2 = o1 + din * 10, ob1 + 10, o2 + 10 * dout, ob2 + dout
        a = (1.0 + model.eps) * h + adj @ h
        h = np.maximum(a @ w1 + b1, 0) @ w2 + b2
        if l + 1 < model.layers:
            h = np.maximum(h, 0)
    z = np.exp(h - h.max(axis=1, keepdims=True))
    z /= z.sum(axis=1, keepdims=True)
    lg, zo = oracle.gin_forward(g.row_ptr, g.col_idx, x, model)
    scale = np.maximum(np.abs(h).max(axis=1, keepdims=True), 1e-6)
    assert (np.abs(lg - h) / scale).max() < 2e-6
    assert np.abs(zo - z).max() < 2e-6 + 4 * np.abs(h).max() * 2.0 ** -24
