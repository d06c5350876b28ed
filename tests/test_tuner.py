"""Tuner parity: the product's optimize/exhaustive produce the reference's
exact traces for the same SimulateFn (R:proj/src/tuner.cpp:40-243), on the
reference's own test surfaces (R:proj/tests/test_tuner.cpp) and on random
surfaces; plus the reference's behavioural expectations."""
import math

import numpy as np
import pytest

import oracle

HW = dict(num_sms=108, max_warps=64, smem_per_sm=164 * 1024)


def convex_surface(c):
    ps, dist, wpb = c
    d = (30.0 * (math.log2(ps) - 2.0) ** 2 + 20.0 * (math.log2(dist) - 1.0) ** 2
         + 10.0 * (math.log2(wpb) - 1.0) ** 2)
    return 1000 + int(round(d))


def retreat_latency(c):
    ps, dist, wpb = c
    if wpb == 1:
        base = {2: 900, 4: 850, 8: 800, 16: 950}.get(ps, 1000)
        return base - dist
    if ps == 4 and wpb == 2:
        return 700
    return 2000


def retreat_value(c):
    ps, dist, wpb = c
    if wpb == 1:
        return {2: 820, 4: 900, 8: 800, 16: 990}.get(ps, 1000)
    if ps == 2 and wpb == 2:
        return 700
    if ps == 4 and wpb == 2:
        return 650
    return 2000


SURFACES = {
    "convex": convex_surface,
    "flat": lambda c: 500,
    "decreasing": lambda c: 1000000 - 100 * c[0] - 10 * c[1] - c[2],
    "retreat_latency": retreat_latency,
    "retreat_value": retreat_value,
}


def _hw(mgg, smem=164 * 1024):
    return mgg.HardwareProfile("a100", 108, 64, smem)


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("name", sorted(SURFACES))
@pytest.mark.parametrize("rule", [False, True])
def test_optimize_trace_matches_reference(mgg, name, rule):
    f = SURFACES[name]
    ours = mgg.optimize(f, _hw(mgg), 16, retreat_value_rank=rule)
    ref = oracle.ref_optimize(f, HW["num_sms"], HW["max_warps"], HW["smem_per_sm"], 16, rule)
    assert ours == ref


@needs_ref
def test_optimize_random_surfaces_match_reference(mgg):
    rng = np.random.default_rng(7007)
    grid = [(p, d, w) for p in (1, 2, 4, 8, 16, 32) for d in (1, 2, 4, 8, 16)
            for w in (1, 2, 4, 8, 16)]
    for trial in range(80):
        hi = 130 if trial % 3 == 0 else 100000  # small range -> many ties
        table = {c: int(rng.integers(100, hi)) for c in grid}
        smem_cap = int(rng.choice([164 * 1024, 4096, 2000]))
        dim = int(rng.choice([8, 16, 602]))
        budget = int(rng.integers(3, 20))
        rule = bool(trial % 2)
        try:
            ours = mgg.optimize(table.__getitem__, _hw(mgg, smem_cap), dim,
                                retreat_value_rank=rule, max_evaluations=budget)
        except mgg.ConfigError:  # origin inadmissible: the reference refuses too
            with pytest.raises(oracle.RefError) as ei:
                oracle.ref_optimize(table.__getitem__, 108, 64, smem_cap, dim, rule, budget)
            assert ei.value.code == 3
            continue
        ref = oracle.ref_optimize(table.__getitem__, 108, 64, smem_cap, dim, rule, budget)
        assert ours == ref, trial


@needs_ref
def test_exhaustive_matches_reference(mgg):
    for smem_cap in (164 * 1024, 5000):
        ours = mgg.exhaustive(convex_surface, _hw(mgg, smem_cap), 16)
        ref = oracle.ref_exhaustive(convex_surface, 108, 64, smem_cap, 16)
        assert ours == ref


def test_optimize_convex_minimum(mgg):
    trace, best = mgg.optimize(convex_surface, _hw(mgg), 16)
    assert best[:3] == (4, 2, 2) and best[3] == 1000
    assert len(trace) <= 15
    assert len({t[:3] for t in trace}) == len(trace)


def test_optimize_flat_and_budget(mgg):
    trace, best = mgg.optimize(lambda c: 500, _hw(mgg), 16)
    assert best[:3] == (1, 1, 1) and len(trace) <= 4
    trace, _ = mgg.optimize(SURFACES["decreasing"], _hw(mgg), 16)
    assert len(trace) <= 15


def test_optimize_never_invalid_and_errors(mgg):
    hw = _hw(mgg, mgg.smem(8, 1, 2, 16))
    trace, best = mgg.optimize(convex_surface, hw, 16)
    for t in trace:
        assert mgg.validate(*t[:3], 16, hw) == []
    with pytest.raises(mgg.ConfigError):
        mgg.optimize(convex_surface, _hw(mgg, 4), 16)

    def failing(c):
        if c[0] == 2:
            raise RuntimeError("boom")
        return 100
    with pytest.raises(RuntimeError, match="ps=2"):
        mgg.optimize(failing, _hw(mgg), 16)


def test_exhaustive_guards(mgg):
    with pytest.raises(mgg.ConfigError):
        mgg.exhaustive(convex_surface, _hw(mgg, 4), 16)


def test_costmodel_matches_reference_grid(mgg):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    for ps in (1, 3, 7, 16, 32, 33, 0):
        for dist in (1, 2, 5, 16, 17):
            for wpb in (1, 2, 9, 16, 17):
                for dim in (1, 16, 602):
                    assert mgg.wpw(ps, dist, wpb, dim) == oracle.ref_wpw(ps, dist, wpb, dim)
                    assert mgg.smem(ps, dist, wpb, dim) == oracle.ref_smem(ps, dist, wpb, dim)
                    for cap in (100, 164 * 1024):
                        hw = mgg.HardwareProfile("x", 108, 8, cap)
                        assert mgg.validate(ps, dist, wpb, dim, hw) == oracle.ref_validate(
                            ps, dist, wpb, dim, 108, 8, cap)


def test_profiles(mgg):
    a = mgg.resolve_profile("a100")
    assert (a.num_sms, a.smem_per_sm_bytes) == (108, 164 * 1024)
    b = mgg.resolve_profile("b200")
    assert (b.num_sms, b.max_warps_per_sm, b.smem_per_sm_bytes) == (148, 64, 228 * 1024)
    assert mgg.resolve_profile("v100").num_sms == 80
    assert mgg.resolve_profile("desk").max_warps_per_sm == 2
    wb = mgg.launch_geometry(4, 4, 1, 2, 1, "a100")
    assert wb[:2] == (2, 2)


def test_remote_partition_bytes_acceptance(mgg):
    """R:proj/tests/acceptance.cpp:378-390 (criterion 8)."""
    for size in (1, 2, 5, 16, 32):
        fine = mgg.remote_partition_bytes(size, 16, False, 4096)
        paged = mgg.remote_partition_bytes(size, 16, True, 4096)
        assert fine == size * 64 and paged == size * 4096
        assert paged >= 64 * fine
    assert mgg.remote_partition_bytes(3, 602, True, 4096) == 3 * 4096
    assert mgg.remote_partition_bytes(3, 2000, True, 4096) == 3 * 8192


def test_shipped_profiles_match_builtins(mgg):
    """R:proj/tests/test_costmodel.cpp:162-178, plus the b200 preset."""
    import os
    d = os.path.join(os.path.dirname(mgg.LIB_PATH), "profiles")
    for name in ("a100", "v100", "desk", "b200"):
        shipped = mgg.resolve_profile(os.path.join(d, name + ".json"))
        built = mgg.resolve_profile(name)
        assert shipped == built, name


def test_refit_latencies_arithmetic():
    # K5 numbers -> the reference LatencyModel schema (costmodel.hpp:32-49)
    from paper_2209_06800_b200 import probes
    m = {"local_chase_ns": 417.6, "local_gather_gbps": 6500.0}
    f = probes.refit_latencies(m, 1.965, 148)
    assert f["latencies"]["localLoadBase"] == 821
    assert f["latencies"]["perElemLocal"] == 1
    assert "remoteGetBase" not in f["latencies"]  # one GPU: keep the previous value
    m.update(peer_chase_ns=1000.0, peer_gather_gbps=700.0)
    f = probes.refit_latencies(m, 1.965, 148)
    assert f["latencies"]["remoteGetBase"] == 1965
    # 700 GB/s over 148 SMs = 2.41 B/cycle/SM -> 4 B take 1.66 cycles -> 2
    assert f["latencies"]["perElemRemote"] == 2
    assert "NVLink" in f["source"]["remoteGetBase"]
