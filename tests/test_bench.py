"""bench.py contract on CPU: the reference arm's JSON line (the only arm that
runs without a GPU), the algorithmic-byte formula of the roofline, the
aggregation widths of the layer programs, and the product arm's loud failure
without a device (no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_agg_bytes_formula():
    # E*(4*pitch + 4) + 8*P + 8*rows*pitch, pitch = round4(dim)
    assert bench.agg_bytes(10, 3, 5, 16) == 10 * (64 + 4) + 24 + 8 * 5 * 16
    assert bench.agg_bytes(7, 1, 2, 41) == 7 * (4 * 44 + 4) + 8 + 8 * 2 * 44
    assert bench.agg_bytes(0, 0, 0, 1) == 0


def test_agg_widths(mgg):
    assert bench.agg_widths(mgg.make_gcn(602, 16, 41)) == [16, 16]
    assert bench.agg_widths(mgg.make_gcn(16, 16, 16)) == [16, 16]
    assert bench.agg_widths(mgg.make_gcn(8, 32, 4)) == [8, 4]
    assert bench.agg_widths(mgg.make_gin(100, 64, 47, layers=5)) == [64] * 5


def test_workload_table_matches_baseline():
    # configs[0..3] of BASELINE.json + the RMAT variants; tuned configs valid
    labels = " ".join(w[0] for w in bench.WORKLOADS.values())
    for key in ("configs[0]", "configs[1]", "configs[2]", "configs[3]"):
        assert key in labels
    for name, (_, g, m, tuned) in bench.WORKLOADS.items():
        ps, dist, wpb = tuned[:3]
        assert 1 <= ps <= 32 and 1 <= dist <= 16 and 1 <= wpb <= 16, name
        assert len(tuned) == 3 or tuned[3] in (0, 1, 2, 3), name
        assert g[0] in ("powerlaw", "rmat") and m[0] in ("gcn", "gcn-norm", "gin"), name


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
         "--workload", "config1", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, cwd=ROOT,
        env={**os.environ, "RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "GEdges/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_never_loads_the_product():
    # the reference arm builds its graph/X/W from oracle/ and numpy only
    code = (f"import runpy, sys; sys.path.insert(0, {ROOT!r}); "
            "sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'config1', "
            "'--steps', '1', '--warmup', '0']; "
            f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__'); "
            "bad = [m for m in sys.modules if m.startswith('paper_2209_06800_b200')]; "
            "assert not bad, bad; "
            "maps = open('/proc/self/maps').read(); assert 'libmgg' not in maps")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env={**os.environ, "RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]


def test_reference_inputs_identical_to_product_inputs(mgg):
    import numpy as np
    for name in ("config1", "products-gcn", "products-gin", "reddit-gcn-norm"):
        mspec = bench.WORKLOADS[name][2]
        a = bench.np_model(mspec)
        mk, din, hid, out, layers = mspec
        b = (mgg.make_gcn(din, hid, out, seed=2, norm=mk == "gcn-norm") if mk != "gin"
             else mgg.make_gin(din, hid, out, layers=layers, seed=2))
        for f in ("kind", "layers", "in_dim", "hidden", "out_dim", "eps", "norm"):
            assert getattr(a, f) == getattr(b, f), (name, f)
        for f in ("w1", "b1", "w2", "b2"):
            x, y = getattr(a, f), getattr(b, f)
            assert (x is None and y is None) or np.array_equal(x, y), (name, f)
    assert np.array_equal(bench.np_features(1000, 37, 1), mgg.random_features(1000, 37, 1))
    rp, cl, _, _ = bench.ref_graph("config1")
    g = mgg.gen_rmat(100_000, 1_600_000, 0)
    assert np.array_equal(rp, g.row_ptr) and np.array_equal(cl, g.col_idx)


def test_reference_and_product_configs_agree():
    import types
    args = types.SimpleNamespace(ps=16, dist=8, wpb=8, k1_form=0, fetch="auto")
    m = bench.np_model(bench.WORKLOADS["products-gcn"][2])
    a = bench.workload_config("products-gcn", args, 10, 20, m, 1)
    assert a == bench.workload_config("products-gcn", args, 10, 20, m, 1)
    assert "layer_forward_ms" not in a  # nothing measured in the config


def test_roofline_bound_by_table_size():
    # Reddit-shaped width 16: 15 MB table -> L2-bound, rows-only bytes vs probe
    r = bench.roofline(232_965, 114_166_771, 3_700_000, 232_965, 16, 0.53, 15_000.0,
                       534_887_424, ["agg_local<4, false, 2>"])
    assert r["bound"] == "l2" and r["peak"] == 15_000.0
    assert abs(r["achieved"] - 114_166_771 * 64 / 0.53e-3 / 1e9) < 1
    assert r["frac"] < 1.2 and r["dram"]["frac"] < 0.2
    # products-shaped: 157 MB table -> HBM-bound on the algorithmic bytes
    r = bench.roofline(2_449_029, 60_800_000, 4_000_000, 2_449_029, 16, 0.71, 15_000.0,
                       4_390_000_000, ["agg_group_hint<4, false, 8>"])
    assert r["bound"] == "hbm" and r["peak_source"] in ("measured", "fallback")
    assert 0.5 < r["frac"] < 1.2
    assert "agg_group_hint" in r["kernel"]


def test_reference_arm_nonzero_rank_is_silent():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
         "--workload", "config1", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=300, cwd=ROOT,
        env={**os.environ, "RANK": "1"})
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_product_arm_fails_loudly_without_gpu(mgg):
    if mgg.cuda_available():
        pytest.skip("a GPU is visible: the product arm would run")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "config1", "--steps",
         "1", "--warmup", "3", "--no-cpu", "--no-e2e"],
        capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "no CUDA device" in (out.stderr + out.stdout)


def test_traffic_table_covers_every_workload():
    # roofline.traffic comes from the committed ncu capture of each workload's
    # tuned config (profiles/k1_traffic.json); a retune must come with a capture
    import types
    for name, (_, g, _, tuned) in bench.WORKLOADS.items():
        ps, dist, wpb = tuned[:3]
        parts = 2 if name == "config1" else 1
        args = types.SimpleNamespace(workload=name, ps=ps, dist=dist, wpb=wpb)
        t = bench._traffic(args, parts)
        assert t is not None and t > 0, f"no ncu traffic for {name} {tuned} parts={parts}"


def test_k1_form_rule():
    # mirrors pick_lean: ps <= 16 or partitions under 2/3 full -> group kernel
    import numpy as np
    full = np.arange(0, 33 * 100, 33)          # rows of 33 -> windows 32 + 1 (avg 16.5)
    assert bench.k1_form(full, 32, 1).startswith("agg_group")
    long_rows = np.arange(0, 64 * 100, 64)     # rows of 64 at ps 32 -> full windows
    assert bench.k1_form(long_rows, 32, 1).startswith("agg_local")
    assert bench.k1_form(long_rows, 16, 1).startswith("agg_group_hint")
    assert bench.k1_form(long_rows, 16, 1, width=64) == "agg_group (group per partition)"
    assert bench.k1_form(long_rows, 32, 2).startswith("agg_gpair")
    assert bench.k1_form(long_rows, 16, 1, form=1).startswith("agg_local")
    assert "4 rows" in bench.k1_form(long_rows, 32, 1, form=3)


def test_gpus_n_without_torchrun_needs_n_devices():
    # `--gpus N` outside torchrun re-executes under torch.distributed.run with N
    # ranks; with fewer devices visible it says so instead of faking N logical parts
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
         "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT,
        env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs visible: the re-exec would run")
    assert out.returncode != 0
    assert "CUDA device(s) visible" in (out.stderr + out.stdout)


def test_link_roofline_picks_the_binding_term():
    # per GPU the roofline is the larger of the HBM and NVLink terms
    import bench
    base = {"algorithmic_bytes_per_launch": 650_000_000, "bound": "hbm", "achieved": 5000.0,
            "peak": 6500.0, "frac": 0.77}
    # 0.1 ms launch, 130 MB over the link: 130e6/900e9 = 0.144 ms > 650e6/6500e9 = 0.1 ms
    r = bench.link_roofline(dict(base), 130_000_000, 0.2, 6500.0)
    assert r["bound"] == "nvlink" and r["peak"] == 900.0
    assert abs(r["achieved"] - 650.0) < 1e-6 and abs(r["frac"] - 650 / 900) < 1e-4
    assert r["hbm_bound"]["frac"] == 0.77
    # a small link term leaves the HBM bound in place
    r = bench.link_roofline(dict(base), 10_000_000, 0.2, 6500.0)
    assert r["bound"] == "hbm" and r["nvlink"]["bytes_per_launch"] == 10_000_000


def test_locality_csr_for_the_hiding_line():
    # the slow-peer hiding measurement's graph: rows sorted, neighbours within
    # the window except the `far` fraction
    import numpy as np

    import bench
    rp, cl = bench.locality_csr(20000, 10.0, 8, 0.02, seed=3)
    assert rp[0] == 0 and np.all(np.diff(rp.astype(np.int64)) >= 1) and int(rp[-1]) == len(cl)
    assert cl.max() < 20000
    tgt = np.repeat(np.arange(20000), np.diff(rp.astype(np.int64)))
    far = np.abs(cl.astype(np.int64) - tgt) > 8
    assert 0.01 < far.mean() < 0.03
    for r in range(0, 20000, 997):  # rows sorted
        row = cl[int(rp[r]):int(rp[r + 1])]
        assert np.all(np.diff(row.astype(np.int64)) >= 0)
