"""The C-ABI boundary: libmgg.so loads on a CPU-only host and exports every
function include/mgg.h declares; errors map to the documented status codes."""
import ctypes
import os
import re

import pytest


def _declared(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(mgg_[a-z0-9_]+)\s*\(", text)
    # drop the typedef'd callback name
    return sorted(set(n for n in names if n != "mgg_measure_fn"))


def test_header_symbols_exported(mgg):
    from paper_2209_06800_b200 import _lib
    names = _declared(_lib.HEADER)
    assert len(names) > 60
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    # and the raw dynamic symbol table agrees (no Python-side aliasing)
    so = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        getattr(so, n)


def test_library_is_in_tree(mgg):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    assert mgg.LIB_PATH.startswith(root)
    assert os.path.exists(mgg.LIB_PATH)


def test_sm100a_code_in_library(mgg):
    # the fatbin carries sm_100a SASS for the kernels (cuobjdump if present)
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", mgg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_codes(mgg, tmp_path):
    with pytest.raises(mgg.InputError):
        mgg.split_by_edges(mgg.gen_synthetic(mgg.UNIFORM, 10, 2, 0), 0)
    with pytest.raises(mgg.ConfigError):
        mgg.build_flat_plan(mgg.gen_synthetic(mgg.UNIFORM, 10, 2, 0), 1, 0, 33, 1, 1, 4)
    with pytest.raises(mgg.ConfigError):
        mgg.build_flat_plan(mgg.gen_synthetic(mgg.UNIFORM, 10, 2, 0), 1, 0, 4, 17, 1, 4)
    with pytest.raises(mgg.ConfigError):
        mgg.build_flat_plan(mgg.gen_synthetic(mgg.UNIFORM, 10, 2, 0), 1, 0, 4, 1, 17, 4)
    bad = tmp_path / "broken.json"
    bad.write_text("{not json")
    with pytest.raises(mgg.ParseError):
        mgg.resolve_profile(str(bad))
    with pytest.raises(mgg.ConfigError):
        mgg.resolve_profile("h100")


def test_no_cpu_fallback_without_gpu(mgg):
    if mgg.cuda_available():
        pytest.skip("GPU present")
    g = mgg.gen_synthetic(mgg.UNIFORM, 16, 2, 0)
    with pytest.raises(mgg.CudaError):
        mgg.Engine(g, 1, [0], mgg.make_gcn(4, 4, 2))


def test_same_process_barrier_has_no_host_sync():
    # the barrier between parts of one process (one device or
    # several) is stream-ordered (events), never a host join
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2209_06800_b200", "csrc", "cuda", "runtime.cu")).read()
    body = src[src.index("int mgg_barrier(mgg_ctx* ctx, mgg_store* flags) {"):]
    body = body[:body.index("\nint ", 10)]
    for bad in ("Synchronize", "cudaDeviceSynchronize", "cudaEventQuery"):
        assert bad not in body, bad
    assert "cudaStreamWaitEvent" in body
    cap = src[src.index("int mgg_capture_begin("):]
    cap = cap[:cap.index("\nint ", 10)]
    assert "single_device" not in cap  # multi-device contexts capture too
