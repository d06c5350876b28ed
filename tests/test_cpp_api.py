"""Builds tests/cpp/test_host_api.cpp against the C++ host API (include/mgg)
and libmgg.so, and runs it (CPU only)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def test_cpp_host_api(tmp_path):
    exe = tmp_path / "test_host_api"
    lib_dir = os.path.join(ROOT, "paper_2209_06800_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", JSON_INC,
           os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp"), "-L", lib_dir, "-lmgg",
           f"-Wl,-rpath,{lib_dir}", "-pthread", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
