"""The C-ABI consumed from C++ without Python/torch (tests/cpp/capi_smoke.cpp),
the way the reference would bind it."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_consumer(product_lib, tmp_path):
    exe = tmp_path / "capi_smoke"
    lib_dir = ROOT / "paper_2307_16894_b200"
    gxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
    subprocess.run([gxx, "-O2", "-std=c++17", str(ROOT / "tests" / "cpp" / "capi_smoke.cpp"), "-o", str(exe),
                    "-I/usr/local/cuda/include", f"-L{lib_dir}", "-lpodecm_cuda", "-L/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib_dir}", "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
