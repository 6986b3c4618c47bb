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
    dump = tmp_path / "assembly.bin"
    r = subprocess.run([str(exe), str(dump)], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    # the C++ consumer's assembly (16x16 cell, a = 0.3, b = 0.2, Fbar, zero
    # fluctuation, virgin history) against the oracle on the same inputs
    import numpy as np

    import oracle
    from paper_2307_16894_b200 import api
    raw = np.fromfile(dump, dtype=np.float64)
    nr, nnz = raw[:2].view(np.int64)
    f, K = raw[2:2 + nr], raw[2 + nr:2 + nr + nnz]
    mats = [api.matrix_params(), api.inclusion_params()]
    assert (mats[0].E, mats[0].nu, mats[0].sigma_y0, mats[0].H) == (1.0, 0.3, 0.01, 0.1)
    assert (mats[1].E, mats[1].nu, mats[1].sigma_y0, mats[1].H) == (10.0, 0.3, 1e300, 0.0)
    o = oracle.Rve(16, mats)
    nq = o.n_qp
    st0 = np.zeros((1, 6, nq))
    st0[0, 0] = st0[0, 3] = st0[0, 4] = 1.0
    ro = o.assemble(np.array([[0.3, 0.2]]), np.array([[1.02, 0.01, 0.0, 0.99]]), np.zeros((1, o.n_red)), st0)
    ef = np.linalg.norm(f - ro["f"][0]) / np.linalg.norm(ro["f"][0])
    eK = np.linalg.norm(K - ro["K"][0]) / np.linalg.norm(ro["K"][0])
    print(f"C++ consumer assembly vs oracle: f {ef:.2e}, K {eK:.2e}")
    assert ef <= 1e-10 and eK <= 1e-9
