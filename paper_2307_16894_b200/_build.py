"""In-tree build of the sm_100a CUDA library (and, for tests, the CPU oracle).

The product library ``libpodecm_cuda.so`` is compiled with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` (tcgen05-era features need the
``a`` target; plain ``-arch=sm_100a`` would embed compute_100 PTX).  All
device code is compiled with ``--fmad=false`` so the material arithmetic keeps
the reference's un-contracted evaluation order; kernels that want fused
multiply-adds (the DMMA/DFMA contractions) call ``fma()`` explicitly.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpodecm_cuda.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "liboracle.so"

CU_SOURCES = ["k_material.cu", "rve_host.cu", "k_assemble.cu", "k_rom.cu", "k_pod.cu", "k_ecm.cu",
              "k_probe.cu", "k_fe.cu", "twoscale.cu", "store.cpp"]
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nvcc_flags() -> list[str]:
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
        "-ccbin", HOST_CXX,
        "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
        "-Xptxas", "-v",
        *os.environ.get("PODECM_NVCC_DEFS", "").split(),  # A/B builds, e.g. -DPODECM_Q2_UNI=0
    ]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_product(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in CU_SOURCES if (CSRC / s).exists()]
    deps = srcs + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "podecm_cuda.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    logs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        cmd = [_nvcc(), *nvcc_flags(), "-c", str(s), "-o", str(o)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s.name}:\n{r.stderr}")
        objs.append(str(o))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-ccbin", HOST_CXX,
           "-o", str(tmp), *objs, "-lcudart", "-lcusolver", "-lcusparse"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    (ROOT / "build" / "ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(l for l in "\n".join(logs).splitlines() if "registers" in l or "spill" in l))
    return LIB


def build_oracle(force: bool = False) -> Path:
    """Checker only (tests / bench cpu_baseline); never linked by the product."""
    args = ["make", "-C", str(ORACLE_DIR), "-s"]
    if force:
        subprocess.run(["make", "-C", str(ORACLE_DIR), "clean", "-s"], check=True)
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    # oracle/_ref: the reference's own sources compiled unchanged (only where
    # /root/reference exists, i.e. in the build container; the GPU box uses the
    # prebuilt .so files that travel with the snapshot)
    ref_src = Path(os.environ.get("PODECM_REF", "/root/reference/proj"))
    if (ref_src / "src" / "material.cpp").exists():
        rargs = ["make", "-C", str(ORACLE_DIR / "ref"), "-s", f"REF={ref_src}"]
        if force:
            subprocess.run(["make", "-C", str(ORACLE_DIR / "ref"), "clean", "-s"], check=True)
        r = subprocess.run(rargs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"oracle/_ref build failed:\n{r.stdout}\n{r.stderr}")
    return ORACLE_LIB


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_product(force=force, verbose=True))
    print(build_oracle(force=force))
