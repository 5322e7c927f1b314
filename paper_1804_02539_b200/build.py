"""Build the native libraries in-tree.

  paper_1804_02539_b200/lib/libpmg_host.so  hierarchy builder (g++)
  paper_1804_02539_b200/lib/libpmg_cuda.so  sm_100a kernels + C ABI (nvcc)
  oracle/_build/liboracle.so                CPU parity oracle (g++), test-only

The .so files are git-ignored but travel to the GPU box with the snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "lib"
ORACLE_BUILD = ROOT / "oracle" / "_build"

HOST_SRC = sorted((PKG / "csrc" / "host").glob("*.cpp"))
# numerics.cpp (quadrature, B-spline evaluation) is shared with the host
# builder: device assembly tabulates its univariate tables with it
CUDA_SRC = sorted((PKG / "csrc" / "cuda").glob("*.cu")) + [PKG / "csrc" / "host" / "numerics.cpp"]
ORACLE_SRC = [ROOT / "oracle" / "oracle.cpp"]

CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-ffp-contract=off", "-Wall"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCCFLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills",
    # host code (numerics.cpp) rounds exactly as in libpmg_host
    "-Xcompiler", "-ffp-contract=off",
    "-I" + str(ROOT / "include"),
]


def _stale(out: Path, srcs) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    deps = list(srcs)
    for d in (PKG / "csrc", ROOT / "include", ROOT / "oracle"):
        deps += list(d.rglob("*.h")) + list(d.rglob("*.hpp")) + list(d.rglob("*.cuh"))
    return any(Path(s).stat().st_mtime > t for s in deps)


def _run(cmd):
    print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_host(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libpmg_host.so"
    if force or _stale(out, HOST_SRC):
        _run(["g++", *CXXFLAGS, "-o", out, *HOST_SRC])
    return out


def build_oracle(force: bool = False) -> Path:
    ORACLE_BUILD.mkdir(parents=True, exist_ok=True)
    out = ORACLE_BUILD / "liboracle.so"
    if force or _stale(out, ORACLE_SRC):
        _run(["g++", *CXXFLAGS, "-o", out, *ORACLE_SRC])
    return out


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libpmg_cuda.so"
    if CUDA_SRC and (force or _stale(out, CUDA_SRC)):
        _run([NVCC, *NVCCFLAGS, "-o", out, *CUDA_SRC, "-ldl"])
    return out


def build_example(force: bool = False) -> Path:
    """C++ driver of include/patchmg_gpu.hpp (the Backend-concept mirror)."""
    host, cuda = build_host(force), build_cuda(force)
    src = PKG / "csrc" / "examples" / "pcg_cpp.cpp"
    out = LIB / "pcg_cpp"
    if force or _stale(out, [src, host, cuda]):
        _run(["g++", "-O2", "-std=c++17", "-I" + str(ROOT / "include"), "-o", out, src, "-L" + str(LIB),
              "-lpmg_cuda", "-lpmg_host", "-Wl,-rpath,$ORIGIN", "-pthread"])
    return out


REF_INCLUDE = Path("/root/reference/proj/include")
REF_TEMPLATES = ROOT / "oracle" / "_ref" / "pcg_ref_templates"


def build_ref_templates(force: bool = False):
    """oracle/_ref/pcg_ref_templates: the reference's own multigrid.hpp
    templates over the GPU backend (oracle/ref_templates/build.sh).  Built only
    where the reference tree exists (this container); the binary travels to the
    GPU box.  Returns the path, or None when the reference is absent."""
    if not (REF_INCLUDE / "patchmg" / "multigrid.hpp").exists():
        return REF_TEMPLATES if REF_TEMPLATES.exists() else None
    host, cuda = build_host(force), build_cuda(force)
    src = ROOT / "oracle" / "ref_templates"
    deps = list(src.rglob("*")) + [host, cuda, ROOT / "include" / "patchmg_gpu.hpp",
                                   ROOT / "include" / "patchmg_gpu_reference.hpp"]
    if force or not REF_TEMPLATES.exists() or any(
            d.is_file() and d.stat().st_mtime > REF_TEMPLATES.stat().st_mtime for d in deps):
        _run(["bash", src / "build.sh"])
    return REF_TEMPLATES


def build_all(force: bool = False) -> None:
    build_host(force)
    build_oracle(force)
    build_cuda(force)
    build_example(force)
    build_ref_templates(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
