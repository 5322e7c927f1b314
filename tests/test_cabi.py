"""The C ABI boundary: every entry point declared in include/*.h is exported by
the built libraries, the CUDA library loads without a GPU, and the product
path fails loudly (no CPU fallback) when the CUDA library is missing."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1804_02539_b200 import _native as N
from paper_1804_02539_b200 import build

ROOT = Path(__file__).resolve().parents[1]


def declared(header: str):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pmgh?_[a-z0-9_]+)\s*\(", text)))


def exported(lib: Path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_host_library_exports_its_header():
    lib = build.build_host()
    names = declared("pmg_host.h")
    assert len(names) >= 10
    missing = [n for n in names if n not in exported(lib)]
    assert not missing, missing


def test_cuda_library_exports_its_header():
    lib = build.build_cuda()
    names = declared("pmg_cuda.h")
    assert len(names) >= 25
    missing = [n for n in names if n not in exported(lib)]
    assert not missing, missing
    # it loads on a CPU-only host (cudart is linked statically)
    C.CDLL(str(lib))
    assert set(names) <= set(N.CUDA_SYMBOLS) | {"pmg_profile", "pmg_profile_read"}


def test_cuda_library_is_sm100a():
    lib = build.build_cuda()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    assert "DMMA" in sass      # fast diagonalization on FP64 tensor cores
    assert "UBLKCP" in sass    # TMA bulk copies in the band SpMV


def test_ctx_create_without_gpu_reports_cuda_error():
    lib = N.cuda_lib()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1804_02539_b200 import Hierarchy
    h = Hierarchy("lshape", 2, 1, n0=1)
    ctx = C.c_void_p()
    rc = lib.pmg_ctx_create(C.byref(h.desc), 0, None, C.byref(ctx))
    assert rc == N.PMG_ERR_CUDA
    assert lib.pmg_last_error(None)


def test_missing_cuda_library_is_an_error(monkeypatch, tmp_path):
    monkeypatch.setattr(N, "LIB_DIR", tmp_path)
    monkeypatch.setattr(N, "_cuda", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        N.cuda_lib()
