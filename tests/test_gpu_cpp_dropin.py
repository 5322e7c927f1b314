"""The C++ drop-in: the reference's templates (pcg_generic / mg_precondition,
restated in include/patchmg_gpu.hpp against the Backend concept) drive
GpuBackend through the C ABI from a compiled C++ program; the result must
match the fused device solve and the CPU oracle."""
import json
import subprocess

import numpy as np
import pytest

import oracle
from paper_1804_02539_b200 import Hierarchy, build

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("args", [("lshape", 2, 3, 1), ("c4", 3, 2, 2)])
def test_cpp_templates_over_c_abi(args):
    exe = build.build_example()
    out = subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["template_iterations"] == res["fused_iterations"]
    assert res["max_rel_diff"] < 1e-10
    dom, p, lv, n0 = args
    h = Hierarchy(dom, p, lv, n0=n0)
    u_ref, hist, _, _ = oracle.Oracle(h).pcg_solve(h.rhs())
    assert res["template_iterations"] == len(hist) - 1
    k = len(res["u"])
    assert np.abs(np.array(res["u"]) - u_ref[:k]).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("args", [("lshape", 2, 3, 1), ("c4", 3, 2, 2), ("c2", 4, 4, 2)])
def test_reference_templates_drive_the_gpu_backend(args):
    """The reference's OWN templates -- patchmg::pcg_generic / mg_precondition /
    mg_cycle_generic from /root/reference/proj/include/patchmg/multigrid.hpp,
    compiled unchanged into oracle/_ref/pcg_ref_templates -- over
    patchmg_gpu::ReferenceGpuBackend (params() is a const patchmg::CycleParams&,
    errors are patchmg:: exceptions).  The result matches the fused device
    solve and the oracle, and the backend raises the reference's exception
    classes."""
    exe = build.build_ref_templates()
    if exe is None or not exe.exists():
        pytest.fail("oracle/_ref/pcg_ref_templates was not built (build it where /root/reference exists)")
    out = subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["template_iterations"] == res["fused_iterations"]
    assert res["max_rel_diff"] < 1e-10 and res["history_head_max_rel_diff"] < 1e-10
    assert res["domain_error"] and res["divergence_error"]
    dom, p, lv, n0 = args
    h = Hierarchy(dom, p, lv, n0=n0)
    u_ref, hist, _, _ = oracle.Oracle(h).pcg_solve(h.rhs())
    assert res["template_iterations"] == len(hist) - 1
    k = len(res["u"])
    assert np.abs(np.array(res["u"]) - u_ref[:k]).max() <= 1e-10 * np.abs(u_ref).max()
