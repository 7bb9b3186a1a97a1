"""JIT-specialized fusion, host side (-m "not gpu"): the
specialized kernels of representative fused groups NVRTC-compile for sm_100a
from the library's embedded device headers on a host without a GPU (the GPU
tests run them against the oracle)."""
import pytest

from paper_2012_08141_b200 import sg


@pytest.mark.parametrize("ops,nd,gl", [
    (["JACOBI", "REDUCE_SUM"], 3, 1),            # C2 / SF-XL: Jacobi + reduction
    (["FILL", "FILL"], 3, 1),                    # C2's fused fills
    (["STENCIL", "REDUCE_SUM"], 2, 3),           # C1 STENCIL + REDUCE on 4x4 blocks
    (["GRID_OP"], 3, 2),                         # MPM grid op on 4^3 blocks
    (["SMOOTH_RB", "RESID_NORM2"], 2, 0),        # multigrid, runtime geometry
    (["INC", "INC", "ADD_CONST"], 0, 0),          # generic cell path
])
def test_specialized_kernel_compiles(ops, nd, gl):
    ok, log = sg.jit_selftest(ops, nd=nd, gl=gl)
    if not ok and "not found" in log:
        pytest.skip(log)
    assert ok, log


def test_i32_group_compiles():
    ok, log = sg.jit_selftest(["FILL", "STENCIL"], nd=2, gl=3, i32=True)
    if not ok and "not found" in log:
        pytest.skip(log)
    assert ok, log
