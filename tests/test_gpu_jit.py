"""JIT-specialized fusion on the device (-m gpu): with the JIT
synchronous (every fused struct-for group launches its NVRTC-specialized
kernel), results match the oracle at the same bars as the interpreter: masks
and lists exact, i32 fields exact, f32 within 1e-5 of the shadow magnitude."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402
from test_gpu_parity import compare  # noqa: E402


@pytest.fixture(autouse=True)
def jit_sync():
    sg.jit_set_mode(2)
    if sg.jit_info()["mode"] != 2:
        pytest.skip("NVRTC unavailable")
    yield
    sg.jit_set_mode(-1)


@pytest.mark.parametrize("prog_fn", [
    lambda: W.c1_program(steps=2), lambda: W.c1_program(steps=2, dtype="i32"),
    lambda: W.c1_program(steps=2, disk=False), lambda: W.c2_small_program(iters=4),
    lambda: W.mg_program(n=64, levels=3, block=8, cycles=1, radius_frac=0.3),
    lambda: W.c3_program(n_grid=32, n_particles=2000, steps=1, seed=5, v_scale=1.0, lo=0.2, hi=0.7),
], ids=["c1", "c1_i32", "c1_random", "c2_small", "mg", "c3"])
def test_jit_matches_oracle(prog_fn):
    prog = prog_fn()
    before = sg.jit_info()
    g, st = sg.run_program(prog)
    o = oracle.run_program(prog)
    if "levels" in prog:
        from test_gpu_mg import compare as mg_compare
        mg_compare(g, o, prog)
    elif prog["name"] == "C3":
        from test_gpu_mpm import compare_mpm
        compare_mpm(g, g.tensors, o, prog)
    else:
        compare(g, o, prog)
    after = sg.jit_info()
    assert after["ready"] > 0 and after["hits"] > before["hits"], after
    assert after["failed"] == 0, after


@pytest.mark.parametrize("seed", range(6))
def test_jit_fuzz(seed):
    prog = W.fuzz_program(seed)
    o = oracle.run_program(prog)
    g, _ = sg.run_program(prog, passes="all", debug=True)
    compare(g, o, prog)
    assert sg.jit_info()["failed"] == 0


def test_c2_full_size_jit():
    """The bench's C2 solve with specialized kernels for the fused fills and the
    final JACOBI+REDUCE group: s within 1e-5 of the interpreter's."""
    prog = W.c2_program()
    g, st = sg.run_program(prog)
    s_jit = float(g.field(prog["layout"].fields["s"]))
    sg.jit_set_mode(0)
    g2, _ = sg.run_program(prog)
    s_int = float(g2.field(prog["layout"].fields["s"]))
    assert s_jit == pytest.approx(s_int, rel=1e-5)


_EXIT_CHILD = r"""
import os, sys
sys.path.insert(0, {root!r})
import workloads as W
from paper_2012_08141_b200 import sg
sg.jit_set_mode(1)                       # asynchronous: compiles run in worker threads
prog = W.mg_program(n=64, levels=3, block=8, cycles=1, radius_frac=0.3)
g, _ = sg.run_program(prog)              # submits every fused group's kernel for compilation
print("compiling", sg.jit_info()["compiling"], flush=True)
"""   # ... and the interpreter exits right away, compiles still in flight


def test_process_exit_with_compiles_in_flight():
    """Exit while NVRTC worker threads are compiling must not crash: NVRTC's
    exit-time teardown under a running compile segfaulted a 2-process test;
    the binding's atexit hook (sg_jit_shutdown) drains the workers first."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for _ in range(3):
        r = subprocess.run([sys.executable, "-c", _EXIT_CHILD.format(root=root)], capture_output=True, text=True,
                           timeout=300, env=dict(os.environ, SG_JIT="1"))
        assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
        assert "compiling" in r.stdout
