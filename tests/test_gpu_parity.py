"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the CPU oracle.

Bar (BASELINE.json north_star): masks and lists bit-exact as sorted sets,
integer fields bit-exact, float fields within 1e-5 relative to the shadow
magnitude M the oracle carries (|g - o| <= 1e-5 * max(|o|, M), DESIGN.md
reading R15).  Every program is replayed both unoptimized (passes=0, one
launch per lowered task) and optimized (all passes), which is also the T3
soundness check on the device ("transparent to users").
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402

TOL = 1e-5


def as_set(a):
    return sorted(map(tuple, np.asarray(a).tolist()))


def assert_field_close(got, want, mag, dtype, what=""):
    if dtype == "i32":
        np.testing.assert_array_equal(got, want.astype(np.int64), err_msg=what)
        return
    bound = TOL * np.maximum(np.abs(want), mag)
    err = np.abs(got.astype(np.float64) - want)
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} elements off, worst {err[bad].max()} at {np.argwhere(bad)[:3]}"


def compare(g, o, prog):
    L = prog["layout"]
    for name, fid in L.fields.items():
        want, mag = o.field(fid, with_mag=True)
        assert_field_close(g.field(fid), want, mag, L.field_dtype[name], f"field {name}")
    for s in range(1, len(L.rows)):
        if L.rows[s][0] in (W.BITMASKED, W.POINTER):
            assert as_set(g.mask(s)) == as_set(o.mask(s)), f"mask of snode {s}"


@pytest.mark.parametrize("passes", [0, "all"])
@pytest.mark.parametrize("dtype", ["f32", "i32"])
@pytest.mark.parametrize("disk", [True, False])
def test_c1(passes, dtype, disk):
    prog = W.c1_program(steps=2, disk=disk, dtype=dtype)
    g, st = sg.run_program(prog, passes=passes)
    o = oracle.run_program(prog)
    compare(g, o, prog)
    if disk:
        assert float(g.field(prog["layout"].fields["s"])) == -192.0
    assert st[0]["launches"] == (8 if passes == 0 else 5)


@pytest.mark.parametrize("passes", [0, "all", "all+chain"])
def test_c2_small(passes):
    prog = W.c2_small_program(iters=6)
    g, st = sg.run_program(prog, passes=passes)
    o = oracle.run_program(prog)
    compare(g, o, prog)


def test_c2_small_lists_and_fig_counts():
    prog = W.c2_small_program(iters=2)
    L = prog["layout"]
    lv = [s for s in range(1, len(L.rows)) if L.rows[s][0] in (W.BITMASKED, W.POINTER)]
    g, _ = sg.run_program(prog)
    o = oracle.run_program(prog)
    for s in lv:
        g.listgen(s)
        o.call(W.listgen(s))
        assert as_set(g.list(s)) == as_set(o.list(s)), s


@pytest.mark.parametrize("seed", range(80))
def test_fuzz_programs(seed):
    prog = W.fuzz_program(seed)
    o = oracle.run_program(prog)
    for passes in (0, "all", "listgen+demotion", "fusion+dse", "all+chain"):
        g, _ = sg.run_program(prog, passes=passes, debug=True)
        compare(g, o, prog)
        g.close()


def test_fig3_activation_on_write():
    L = W.Layout()
    xl = L.chain([("pointer", (4,)), ("dense", (2,))], [("x", "i32")])
    yl = L.chain([("pointer", (2,)), ("dense", (2,))], [("y", "i32")])
    calls = [W.activate(0, np.array([[2], [6]], dtype=np.int32)),
             W.struct_for("DOWNSAMPLE", xl[-1], [1, -1], [0.0, 1.0], [True]), W.flush()]
    prog = W.program(L, calls)
    g, _ = sg.run_program(prog)
    assert g.field(1).tolist() == [0, 2, 0, 2]
    assert as_set(g.mask(yl[0])) == [(0,), (1,)]


def test_listgen_random_masks_deep():
    for seed in range(20):
        rng = np.random.default_rng(100 + seed)
        L, main, half = W.fuzz_layout(rng)
        shape = L.shape("a")
        k = int(rng.integers(1, 40))
        cells = np.stack([rng.integers(0, s, size=k) for s in shape], axis=1).astype(np.int32)
        sparse = [s for s in main if L.rows[s][0] in (W.BITMASKED, W.POINTER)]
        if not sparse:
            continue
        calls = [W.activate(0, cells), W.listgen(sparse[-1]), W.flush()]
        prog = W.program(L, calls)
        g, _ = sg.run_program(prog)
        o = oracle.run_program(prog)
        assert as_set(g.list(sparse[-1])) == as_set(o.list(sparse[-1])), seed


def test_debug_trap_and_pool_exhaustion():
    L = W.Layout()
    xl = L.chain([("pointer", (4,)), ("dense", (2,))], [("x", "i32")])
    yl = L.chain([("pointer", (2,)), ("dense", (2,))], [("y", "i32")])
    g = sg.Grid(L.desc(), debug=True)
    c = torch.tensor([[2]], dtype=torch.int32, device="cuda")
    g.activate(0, c)
    g.struct_for("DOWNSAMPLE", xl[-1], [1, -1], [0.0, 1.0], [False])
    g.flush(0)
    with pytest.raises(sg.SgError) as e:
        g.sync()
    assert e.value.kind == "DEMOTION_TRAP"
    g2 = sg.Grid(L.desc(), pool_capacity=1)
    g2.activate(0, torch.tensor([[0], [7]], dtype=torch.int32, device="cuda"))
    g2.flush()
    with pytest.raises(sg.SgError) as e:
        g2.sync()
    assert e.value.kind == "POOL_EXHAUSTED"


def test_c2_full_size_properties():
    """BASELINE configs[1] at full size (256^3, 50 iterations), in the launch
    configuration bench.py times: properties that hold at any size."""
    prog = W.c2_program()
    L = prog["layout"]
    f = L.fields
    g, st = sg.run_program(prog)
    assert (st[0]["tasks_lowered"], st[0]["launches"]) == (161, 55)
    coords = W.block_ball_coords(32, 8, 68.0)
    lv = [s for s in range(1, len(L.rows)) if L.rows[s][0] == W.BITMASKED][0]
    blocks = as_set(coords // 8)
    assert as_set(g.mask(lv)) == blocks                            # exactly the activated blocks
    g.listgen(lv)
    assert as_set(g.list(lv)) == blocks
    x = g.field(f["x0"])                                          # 50 iterations: result in x0
    act = np.zeros((256,) * 3, dtype=bool)
    for c in coords:
        act[c[0]:c[0] + 8, c[1]:c[1] + 8, c[2]:c[2] + 8] = True
    assert (x[~act] == 0).all() and (x[act] > 0).all()
    assert x.max() <= 50 / 6 + 1e-4                                # max principle: +1/6 per iteration
    # block-ball symmetric under axis reflections about the centre
    for ax in range(3):
        np.testing.assert_allclose(x, np.flip(x, ax), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(x, np.transpose(x, (1, 0, 2)), rtol=1e-5, atol=1e-6)
    s = float(g.field(f["s"]))
    np.testing.assert_allclose(s, x.astype(np.float64).sum(), rtol=1e-5)
    # exact oracle parity at full size for one iteration (what the oracle can
    # finish in seconds), same kernels and launch configuration
    L1, lv1 = W.c2_layout()
    calls, _ = W.c2_solve_calls(L1, lv1, coords, iters=1)
    prog1 = W.program(L1, calls + [W.flush()])
    g1, _ = sg.run_program(prog1)
    o1 = oracle.run_program(prog1)
    for name in ("x1", "s"):
        want, mag = o1.field(L1.fields[name], with_mag=True)
        assert_field_close(g1.field(L1.fields[name]), want, mag, "f32", f"C2 full size, 1 iteration, {name}")


@pytest.mark.parametrize("iters", [2, 3])
def test_c2_full_size_unfused_jacobi(iters):
    """BASELINE configs[1] at full size (256^3, 3,280 8^3 blocks): `iters`
    JACOBI sweeps with no reduction after them, so every sweep is a lone JACOBI
    group and runs in k_jacobi8 -- the bench's dominant kernel, in the launch
    configuration bench.py times (grid-stride over 6,560 half blocks, the
    block-table path) -- compared element by element with the oracle at 1e-5."""
    coords = W.block_ball_coords(32, 8, 68.0)
    L, lv = W.c2_layout()
    calls, _ = W.c2_solve_calls(L, lv, coords, iters=iters, reduce_result=False)
    prog = W.program(L, calls + [W.flush()])
    g, st = sg.run_program(prog)
    o = oracle.run_program(prog)
    for name in ("x0", "x1", "b"):
        want, mag = o.field(L.fields[name], with_mag=True)
        assert_field_close(g.field(L.fields[name]), want, mag, "f32", f"C2 full size, {iters} sweeps, {name}")
    assert st[0]["launches"] == 4 + iters   # activate, 2 listgens, FILL b + FILL x0, the sweeps


_FLOW_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import workloads as W
from paper_2012_08141_b200 import sg
iters, reduce = {iters}, {reduce}
coords = W.block_ball_coords(32, 8, 68.0)
L, lv = W.c2_layout()
calls, _ = W.c2_solve_calls(L, lv, coords, iters=iters, reduce_result=reduce)
prog = W.program(L, calls + [W.flush()])
g, st = sg.run_program(prog, passes="all+chain")
np.savez({out!r}, **{{n: np.asarray(g.field(L.fields[n])) for n in ("x0", "x1", "s")}})
print(json.dumps({{"launches": st[0]["launches"], "chained": st[0]["launches_chained"]}}))
"""


@pytest.mark.parametrize("iters,reduce", [(3, False), (50, True)])
def test_c2_full_size_flag_chain(iters, reduce, tmp_path):
    """N2 (SG_PASS_CHAIN, opt-in SG_FLOW=1): the C2 solve's JACOBI sweeps as ONE
    persistent launch with per-half-block completion flags (kernels_flow.cu),
    run in a child process with SG_FLOW=1.  Same arithmetic per cell as one
    launch per sweep, so the fields equal the unchained plan's bit for bit
    (and the oracle's within 1e-5 for the 3-sweep case); the 50-sweep solve
    ends with the fused reduction, as bench.py times it."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "flow.npz")
    code = _FLOW_CHILD.format(root=root, iters=iters, reduce=reduce, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SG_FLOW="1"), capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    st1 = json.loads(r.stdout.strip().splitlines()[-1])
    flow = np.load(out)
    coords = W.block_ball_coords(32, 8, 68.0)
    L, lv = W.c2_layout()
    calls, _ = W.c2_solve_calls(L, lv, coords, iters=iters, reduce_result=reduce)
    prog = W.program(L, calls + [W.flush()])
    g0, st0 = sg.run_program(prog, passes="all")
    assert st1["chained"] == 1 and st1["launches"] < st0[0]["launches"], (st0[0], st1)
    names = ("x0", "x1", "s") if reduce else ("x0", "x1")
    for name in names:
        np.testing.assert_array_equal(flow[name], np.asarray(g0.field(L.fields[name])), err_msg=name)
    if not reduce:
        o = oracle.run_program(prog)
        for name in names:
            want, mag = o.field(L.fields[name], with_mag=True)
            assert_field_close(flow[name], want, mag, "f32", f"C2 flag chain, {iters} sweeps, {name}")


_T2_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import workloads as W
from paper_2012_08141_b200 import sg
iters, reduce = {iters}, {reduce}
coords = W.block_ball_coords(32, 8, 68.0)
L, lv = W.c2_layout()
calls, _ = W.c2_solve_calls(L, lv, coords, iters=iters, reduce_result=reduce)
prog = W.program(L, calls + [W.flush()])
g, st = sg.Grid(prog["desc"]), []
res = []
for _ in range(3):   # the second flush is captured as a CUDA graph, the third replays it
    st = sg.replay(g, prog, passes="all+chain", device="cuda")
    g.sync()
    res.append({{n: np.asarray(g.field(L.fields[n])) for n in ("x0", "x1", "s")}})
np.savez({out!r}, **{{f"{{n}}_{{i}}": r[n] for i, r in enumerate(res) for n in r}})
print(json.dumps({{"launches": st[0]["launches"], "chained": st[0]["launches_chained"]}}))
"""


@pytest.mark.parametrize("iters,reduce", [(4, False), (7, False), (50, True)])
def test_c2_full_size_two_sweep_chain(iters, reduce, tmp_path):
    """N2 (SG_PASS_CHAIN, opt-in SG_T2=1, run in a child process): the C2
    solve's JACOBI sweeps two per launch (temporal blocking with a scratch
    field, kernels_flow.cu): each cell sees the same float operations in the
    same order as one launch per sweep, so both ping-pong fields equal the
    unchained plan's bit for bit, on the first flush, the captured second and
    the replayed third; the fused reduction sums in another order (1e-6).
    7 sweeps: 3 single launches + one A/B cycle; 50: 2 singles + 12 cycles."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "t2.npz")
    code = _T2_CHILD.format(root=root, iters=iters, reduce=reduce, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SG_T2="1"), capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    st1 = json.loads(r.stdout.strip().splitlines()[-1])
    t2 = np.load(out)
    coords = W.block_ball_coords(32, 8, 68.0)
    L, lv = W.c2_layout()
    calls, _ = W.c2_solve_calls(L, lv, coords, iters=iters, reduce_result=reduce)
    prog = W.program(L, calls + [W.flush()])
    g0, st0 = sg.run_program(prog, passes="all")
    assert st1["chained"] == 1 and st1["launches"] <= st0[0]["launches"], (st0[0], st1)
    for i in range(3):
        for name in ("x0", "x1"):
            np.testing.assert_array_equal(t2[f"{name}_{i}"], np.asarray(g0.field(L.fields[name])),
                                          err_msg=f"flush {i}: {name}")
        if reduce:
            a, b = float(t2[f"s_{i}"]), float(g0.field(L.fields["s"]))
            assert abs(a - b) <= 1e-6 * abs(b), (i, a, b)
