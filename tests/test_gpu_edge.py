"""Edge cases of the GPU path against the oracle (-m gpu): empty inputs,
empty trees, degenerate particle positions, whole-tree resets, repeated flushes
(plan cache + CUDA-graph replay) and the warp-aggregated activation of dense
coordinate runs."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402
from test_gpu_parity import as_set  # noqa: E402


def run_both(prog):
    o = oracle.run_program(prog)
    g = sg.Grid(prog["desc"])
    st = sg.replay(g, prog, device="cuda")
    g.sync()
    return g, o, st


def test_empty_activation_and_empty_tree():
    """No active cell anywhere: listgen gives empty lists, struct-fors and the
    reduction do nothing (s stays 0), deactivate of an empty tree is a no-op."""
    L, lv = W.c1_layout()
    f = L.fields
    calls = [W.activate(f["x"], np.zeros((0, 2), np.int32)),
             W.struct_for("FILL", lv[-1], [f["x"]], [1.0]),
             W.struct_for("STENCIL", lv[-1], [f["y"], f["x"]]),
             W.serial("CLEAR_SCALAR", [f["s"]]),
             W.struct_for("REDUCE_SUM", lv[-1], [f["s"], f["y"]]),
             W.deactivate(lv[0]), W.flush()]
    g, o, st = run_both(W.program(L, calls))
    assert float(g.field(f["s"])) == float(o.field(f["s"])) == 0.0
    for s in lv:
        assert as_set(g.mask(s)) == as_set(o.mask(s)) and len(as_set(o.mask(s))) == 0


def test_zero_particles_mpm_step():
    """A range-for over 0 particles (P2G/G2P) is a no-op; the grid stays empty."""
    prog = W.c3_program(n_grid=32, n_particles=0, steps=1)
    g, o, st = run_both(prog)
    L = prog["layout"]
    assert as_set(g.mask(1)) == as_set(o.mask(1)) and len(as_set(o.mask(1))) == 0


def test_particles_on_cell_faces():
    """Particles exactly on node-aligned positions (x/dx - 1/2 integral: the
    third B-spline weight is exactly 0) -- the stencil still activates every
    block the oracle activates and the transfers agree."""
    n_grid, n = 32, 1000
    rng = np.random.default_rng(4)
    cells = rng.integers(8, 24, size=(3, n))
    x = ((cells + 0.5) / n_grid).astype(np.float32)   # X - 0.5 integral, fx = 0.5 exactly
    parts = W.mpm_particles(n, seed=4, v_scale=0.5)
    parts["x"] = x
    L, lv = W.c3_layout(n_grid)
    prm = W.mpm_params(n_grid)
    prog = W.program(L, W.c3_step_calls(L, lv, n, prm) + [W.flush()], arrays=parts)
    g, o, st = run_both(prog)
    for s in lv:
        if L.rows[s][0] in (W.BITMASKED, W.POINTER):
            assert as_set(g.mask(s)) == as_set(o.mask(s)), s
    want, mag = o.field(L.fields["m"], with_mag=True)
    got = np.asarray(g.field(L.fields["m"]), dtype=np.float64)
    assert (np.abs(got - want) <= 1e-5 * np.maximum(np.abs(want), mag)).all()
    wx, mx = o.array(0, with_mag=True)
    gx = g.tensors["x"].cpu().numpy().astype(np.float64)
    assert (np.abs(gx - wx) <= 1e-5 * np.maximum(np.abs(wx), mx)).all()


def test_dense_coordinate_runs_activate_like_the_oracle():
    """Whole 4x4 bitmasked blocks activated with many lanes per mask word
    (the warp-aggregated atomicOr path), including duplicate coordinates."""
    L, lv = W.c1_layout()
    f = L.fields
    xs, ys = np.meshgrid(np.arange(16, 48), np.arange(8, 40), indexing="ij")
    co = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.int32)
    co = np.concatenate([co, co[::7]])                   # duplicates
    calls = [W.activate(f["x"], co), W.struct_for("FILL", lv[-1], [f["x"]], [2.0]),
             W.serial("CLEAR_SCALAR", [f["s"]]), W.struct_for("REDUCE_SUM", lv[-1], [f["s"], f["x"]]), W.flush()]
    g, o, st = run_both(W.program(L, calls))
    for s in lv:
        assert as_set(g.mask(s)) == as_set(o.mask(s)), s
    assert float(g.field(f["s"])) == float(o.field(f["s"])) == 2.0 * 32 * 32


def test_repeated_flushes_replay_the_graph_identically():
    """The same C1 step flushed 6 times: plan-cache hits from the second flush
    on, CUDA-graph replay from the third; every flush's result equals the
    eager oracle's (x, y identical, s = -192)."""
    prog = W.c1_program(steps=6)
    g, o, st = run_both(prog)
    assert [s["plan_cache_hits"] for s in st] == [0, 1, 1, 1, 1, 1]
    f = prog["layout"].fields
    assert float(g.field(f["s"])) == float(o.field(f["s"])) == -192.0
    np.testing.assert_array_equal(g.field(f["y"]), o.field(f["y"]).astype(np.float32))


def test_reset_deactivate_then_reuse():
    """Pool-reset DEACTIVATE (R33) followed by re-activation of a different
    region: containers are reused from the reset pool and read 0."""
    n_grid = 32
    L, lv = W.c3_layout(n_grid)
    f = L.fields
    a = np.array([[0, 0, 0], [16, 16, 16], [28, 4, 8]], np.int32)
    b = np.array([[4, 4, 4], [20, 0, 12]], np.int32)
    calls = [W.activate(f["vx"], a), W.struct_for("FILL", lv[-1], [f["vx"]], [3.0]), W.flush(),
             W.deactivate(lv[0]), W.activate(f["m"], b), W.struct_for("INC", lv[-1], [f["m"]], [1.0]), W.flush()]
    g, o, st = run_both(W.program(L, calls))
    for s in lv:
        if L.rows[s][0] in (W.BITMASKED, W.POINTER):
            assert as_set(g.mask(s)) == as_set(o.mask(s)), s
    for name in ("vx", "m"):
        np.testing.assert_array_equal(g.field(f[name]), o.field(f[name]).astype(np.float32))


@pytest.mark.parametrize("seed", [0, 1])
def test_big_activation_batch_matches_oracle(seed):
    """A 1M-request activation batch (grid-strided k_activate, many requests per
    thread): masks and the leaf list bit-exact against the oracle, with
    duplicates, dense runs sharing mask words and out-of-order coordinates."""
    rng = np.random.default_rng(seed)
    L = W.Layout()
    lv = L.chain([("pointer", (16,) * 3), ("bitmasked", (16,) * 3)], [("m", "f32")])
    n = (1 << 20) + 12345
    cells = rng.integers(0, 256, size=(n, 3)).astype(np.int32)
    cells[: 4096] = np.stack(np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij"), -1).reshape(-1, 3)
    cells[-1000:] = cells[:1000]   # repeats in the same batch
    prog = W.program(L, [W.activate(0, cells), W.listgen(lv[-1]), W.flush()])
    g, _ = sg.run_program(prog)
    o = oracle.run_program(prog)
    for s_ in lv:
        if L.rows[s_][0] in (W.BITMASKED, W.POINTER):
            assert as_set(g.mask(s_)) == as_set(o.mask(s_))
    assert as_set(g.list(lv[-1])) == as_set(o.list(lv[-1]))
