"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's
formula: they use the paper's worked examples (tests/golden/), closed forms
counted independently with numpy, a textbook routine (scipy sparse Jacobi),
a brute-force dense formulation (tests/brute.py) and invariants.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import workloads as W
from brute import run as brute_run

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def chain(L, levels, fields):
    return L.chain([(k, (e,)) for k, e in levels], fields)


# ---------------------------------------------------------------------------
# Worked examples
# ---------------------------------------------------------------------------
def test_fig2_layout_and_lists():
    g = golden("fig2_listgen.json")
    L = W.Layout()
    lv = chain(L, g["layout"], [("x", "f32")])
    assert L.shape("x") == (g["x_shape"],)
    o = oracle.Oracle(L.desc())
    assert o.field_shape(0) == (8,)
    o.activate(0, np.array(g["activate_cells"], dtype=np.int32)[:, None])
    o.listgen(lv[0])
    assert o.list(lv[0])[:, 0].tolist() == g["expect_pointer_list"]
    # a struct-for visits exactly the dense cells of the listed pointer cells
    o.struct_for_task("FILL", lv[1], [0], [7.0])
    x = o.field(0)
    assert np.flatnonzero(x == 7.0).tolist() == g["expect_active_cells"]


def test_layout_2d_shape():
    # SPEC.md:54 root->pointer(4x4)->dense(2x2)->place(y): y shape 8x8
    L = W.Layout()
    L.chain([("pointer", (4, 4)), ("dense", (2, 2))], [("y", "f32")])
    assert oracle.Oracle(L.desc()).field_shape(0) == (8, 8)


def test_fig3_activation_on_write():
    g = golden("fig3_activate_on_write.json")
    L = W.Layout()
    xl = chain(L, g["x_layout"], [("x", "i32")])
    yl = chain(L, g["y_layout"], [("y", "i32")])
    o = oracle.Oracle(L.desc())
    o.activate(0, np.array(g["x_active"], dtype=np.int32)[:, None])
    o.call(W.struct_for("DOWNSAMPLE", xl[-1], [1, -1], [0.0, 1.0], [True]))
    y = o.field(1)
    assert y.tolist() == g["expect_y_values"]
    assert o.mask(yl[0])[:, 0].tolist() == g["expect_y_pointer_cells"]
    # y[0] and y[2] are active (dense constraint): a struct-for over y visits them
    o.call(W.struct_for("INC", yl[-1], [1], [10.0]))
    y2 = o.field(1)
    assert sorted(np.flatnonzero(y2 >= 10).tolist()) == g["expect_y_active"]
    # each newly active pointer cell counted once by the allocator
    assert o.counters()["allocated"] == 2 + 2   # x pointer cells {1,3}, y pointer cells {0,1}


def test_activation_idempotent_and_zero_fill():
    # SPEC.md:92 idempotence; "zero-fill the initial data"
    L, lv = W.c1_layout("i32")
    o = oracle.Oracle(L.desc())
    c = W.c1_random_coords(3)
    o.activate(0, c)
    m1 = [o.mask(s).copy() for s in lv]
    a1 = o.counters()["allocated"]
    o.activate(0, c)
    assert all(np.array_equal(a, o.mask(s)) for a, s in zip(m1, lv))
    assert o.counters()["allocated"] == a1
    assert not o.field(0).any()           # newly active cells read 0
    assert a1 == len({(i // 4, j // 4) for i, j in c.tolist()})


def test_inactive_reads_zero_and_never_activate():
    # PAPER.md:195 "the inactive voxel has value 0"; reads never activate
    L, lv = W.c1_layout("i32")
    o = oracle.Oracle(L.desc())
    o.activate(0, np.array([[5, 5]], dtype=np.int32))
    o.call(W.struct_for("FILL", lv[-1], [0], [3]))
    o.call(W.struct_for("STENCIL", lv[-1], [1, 0]))   # reads 4 inactive neighbours
    assert o.field(1)[5, 5] == -12                  # 0*4 - 4*3
    assert len(o.mask(lv[-1])) == 1


def test_demotion_trap():
    # a non-activating write to an inactive cell is an error
    L = W.Layout()
    xl = chain(L, [["pointer", 4], ["dense", 2]], [("x", "i32")])
    yl = chain(L, [["pointer", 2], ["dense", 2]], [("y", "i32")])
    o = oracle.Oracle(L.desc())
    o.activate(0, np.array([[2]], dtype=np.int32))
    with pytest.raises(oracle.OracleError) as e:
        o.call(W.struct_for("DOWNSAMPLE", xl[-1], [1, -1], [0.0, 1.0], [False]))
    assert e.value.kind == "DEMOTION_TRAP"


def test_layout_errors():
    # SPEC.md:50 errors: non-power-of-two extent; place with children; axis mismatch
    bad = [
        [[0, -1, 0, 1, 1, 1, 0], [3, 0, 1, 3, 1, 1, 0], [4, 1, 1, 1, 1, 1, 0]],
        [[0, -1, 0, 1, 1, 1, 0], [1, 0, 1, 4, 1, 1, 0], [4, 1, 1, 1, 1, 1, 0], [1, 2, 1, 2, 1, 1, 0]],
        [[0, -1, 0, 1, 1, 1, 0], [1, 0, 2, 4, 4, 1, 0], [1, 1, 1, 2, 1, 1, 0], [4, 2, 1, 1, 1, 1, 0]],
    ]
    for d in bad:
        with pytest.raises(oracle.OracleError):
            oracle.Oracle(np.array(d, dtype=np.int32))


# ---------------------------------------------------------------------------
# Closed forms
# ---------------------------------------------------------------------------
def _boundary_faces(mask):
    """# of (active, inactive-or-outside) neighbour pairs, counted on a padded array."""
    m = np.pad(mask, 1)
    n = 0
    for ax in range(mask.ndim):
        a = np.take(m, range(1, m.shape[ax]), axis=ax)
        b = np.take(m, range(0, m.shape[ax] - 1), axis=ax)
        n += np.count_nonzero(a != b)
    return n


@pytest.mark.parametrize("dtype", ["f32", "i32"])
def test_c1_stencil_reduce_closed_form(dtype):
    # sum over active cells of the Laplacian of the indicator = -(# active/inactive faces)
    p = W.c1_program(dtype=dtype)
    o = oracle.run_program(p)
    i, j = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    disk = (i + .5 - 32) ** 2 + (j + .5 - 32) ** 2 < 24 ** 2
    expect = -_boundary_faces(disk)
    assert expect == -192
    assert o.field(p["layout"].fields["s"]) == expect
    # eager lowering counts (readings R3/R5/R19)
    assert (o.tasks_eager_folded, o.tasks_eager_faithful) == (8, 11)


def test_stencil_3d_closed_form_block_ball():
    L, lv = W.c2_layout(ptr=2)
    coords = W.block_ball_coords(8, 8, 20.0)
    o = oracle.Oracle(L.desc())
    f = L.fields
    o.call(W.activate(f["b"], coords))
    o.call(W.struct_for("FILL", lv[-1], [f["x0"]], [1.0]))
    o.call(W.struct_for("STENCIL", lv[-1], [f["x1"], f["x0"]]))
    o.call(W.serial("CLEAR_SCALAR", [f["s"]]))
    o.call(W.struct_for("REDUCE_SUM", lv[-1], [f["s"], f["x1"]]))
    act = np.zeros((64, 64, 64), dtype=bool)
    for c in coords:
        act[c[0]:c[0] + 8, c[1]:c[1] + 8, c[2]:c[2] + 8] = True
    assert o.field(f["s"]) == -_boundary_faces(act)


def test_jacobi_isolated_block_is_textbook_dirichlet_jacobi():
    # An isolated 8^3 block with inactive surroundings = dense 8^3 Dirichlet
    # problem; compare with the matrix form x <- x + D^-1 (b - A x), A = 7-point
    # Laplacian assembled with scipy.sparse kron sums.
    L, lv = W.c2_layout(ptr=2)
    o = oracle.Oracle(L.desc())
    f = L.fields
    o.call(W.activate(f["b"], np.array([[8, 16, 24]], dtype=np.int32)))
    o.call(W.struct_for("FILL", lv[-1], [f["b"]], [1.0]))
    o.call(W.struct_for("FILL", lv[-1], [f["x0"]], [0.0]))
    src, dst = f["x0"], f["x1"]
    for _ in range(20):
        o.call(W.struct_for("JACOBI", lv[-1], [dst, src, f["b"]]))
        src, dst = dst, src
    got = o.field(src)[8:16, 16:24, 24:32]
    T = sp.diags([-np.ones(7), 2 * np.ones(8), -np.ones(7)], [-1, 0, 1])
    I8 = sp.identity(8)
    A = (sp.kron(sp.kron(T, I8), I8) + sp.kron(sp.kron(I8, T), I8) + sp.kron(sp.kron(I8, I8), T)).tocsr()
    x = np.zeros(512)
    b = np.ones(512)
    res = []
    for _ in range(20):
        x = x + (b - A @ x) / 6.0
        res.append(np.linalg.norm(b - A @ x))
    np.testing.assert_allclose(got.ravel(), x, rtol=1e-5, atol=0)
    assert all(r2 <= r1 * (1 + 1e-12) for r1, r2 in zip(res, res[1:]))   # non-increasing residual
    assert not o.field(src)[:8].any()                                   # nothing leaks outside


# ---------------------------------------------------------------------------
# Listgen soundness / completeness (brute force exhaustive scan)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(25))
def test_listgen_equals_exhaustive_scan(seed):
    rng = np.random.default_rng(seed)
    L, main, half = W.fuzz_layout(rng)
    o = oracle.Oracle(L.desc())
    shape = L.shape("a")
    k = int(rng.integers(1, 20))
    cells = np.stack([rng.integers(0, s, size=k) for s in shape], axis=1).astype(np.int32)
    o.activate(0, cells)
    from brute import Brute
    b = Brute(L.desc())
    b.activate_cells(b.levels_of_field(0), cells)
    sparse = [s for s in main if L.rows[s][0] in (W.BITMASKED, W.POINTER)]
    for s in sparse:                        # listgen top-down: each parent list current
        o.listgen(s)
    for s in sparse:
        got = o.list(s)
        # exhaustive scan: level cells set in their own mask AND under active ancestors
        want = np.argwhere(b.active(main[: main.index(s) + 1]))
        assert got.tolist() == want.tolist(), (s, got, want)
        assert np.array_equal(o.mask(s), b.mask(s))


# ---------------------------------------------------------------------------
# T0: oracle == brute-force dense checker on random integer programs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(200))
def test_oracle_matches_brute_force(seed):
    p = W.fuzz_program(seed)
    o = oracle.run_program(p)
    b = brute_run(p)
    L = p["layout"]
    for name, fid in L.fields.items():
        got = o.field(fid)
        want = b.read(fid)
        assert np.array_equal(got, want), (seed, name)
    for s in range(1, len(L.rows)):
        if L.rows[s][0] in (W.BITMASKED, W.POINTER):
            assert np.array_equal(o.mask(s), b.mask(s)), (seed, s)
